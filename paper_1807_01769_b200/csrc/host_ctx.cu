// host_ctx.cu -- context helpers of libskgpu (see host_ctx.h): NCCL binding,
// error state, twiddle and integrating-factor tables, kernel arguments and
// the state I/O between the reference layout and the internal layouts.
#include "host_ctx.h"

#include <nvtx3/nvToolsExt.h>

namespace skh {

// NCCL is loaded on first use (multi-GPU contexts only) instead of at link
// time: a process that imports PyTorch after this library would otherwise
// bind torch's NCCL symbols to whichever libnccl.so.2 came first.  When torch
// is already loaded, dlopen returns its (newer) NCCL.
const char* nccl_unloaded_error(ncclResult_t) { return "NCCL not loaded"; }

NcclApi load_nccl() {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    a.GetErrorString = nccl_unloaded_error;
    if (!h) {
        const char* e = dlerror();
        a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
        return a;
    }
    bool ok = true;
    auto sym = [&](auto& f, const char* name) {
        f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
        if (!f) ok = false;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GetErrorString, "ncclGetErrorString");
    if (!a.GetErrorString) a.GetErrorString = nccl_unloaded_error;
    a.ok = ok;
    if (!ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
}

NcclApi& nccl() {
    static NcclApi a = load_nccl();
    return a;
}

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}



// W_n^m = exp(-2 pi i m / n), m in [0, n), in extended precision.
std::vector<cd> twiddles(int n) {
    std::vector<cd> w(n);
    const long double tp = 6.283185307179586476925286766559005768L;
    for (int m = 0; m < n; ++m) {
        long double a = tp * (long double)m / (long double)n;
        w[m] = make_double2((double)cosl(a), (double)-sinl(a));
    }
    return w;
}

// Largest |signed index| kept by the dealias rule |k_d| <= kcut_d of
// make_grid (grid.cpp:78-100), evaluated with the same double arithmetic.
int cut_index(int n, double L, double coef, bool half) {
    const double spacing = skh::kTwoPi / L;
    const double kcut = coef * (skh::kTwoPi / L) * (n / 2);
    int best = -1;
    const int hi = half ? n / 2 : n / 2;
    for (int i = 0; i <= hi; ++i)
        if (std::abs(spacing * i) <= kcut) best = i;
    // negative indices -(n/2-1)..-1 mirror the positive ones for |k|
    return best;
}

cudaEvent_t take_event(skg_ctx* c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void timing_hook(void* user, int cls, int phase, double bytes) {
    auto* c = static_cast<skg_ctx*>(user);
    cudaEvent_t e = take_event(c);
    cudaEventRecord(e, c->stream);
    if (phase == 0) {
        c->cur = e;
    } else {
        c->pend.push_back({c->cur, e, cls, bytes});
        c->cur = nullptr;
    }
}

// SKG_NVTX=1: an NVTX range around every pass of the step (named by kernel
// class, visible in Nsight Systems / ncu --nvtx), on top of the per-class
// CUDA-event timing when that is on.  nvtx3 is header-only and a no-op
// without an attached tool.
void nvtx_hook(void* user, int cls, int phase, double bytes) {
    static const char* const names[6] = {"skg x_inverse", "skg physical", "skg x_forward_rk",
                                         "skg y_inverse", "skg exchange", "skg y_forward"};
    auto* c = static_cast<skg_ctx*>(user);
    if (phase == 0) nvtxRangePushA(names[cls >= 0 && cls < 6 ? cls : 1]);
    if (c->timing) timing_hook(user, cls, phase, bytes);
    if (phase != 0) nvtxRangePop();
}

skg::LaunchHook hook_of(skg_ctx* c) {
    static const bool nvtx = [] {
        const char* e = std::getenv("SKG_NVTX");
        return e && std::atoi(e) != 0;
    }();
    skg::LaunchHook h;
    if (nvtx) {
        h.fn = nvtx_hook;
        h.user = c;
    } else if (c->timing) {
        h.fn = timing_hook;
        h.user = c;
    }
    return h;
}

void harvest(skg_ctx* c) {
    for (auto& p : c->pend) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            c->st_ms[p.cls] += ms;
            c->st_n[p.cls] += 1;
            c->st_bytes[p.cls] += p.bytes;
        }
        c->pool.push_back(p.a);
        c->pool.push_back(p.b);
    }
    c->pend.clear();
}

int refresh_exp(skg_ctx* c, double dt) {
    if (dt == c->cached_dt) return SKG_OK;
    // Separable factors: exp(h sigma) = prod_d exp(h (-nu k_d^2)) with
    // sigma = -nu |k|^2 (simulation.cpp:147-157, time_stepping.cpp:49-52).
    const int d = c->dims;
    int ext[3];
    for (int a = 0; a < d; ++a) ext[a] = a == d - 1 ? c->nh : c->n[a];
    std::vector<double> tab;
    for (int which = 0; which < 2; ++which) {
        const double hdt = which == 0 ? 0.5 * dt : dt;
        for (int a = 0; a < d; ++a) {
            for (int i = 0; i < ext[a]; ++i) {
                const int si = a == d - 1 ? i : skg::signed_index(i, c->n[a]);
                const double kv = c->kscale[a] * si;
                tab.push_back(std::exp(hdt * (-c->nu * (kv * kv))));
            }
        }
    }
    CUDA_TRY(cudaMemcpyAsync(c->etab, tab.data(), tab.size() * sizeof(double),
                             cudaMemcpyHostToDevice, c->stream));
    c->cached_dt = dt;
    return SKG_OK;
}

const double* etab_ptr(const skg_ctx* c, int which, int axis) {
    int off = 0;
    int ext[3];
    for (int a = 0; a < c->dims; ++a) ext[a] = a == c->dims - 1 ? c->nh : c->n[a];
    int per = 0;
    for (int a = 0; a < c->dims; ++a) per += ext[a];
    off = which * per;
    for (int a = 0; a < axis; ++a) off += ext[a];
    return c->etab + off;
}

int env_opt() {
    static const int v = [] {
        const char* e = std::getenv("SKG_OPT");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

int sm_count(int device) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

skg::Ns2dArgs args2d(skg_ctx* c, double dt) {
    skg::Ns2dArgs a{};
    a.opt = env_opt();
    a.wave = 2 * c->nsm;
    a.nx = c->n[0];
    a.ny = c->n[1];
    a.nh = c->nh;
    a.kcx = c->kc[0];
    a.kcy = c->kc[1];
    a.pruned = c->pruned ? 1 : 0;
    a.ky_in = c->pruned ? c->kc[1] + 1 : c->nh;
    a.ld_i = a.ky_in;
    a.ld_o = c->kc[1] + 1;
    a.has_sigma = c->nu != 0.0;
    a.rk2 = c->scheme == SKG_RK2;
    a.kx_scale = c->kscale[0];
    a.ky_scale = c->kscale[1];
    a.inv_n = 1.0 / (double)c->P;
    a.dt = dt;
    a.hdt = 0.5 * dt;
    a.sdt = dt / 6.0;
    a.e1x = etab_ptr(c, 0, 0);
    a.e1y = etab_ptr(c, 0, 1);
    a.e2x = etab_ptr(c, 1, 0);
    a.e2y = etab_ptr(c, 1, 1);
    a.dyn = c->adaptive ? c->d_dyn : nullptr;
    a.force = c->forcing ? (c->f_cm ? c->f_cm : c->f_ref) : nullptr;
    a.u = c->u;
    a.k1 = c->k[0];
    a.k2 = c->k[1];
    a.k3 = c->k[2];
    const size_t isz = (size_t)c->n[0] * c->nh;
    for (int m = 0; m < 4; ++m) a.I[m] = c->inter + m * isz;
    a.nl = c->inter + 4 * isz;
    a.twx = c->tw[0];
    a.twy = c->tw[1];
    a.flags = c->flags;
    a.diag = c->diag;
    a.nu = c->nu;
    // one partition covering everything: send and receive buffers alias
    a.G = 1;
    a.r = 0;
    a.lead = 1;
    a.c0 = 0;
    a.ncols = c->kc[1] + 1;
    a.nrl = c->n[0];
    a.lg_nrl = 0;
    while ((1 << a.lg_nrl) < a.nrl) ++a.lg_nrl;
    a.kowner = c->d_kowner;
    a.cstart = c->d_cstart;
    a.sI[0] = a.rI[0] = a.I[0];
    a.sI[1] = a.rI[1] = a.I[1];
    a.sA[0] = a.rA[0] = a.I[2];
    a.sA[1] = a.rA[1] = a.I[3];
    return a;
}

skg::Ns2dArgs args2d_part(skg_ctx* c, double dt, const Part& p) {
    skg::Ns2dArgs a = args2d(c, dt);
    a.u = p.u;
    a.k1 = p.k[0];
    a.k2 = p.k[1];
    a.k3 = p.k[2];
    a.G = c->G;
    a.r = p.r;
    a.c0 = p.c0;
    a.ncols = p.ncols;
    a.nrl = c->nrl;
    a.lg_nrl = 0;
    while ((1 << a.lg_nrl) < a.nrl) ++a.lg_nrl;
    for (int f = 0; f < 2; ++f) {
        a.sI[f] = p.sI[f];
        a.rI[f] = p.rI[f];
        a.sA[f] = p.sA[f];
        a.rA[f] = p.rA[f];
    }
    a.p2p = c->p2p ? 1 : 0;
    if (c->p2p)
        for (int q = 0; q < c->G; ++q)
            for (int f = 0; f < 2; ++f) {
                a.peer_rI[q][f] = c->peer_rI[q][f];
                a.peer_rA[q][f] = c->peer_rA[q][f];
            }
    return a;
}

skg::Ns3dArgs args3d(skg_ctx* c, double dt) {
    skg::Ns3dArgs a{};
    a.opt = env_opt();
    a.wave = 2 * c->nsm;
    a.nx = c->n[0];
    a.ny = c->n[1];
    a.nz = c->n[2];
    a.nh = c->nh;
    a.kcx = c->kc[0];
    a.kcy = c->kc[1];
    a.kcz = c->kc[2];
    a.pruned = c->pruned ? 1 : 0;
    a.has_sigma = c->nu != 0.0;
    a.rk2 = c->scheme == SKG_RK2;
    a.kz_in = c->pruned ? c->kc[2] + 1 : c->nh;
    a.kz_o = c->kc[2] + 1;
    a.ky_lines = c->pruned ? 2 * c->kc[1] + 1 : c->n[1];
    a.kx_scale = c->kscale[0];
    a.ky_scale = c->kscale[1];
    a.kz_scale = c->kscale[2];
    a.inv_n = 1.0 / (double)c->P;
    a.dt = dt;
    a.hdt = 0.5 * dt;
    a.sdt = dt / 6.0;
    a.e1x = etab_ptr(c, 0, 0);
    a.e1y = etab_ptr(c, 0, 1);
    a.e1z = etab_ptr(c, 0, 2);
    a.e2x = etab_ptr(c, 1, 0);
    a.e2y = etab_ptr(c, 1, 1);
    a.e2z = etab_ptr(c, 1, 2);
    a.dyn = c->adaptive ? c->d_dyn : nullptr;
    a.force = c->forcing ? c->f_ref : nullptr;
    a.u = c->u;
    a.k1 = c->k[0];
    a.k2 = c->k[1];
    a.k3 = c->k[2];
    a.vstride = (size_t)c->S;
    a.fstride = (size_t)c->n[0] * c->n[1] * c->nh;
    a.A = c->inter;
    a.B = c->inter + 5 * a.fstride;
    a.twx = c->tw[0];
    a.twy = c->tw[1];
    a.twz = c->tw[2];
    a.flags = c->flags;
    a.diag = c->diag;
    a.nu = c->nu;
    a.G = 1;
    a.r = 0;
    a.lead = 1;
    a.kys = 0;
    a.nkyl = a.ky_lines;
    a.nrl = a.nx;
    a.ystate = a.ny;
    a.kowner = c->d_kowner;
    a.kstart = c->d_cstart;
    a.slab = 0;
    a.sz = c->nh;
    a.xscr = c->xscr;
    a.xscr_mask = c->xscr_mask;
    a.xscr_nsm = c->xscr_nsm;
    return a;
}

skg::Ns3dArgs args3d_part(skg_ctx* c, double dt, const Part& p) {
    skg::Ns3dArgs a = args3d(c, dt);
    a.u = p.u;
    a.k1 = p.k[0];
    a.k2 = p.k[1];
    a.k3 = p.k[2];
    a.vstride = p.vs;
    a.fstride = p.fs;
    a.A = p.A3;
    a.B = p.B3;
    a.rA = p.rA3;
    a.sD = p.sD3;
    a.rfs = p.rfs;
    a.G = c->G;
    a.r = p.r;
    a.lead = &p == c->parts.data() ? 1 : 0;  // the process's first part counts the steps
    a.kys = p.c0;
    a.nkyl = p.ncols;
    a.nrl = c->nrl;
    a.ystate = p.ncols;
    a.slab = 1;
    // kz range of this part (all kept kz unless the pencil layout splits them)
    a.sz = p.nkz;
    a.kz_in = a.kz_o = p.nkz;
    a.kz0 = p.kz0;
    a.e1z += p.kz0;
    a.e2z += p.kz0;
    a.p2p = c->p2p ? 1 : 0;
    if (c->p2p) {
        a.rD = p.rD3;
        a.dfs = c->dfs3;
        for (int q = 0; q < c->G; ++q) {  // peers along the ky / x split: same pz
            a.peer_rA[q] = c->peer_rA3[q * c->Pz + p.pz];
            a.peer_D[q] = c->peer_D3[q * c->Pz + p.pz];
        }
    }
    return a;
}

// launch_energy's metric/layout code: ns2d CM layout 1, ns2d reference layout 2, ns3d 0
int energy_mode(const skg_ctx* c) { return c->solver == 2 ? (c->generic ? 2 : 1) : 0; }

skg::GenArgs args_gen(skg_ctx* c, double dt) {
    skg::GenArgs a{};
    a.dims = c->dims;
    for (int d = 0; d < 3; ++d) {
        a.n[d] = c->n[d];
        a.kc[d] = c->kc[d];
        a.ks[d] = c->kscale[d];
    }
    a.nh = c->nh;
    a.S = c->S;
    a.P = c->P;
    a.nvars = c->nvars;
    a.has_sigma = c->nu != 0.0;
    a.rk2 = c->scheme == SKG_RK2;
    a.dt = dt;
    a.hdt = 0.5 * dt;
    a.sdt = dt / 6.0;
    a.dyn = c->adaptive ? c->d_dyn : nullptr;
    for (int d = 0; d < c->dims; ++d) {
        a.e1[d] = etab_ptr(c, 0, d);
        a.e2[d] = etab_ptr(c, 1, d);
    }
    a.u = c->u;
    a.k1 = c->k[0];
    a.k2 = c->k[1];
    a.k3 = c->k[2];
    a.flags = c->flags;
    a.force = c->forcing ? c->f_ref : nullptr;
    return a;
}

skg::ForceGeo force_geo(const skg_ctx* c) {
    skg::ForceGeo g{};
    g.dims = c->dims;
    double Lmax = 0.0;
    for (int d = 0; d < c->dims; ++d) {
        g.n[d] = c->n[d];
        g.kc[d] = c->kc[d];
        g.ks[d] = c->kscale[d];
        Lmax = std::max(Lmax, c->L[d]);
    }
    g.nh = c->nh;
    g.nvars = c->nvars;
    g.S = c->S;
    g.delta_k = skh::kTwoPi / Lmax;  // grid.cpp:65
    g.k_lo = c->f_klo;
    g.k_hi = c->f_khi;
    return g;
}

int store_state_to_io(skg_ctx* c, const cd* src);


int decide_pruned(skg_ctx* c, const cd* d_ref_layout) {
    // fast path iff every masked-out mode of every variable is exactly zero
    CUDA_TRY(skg::launch_count_masked(d_ref_layout, c->dims, c->n, c->kc, c->nvars, c->S,
                                      c->d_count, c->stream, &c->launches));
    unsigned long long cnt = 0;
    CUDA_TRY(cudaMemcpyAsync(&cnt, c->d_count, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->pruned = cnt == 0;
    return SKG_OK;
}

// ns3d slab <-> reference layout: the compact lines [c0, c0 + ncols) of a
// part are at most two runs of global ky (positive, then negative ky).
int copy_slab3(skg_ctx* c, const Part& p, bool to_part) {
    const int kcy = c->kc[1], ny = c->n[1], nx = c->n[0];
    const size_t nh = (size_t)c->nh, kzc = (size_t)p.nkz;  // the part's kz range [kz0, kz0 + nkz)
    const int runs[2][2] = {{0, kcy + 1}, {kcy + 1, 2 * kcy + 1}};  // compact ranges
    for (int b = 0; b < 2; ++b) {
        const int lo = std::max(runs[b][0], p.c0), hi = std::min(runs[b][1], p.c0 + p.ncols);
        if (lo >= hi) continue;
        const int gy = b == 0 ? lo : lo + ny - (2 * kcy + 1);
        for (int v = 0; v < 3; ++v) {
            // kept kz of lines [gy, gy + hi - lo) for every kx: (kz, line, kx) boxes
            cd* io = c->io + (size_t)v * c->S + (size_t)gy * nh + p.kz0;
            cd* st = p.u + (size_t)v * p.vs + (size_t)(lo - p.c0) * kzc;
            cudaPitchedPtr pio = make_cudaPitchedPtr(io, nh * sizeof(cd), kzc * sizeof(cd), ny);
            cudaPitchedPtr pst = make_cudaPitchedPtr(st, kzc * sizeof(cd), kzc * sizeof(cd), p.ncols);
            cudaMemcpy3DParms m{};
            m.srcPtr = to_part ? pio : pst;
            m.dstPtr = to_part ? pst : pio;
            m.extent = make_cudaExtent(kzc * sizeof(cd), hi - lo, nx);
            m.kind = cudaMemcpyDeviceToDevice;
            CUDA_TRY(cudaMemcpy3DAsync(&m, c->stream));
        }
    }
    return SKG_OK;
}

// reference layout (io) -> internal state
int load_state_from_io(skg_ctx* c) {
    int rc = decide_pruned(c, c->io);
    if (rc) return rc;
    if (c->dist) {
        if (!c->pruned)
            return fail(SKG_EUNSUPPORTED,
                        "slab-decomposed contexts need a dealiased state (masked modes exactly 0)");
        if (c->solver == 3) {
            for (const Part& p : c->parts) {
                int rc2 = copy_slab3(c, p, true);
                if (rc2) return rc2;
            }
            return SKG_OK;
        }
        CUDA_TRY(skg::launch_transpose_c(c->io, c->cmfull, c->n[0], c->nh, 0, c->stream, &c->launches));
        for (const Part& p : c->parts)
            if (p.ncols)
                CUDA_TRY(cudaMemcpyAsync(p.u, c->cmfull + (size_t)p.c0 * c->n[0],
                                         sizeof(cd) * p.ncols * c->n[0], cudaMemcpyDeviceToDevice, c->stream));
        return SKG_OK;
    }
    if (c->solver == 2 && !c->generic) {
        CUDA_TRY(skg::launch_transpose_c(c->io, c->u, c->n[0], c->nh, 0, c->stream, &c->launches));
    } else {
        CUDA_TRY(cudaMemcpyAsync(c->u, c->io, sizeof(cd) * c->S * c->nvars,
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    return SKG_OK;
}

int store_state_to_io(skg_ctx* c, const cd* src) {
    if (c->dist && c->solver == 3) {  // gather the slabs (masked lines are exactly 0)
        CUDA_TRY(cudaMemsetAsync(c->io, 0, sizeof(cd) * c->S * 3, c->stream));
        for (const Part& p : c->parts) {
            int rc2 = copy_slab3(c, p, false);
            if (rc2) return rc2;
        }
        if (c->comm) {
            const ncclResult_t nr = nccl().AllReduce(c->io, c->io, 2 * 3 * (size_t)c->S, ncclDouble,
                                                  ncclSum, c->comm, c->stream);
            if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
        }
        return SKG_OK;
    }
    if (c->dist) {  // gather the slabs (masked columns are exactly 0)
        CUDA_TRY(cudaMemsetAsync(c->cmfull, 0, sizeof(cd) * c->S, c->stream));
        for (const Part& p : c->parts)
            if (p.ncols)
                CUDA_TRY(cudaMemcpyAsync(c->cmfull + (size_t)p.c0 * c->n[0], p.u,
                                         sizeof(cd) * p.ncols * c->n[0], cudaMemcpyDeviceToDevice, c->stream));
        if (c->comm) {
            const ncclResult_t nr = nccl().AllReduce(c->cmfull, c->cmfull, 2 * (size_t)c->S, ncclDouble,
                                                  ncclSum, c->comm, c->stream);
            if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
        }
        CUDA_TRY(skg::launch_transpose_c(c->cmfull, c->io, c->nh, c->n[0], 0, c->stream, &c->launches));
        return SKG_OK;
    }
    if (c->solver == 2 && !c->generic) {
        CUDA_TRY(skg::launch_transpose_c(src, c->io, c->nh, c->n[0], 0, c->stream, &c->launches));
    } else {
        CUDA_TRY(cudaMemcpyAsync(c->io, src, sizeof(cd) * c->S * c->nvars, cudaMemcpyDeviceToDevice,
                                 c->stream));
    }
    return SKG_OK;
}

// physical-space and scratch buffers of the transform operators and the
// grid dump, allocated on first use (the step itself never needs them)
int ensure_fft_bufs(skg_ctx* c) {
    if (c->phys && c->work) return SKG_OK;
    CUDA_TRY(skg::dmalloc(&c->phys, sizeof(double) * (size_t)c->P));
    CUDA_TRY(skg::dmalloc(&c->work, sizeof(cd) * (size_t)c->S));
    return SKG_OK;
}

// ns3d peer exchange: the y-forward receive buffers (B stays private)
int ensure_p2p_bufs(skg_ctx* c) {
    if (c->solver != 3) return SKG_OK;
    size_t maxcols = 0;
    for (int q = 0; q < c->G; ++q) maxcols = std::max(maxcols, (size_t)(c->cstart[q + 1] - c->cstart[q]));
    size_t maxkz = 0;
    for (int z = 0; z < c->Pz; ++z) maxkz = std::max(maxkz, (size_t)(c->zstart[z + 1] - c->zstart[z]));
    c->dfs3 = (size_t)c->n[0] * maxcols * maxkz;
    for (Part& p : c->parts)
        if (!p.rD3) CUDA_TRY(skg::dmalloc(&p.rD3, sizeof(cd) * 3 * c->dfs3));
    return SKG_OK;
}

struct TwCache {
    std::mutex mu;
    std::map<std::pair<int, int>, cd*> tabs;  // (device, n) -> table
} g_tw;

cd* twiddle_table(int device, int n) {
    std::lock_guard<std::mutex> lk(g_tw.mu);
    auto key = std::make_pair(device, n);
    auto it = g_tw.tabs.find(key);
    if (it != g_tw.tabs.end()) return it->second;
    std::vector<cd> w = twiddles(n);
    cd* d = nullptr;
    if (skg::dmalloc(&d, sizeof(cd) * n) != cudaSuccess) return nullptr;
    cudaMemcpy(d, w.data(), sizeof(cd) * n, cudaMemcpyHostToDevice);
    g_tw.tabs[key] = d;
    return d;
}

}  // namespace skh
