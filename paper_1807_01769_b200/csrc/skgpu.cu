// skgpu.cu -- context, device memory and the extern "C" boundary (include/skgpu.h).
//
// Mirrors the reference's Simulation / ExactLinStepper / Solver contract
// (proj/src/simulation.cpp:297-590, proj/src/time_stepping.cpp:72-194) for a
// device-resident state.  The host side only validates arguments, builds the
// small per-axis tables (twiddles, exp factors, dealias cut indices) and
// enqueues kernels; every per-mode operation runs in sm_100a kernels.  There is
// no CPU fallback: a missing device or an unsupported extent is an error.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <random>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>
#include <type_traits>

#include "../../include/skgpu.h"
#include "skg_internal.h"

using skg::cd;

namespace {

// NCCL is loaded on first use (multi-GPU contexts only) instead of at link
// time: a process that imports PyTorch after this library would otherwise
// bind torch's NCCL symbols to whichever libnccl.so.2 came first.  When torch
// is already loaded, dlopen returns its (newer) NCCL.
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&::ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&::ncclCommInitRank) CommInitRank = nullptr;
    decltype(&::ncclCommDestroy) CommDestroy = nullptr;
    decltype(&::ncclGroupStart) GroupStart = nullptr;
    decltype(&::ncclGroupEnd) GroupEnd = nullptr;
    decltype(&::ncclSend) Send = nullptr;
    decltype(&::ncclRecv) Recv = nullptr;
    decltype(&::ncclAllReduce) AllReduce = nullptr;
    decltype(&::ncclGetErrorString) GetErrorString = nullptr;
};

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

}  // namespace

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(SKG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr double kTwoPi = 6.283185307179586476925286766559;  // grid.cpp:11

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
    const double spacing = kTwoPi / L;
    const double kcut = coef * (kTwoPi / L) * (n / 2);
    int best = -1;
    const int hi = half ? n / 2 : n / 2;
    for (int i = 0; i <= hi; ++i)
        if (std::abs(spacing * i) <= kcut) best = i;
    // negative indices -(n/2-1)..-1 mirror the positive ones for |k|
    return best;
}

}  // namespace

// One slab of the decomposed state.  ns2d (see Ns2dArgs): owned kept ky
// columns [c0, c0 + ncols) in CM layout and the exchange buffers.  ns3d (see
// Ns3dArgs): owned compact kept ky lines [c0, c0 + ncols) of the state
// ([kx][kyl][kz], 3 components of vs elements), the x-pass/y-pass
// intermediates A (5 fields) / B (6 fields) of fs elements each, and the
// receive (rA) / send (sD) blocks of the two all-to-alls (rfs per field).
struct Part {
    int r = 0;
    int c0 = 0, ncols = 0;
    cd* u = nullptr;
    cd* k[3] = {nullptr, nullptr, nullptr};
    cd* sI[2] = {nullptr, nullptr};
    cd* rI[2] = {nullptr, nullptr};
    cd* sA[2] = {nullptr, nullptr};
    cd* rA[2] = {nullptr, nullptr};
    cd* A3 = nullptr;
    cd* B3 = nullptr;
    cd* rA3 = nullptr;
    cd* sD3 = nullptr;
    size_t vs = 0, fs = 0, rfs = 0;
};

struct skg_ctx {
    int device = 0;
    int nsm = 148;
    int solver = 2;  // 2: ns2d, 3: ns3d
    int dims = 2;
    int n[3] = {1, 1, 1};
    double L[3] = {kTwoPi, kTwoPi, kTwoPi};
    double coef = 2.0 / 3.0;
    double nu = 0.0;
    int scheme = SKG_RK4;
    int nvars = 1;
    int nh = 0;
    int kc[3] = {0, 0, 0};
    double kscale[3] = {1, 1, 1};
    long long S = 0, P = 0;

    cudaStream_t own = nullptr, stream = nullptr;
    long launches = 0;

    // device buffers
    cd* u = nullptr;      // nvars * S (2D: CM layout; 3D: reference layout)
    cd* k[3] = {nullptr, nullptr, nullptr};
    cd* inter = nullptr;  // intermediates
    size_t inter_elems = 0;
    cd* io = nullptr;     // nvars * S staging in reference layout
    double* phys = nullptr;
    cd* work = nullptr;
    double* etab = nullptr;  // e1[axis], e2[axis] tables
    cd* tw[3] = {nullptr, nullptr, nullptr};
    skg::DevFlags* flags = nullptr;
    unsigned long long* d_count = nullptr;
    double* d_red = nullptr;

    bool pruned = false;
    double cached_dt = -1.0;
    long it = 0;
    double t = 0.0;
    long div_it = -1;
    int div_var = -1;
    long pending_steps = 0;
    double pending_dt = 0.0;

    // slab decomposition (ns2d): G partitions; `parts` are the ones this
    // process runs (all G in the single-process test mode, one with NCCL)
    bool dist = false;
    int G = 1, grank = 0, nrl = 0;
    std::vector<int> cstart;  // G + 1 entries
    std::vector<Part> parts;
    int* d_kowner = nullptr;
    int* d_cstart = nullptr;
    cd* cmfull = nullptr;     // full CM staging for set/get_state
    ncclComm_t comm = nullptr;
    double* diag = nullptr;   // per-step (E, Z, eps) series of skg_run (device)

    // per-kernel-class event timing (skg_set_timing)
    struct Pending {
        cudaEvent_t a, b;
        int cls;
        double bytes;
    };
    bool timing = false;
    std::vector<cudaEvent_t> pool;
    std::vector<Pending> pend;
    cudaEvent_t cur = nullptr;
    double st_ms[6] = {0, 0, 0, 0, 0, 0};
    long st_n[6] = {0, 0, 0, 0, 0, 0};
    double st_bytes[6] = {0, 0, 0, 0, 0, 0};

    // CUDA graph of one RK step (all stage kernels), replayed per step when
    // timing is off; recaptured when dt, the fast-path decision or the
    // stream change.
    cudaGraphExec_t gexec = nullptr;
    double* g_diag = nullptr;

    // generic path (extents outside the fused kernels' range, generic.cu)
    bool generic = false;
    skg::GenScratch gs{};

    // random band forcing (skg_set_forcing): host generator of the reference
    bool forcing = false;
    double f_klo = 2.0, f_khi = 4.0, f_rate = 1.0;
    std::mt19937_64 f_rng;
    cd* f_ref = nullptr;       // nvars S, reference layout
    cd* f_cm = nullptr;        // ns2d fused kernels: CM layout copy
    double* f_noise = nullptr; // pinned host, nvars P
    double* f_red = nullptr;   // device: reductions, coefficients, injection
    double last_injection = 0.0;
    long forcing_fallbacks = 0;

    // adaptive (CFL) dt: skg_set_cfl
    bool adaptive = false;
    double cfl = 0.5, dt_max = 0.1, t_end = -1.0, last_dt = 0.0;
    skg::DynStep* d_dyn = nullptr;
    double g_dt = 0.0;
    long g_launches = 0;
    bool g_pruned = false;
    cudaStream_t g_stream = nullptr;
};

namespace {

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

skg::LaunchHook hook_of(skg_ctx* c) {
    skg::LaunchHook h;
    if (c->timing) {
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
    std::vector<double> h;
    int off = 0;
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
    (void)off;
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
    a.lead = p.r == 0 ? 1 : 0;
    a.kys = p.c0;
    a.nkyl = p.ncols;
    a.nrl = c->nrl;
    a.ystate = p.ncols;
    a.slab = 1;
    a.sz = c->kc[2] + 1;
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
    g.delta_k = kTwoPi / Lmax;  // grid.cpp:65
    g.k_lo = c->f_klo;
    g.k_hi = c->f_khi;
    return g;
}

int store_state_to_io(skg_ctx* c, const cd* src);

// Simulation::refresh_forcing (simulation.cpp:482-533) before a step: the
// reference's generator fills the white noise on the host (one
// normal_distribution per variable, random_field grid.cpp:285-288), the rest
// runs on the device (forcing.cu).
int refresh_forcing(skg_ctx* c) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));  // the pinned noise buffer is reused
    const size_t P = (size_t)c->P;
    const cd* tw[3] = {c->tw[0], c->tw[1], c->tw[2]};
    for (int v = 0; v < c->nvars; ++v) {
        std::normal_distribution<double> gauss(0.0, 1.0);
        double* h = c->f_noise + v * P;
        for (size_t i = 0; i < P; ++i) h[i] = gauss(c->f_rng);
    }
    const skg::ForceGeo g = force_geo(c);
    for (int v = 0; v < c->nvars; ++v) {
        CUDA_TRY(cudaMemcpyAsync(c->phys, c->f_noise + v * P, sizeof(double) * P, cudaMemcpyHostToDevice,
                                 c->stream));
        CUDA_TRY(skg::fft_forward_dev(c->dims, c->n, c->phys, c->f_ref + (size_t)v * c->S, c->work, tw,
                                      c->stream, &c->launches));
    }
    CUDA_TRY(skg::forcing_shape(g, c->f_ref, c->stream, &c->launches));
    const cd* uref = c->u;
    if (c->f_cm) {  // ns2d fused kernels keep the state in CM layout
        int rc = store_state_to_io(c, c->u);
        if (rc) return rc;
        uref = c->io;
    }
    CUDA_TRY(skg::forcing_finish(g, uref, c->f_ref, c->f_rate, c->f_red, c->stream, &c->launches));
    if (c->f_cm)
        CUDA_TRY(skg::launch_transpose_c(c->f_ref, c->f_cm, c->n[0], c->nh, 0, c->stream, &c->launches));
    return SKG_OK;
}

int sync_and_check(skg_ctx* c, long nsteps, double dt) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    harvest(c);
    skg::DevFlags f;
    CUDA_TRY(cudaMemcpy(&f, c->flags, sizeof(f), cudaMemcpyDeviceToHost));
    if (c->forcing) {
        double r[8];
        CUDA_TRY(cudaMemcpy(r, c->f_red, sizeof(r), cudaMemcpyDeviceToHost));
        c->last_injection = r[6];
    }
    skg::DynStep dyn{};
    if (c->adaptive) {
        CUDA_TRY(cudaMemcpy(&dyn, c->d_dyn, sizeof(dyn), cudaMemcpyDeviceToHost));
        c->last_dt = dyn.last_dt;
    }
    if (f.bad_dt) {  // compute_dt gave dt <= 0 (past t_end): the step did not run
        c->it += f.div_step - 1;
        c->t = dyn.t;
        return fail(SKG_ECONFIG, "step: nonpositive dt (past t_end?)");
    }
    if (f.diverged) {
        const long done = f.div_step;
        if (c->adaptive) c->t = dyn.t;
        else
            for (long i = 0; i < done; ++i) c->t += dt;
        c->it += done;
        c->div_it = c->it;
        c->div_var = f.div_var;
        static const char* keys2[] = {"rot_fft"};
        static const char* keys3[] = {"vx_fft", "vy_fft", "vz_fft"};
        const char* key = c->solver == 2 ? keys2[0] : keys3[f.div_var >= 0 && f.div_var < 3 ? f.div_var : 0];
        return fail(SKG_EDIVERGENCE, std::string("non-finite value in field '") + key +
                                         "' at iteration " + std::to_string(c->it));
    }
    if (c->adaptive) {
        c->t = dyn.t;
    } else {
        for (long i = 0; i < nsteps; ++i) c->t += dt;
        if (nsteps > 0) c->last_dt = dt;
    }
    c->it += nsteps;
    return SKG_OK;
}

// All-to-all of the slab decomposition.  which = 0: x-inverse outputs
// (rows(q) x cols(r) from r to q), 1: product spectra (cols(q) x rows(r)).
// Single-process mode: device-to-device copies; otherwise NCCL send/recv
// on the context stream (grouped, one block per peer).
int exchange3(skg_ctx* c, int which);

int exchange(skg_ctx* c, int which) {
    if (c->solver == 3) return exchange3(c, which);
    const int G = c->G;
    const size_t nrl = (size_t)c->nrl;
    auto ncol = [&](int q) { return c->cstart[q + 1] - c->cstart[q]; };
    auto npair = [&](int q) { return (size_t)(ncol(q) + 1) / 2; };
    // block (source r -> destination q): pointers and element count
    auto block = [&](const Part& src, const Part& dst, int f, cd** from, cd** to, size_t* cnt) {
        const int r = src.r, q = dst.r;
        if (which == 0) {
            *cnt = nrl * ncol(r);
            *from = src.sI[f] + (size_t)q * nrl * ncol(r);
            *to = dst.rI[f] + nrl * c->cstart[r];
        } else {
            *cnt = 2 * npair(q) * nrl;
            *from = src.sA[f] + (size_t)(c->cstart[q] / 2) * 2 * nrl;
            *to = dst.rA[f] + (size_t)r * 2 * npair(q) * nrl;
        }
    };
    const skg::LaunchHook hook = hook_of(c);
    hook.begin(4);
    double bytes = 0.0;
    if (c->comm == nullptr) {  // all partitions local
        for (const Part& src : c->parts)
            for (const Part& dst : c->parts)
                for (int f = 0; f < 2; ++f) {
                    cd *from, *to;
                    size_t cnt;
                    block(src, dst, f, &from, &to, &cnt);
                    if (cnt == 0) continue;
                    CUDA_TRY(cudaMemcpyAsync(to, from, cnt * sizeof(cd), cudaMemcpyDeviceToDevice, c->stream));
                    if (src.r != dst.r) bytes += cnt * sizeof(cd);
                }
    } else {
        const Part& me = c->parts[0];
        const int r = me.r;
        ncclResult_t nr = nccl().GroupStart();
        for (int q = 0; q < G && nr == ncclSuccess; ++q) {
            for (int f = 0; f < 2 && nr == ncclSuccess; ++f) {
                cd *sptr, *rptr;
                size_t scnt, rcnt;
                if (which == 0) {
                    sptr = me.sI[f] + (size_t)q * nrl * ncol(r);
                    scnt = nrl * ncol(r);
                    rptr = me.rI[f] + nrl * c->cstart[q];
                    rcnt = nrl * ncol(q);
                } else {
                    sptr = me.sA[f] + (size_t)(c->cstart[q] / 2) * 2 * nrl;
                    scnt = 2 * npair(q) * nrl;
                    rptr = me.rA[f] + (size_t)q * 2 * npair(r) * nrl;
                    rcnt = 2 * npair(r) * nrl;
                }
                if (q == r) {
                    if (scnt) CUDA_TRY(cudaMemcpyAsync(rptr, sptr, scnt * sizeof(cd), cudaMemcpyDeviceToDevice, c->stream));
                    continue;
                }
                if (scnt) nr = nccl().Send(sptr, 2 * scnt, ncclDouble, q, c->comm, c->stream);
                if (nr == ncclSuccess && rcnt) nr = nccl().Recv(rptr, 2 * rcnt, ncclDouble, q, c->comm, c->stream);
                bytes += scnt * sizeof(cd);
            }
        }
        ncclResult_t ne = nccl().GroupEnd();
        if (nr != ncclSuccess || ne != ncclSuccess)
            return fail(SKG_ENCCL, std::string("all-to-all: ") + nccl().GetErrorString(nr != ncclSuccess ? nr : ne));
    }
    hook.end(4, bytes);
    ++c->launches;
    return SKG_OK;
}

// ns3d all-to-alls.  which = 0: x-inverse outputs, 5 fields, block r -> q =
// rows(q) x lines(r) ([xl][kyl_r][kz_in]); 1: y-forward outputs, 3 fields,
// block r -> q = rows(r) x lines(q) ([xl][kyl_q][kz_o]).
int exchange3(skg_ctx* c, int which) {
    const int G = c->G;
    if (G == 1) return SKG_OK;  // one partition: receive buffers alias the send buffers
    const size_t nrl = (size_t)c->nrl;
    const size_t kz = (size_t)c->kc[2] + 1;  // kz_in = kz_o (pruned)
    auto nl = [&](int q) { return (size_t)(c->cstart[q + 1] - c->cstart[q]); };
    const int nf = which == 0 ? 5 : 3;
    // block from rank r (buffers src) to rank q (buffers dst), field f
    auto src_ptr = [&](const Part& src, int q, int f) {
        return which == 0 ? src.A3 + f * src.fs + (size_t)q * nrl * nl(src.r) * kz
                          : src.sD3 + f * src.rfs + nrl * c->cstart[q] * kz;
    };
    auto dst_ptr = [&](const Part& dst, int r, int f) {
        return which == 0 ? dst.rA3 + f * dst.rfs + nrl * c->cstart[r] * kz
                          : dst.B3 + f * dst.fs + (size_t)r * nrl * nl(dst.r) * kz;
    };
    auto count = [&](int r, int q) { return nrl * kz * (which == 0 ? nl(r) : nl(q)); };
    const skg::LaunchHook hook = hook_of(c);
    hook.begin(4);
    double bytes = 0.0;
    if (c->comm == nullptr) {
        for (const Part& src : c->parts)
            for (const Part& dst : c->parts)
                for (int f = 0; f < nf; ++f) {
                    const size_t cnt = count(src.r, dst.r);
                    if (!cnt) continue;
                    CUDA_TRY(cudaMemcpyAsync(dst_ptr(dst, src.r, f), src_ptr(src, dst.r, f),
                                             cnt * sizeof(cd), cudaMemcpyDeviceToDevice, c->stream));
                    if (src.r != dst.r) bytes += cnt * sizeof(cd);
                }
    } else {
        const Part& me = c->parts[0];
        const int r = me.r;
        ncclResult_t nr = nccl().GroupStart();
        for (int q = 0; q < G && nr == ncclSuccess; ++q) {
            for (int f = 0; f < nf && nr == ncclSuccess; ++f) {
                const size_t scnt = count(r, q), rcnt = count(q, r);
                cd* sptr = src_ptr(me, q, f);
                cd* rptr = dst_ptr(me, q, f);
                if (q == r) {
                    if (scnt) CUDA_TRY(cudaMemcpyAsync(rptr, sptr, scnt * sizeof(cd), cudaMemcpyDeviceToDevice, c->stream));
                    continue;
                }
                if (scnt) nr = nccl().Send(sptr, 2 * scnt, ncclDouble, q, c->comm, c->stream);
                if (nr == ncclSuccess && rcnt) nr = nccl().Recv(rptr, 2 * rcnt, ncclDouble, q, c->comm, c->stream);
                bytes += scnt * sizeof(cd);
            }
        }
        ncclResult_t ne = nccl().GroupEnd();
        if (nr != ncclSuccess || ne != ncclSuccess)
            return fail(SKG_ENCCL, std::string("all-to-all: ") + nccl().GetErrorString(nr != ncclSuccess ? nr : ne));
    }
    hook.end(4, bytes);
    ++c->launches;
    return SKG_OK;
}

int dist_dt_update(skg_ctx* c, long* counter) {
    if (c->comm) {  // global max |u_d| over the ranks' x rows
        const ncclResult_t nr = nccl().AllReduce(c->d_dyn->umax, c->d_dyn->umax, 3, ncclDouble, ncclMax,
                                              c->comm, c->stream);
        if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
    }
    CUDA_TRY(skg::launch_dt_update(c->d_dyn, c->flags, c->etab, c->dims, c->n, c->kscale, c->nu,
                                   c->stream, counter));
    return SKG_OK;
}

// One step of a slab-decomposed context.  ns2d: the x-forward of every stage
// runs fused with the next stage's x-inverse (first: the step opens the
// batch and runs its own stage-1 x-inverse; last: no next stage).
int enqueue_dist_step(skg_ctx* c, double dt, long* counter, bool first, bool last) {
    const int nst = c->scheme == SKG_RK2 ? 2 : 4;
    const skg::LaunchHook hook = hook_of(c);
    int rc;
    if (c->solver == 3) {
        for (int st = 1; st <= nst; ++st) {
            for (int pass = 0; pass < 3; ++pass) {
                for (const Part& p : c->parts) {
                    skg::Ns3dArgs a = args3d_part(c, dt, p);
                    CUDA_TRY(skg::ns3d_pass(a, pass, st, c->stream, counter, hook));
                }
                if (pass < 2 && (rc = exchange(c, pass))) return rc;
            }
            if (st == 1 && c->adaptive && (rc = dist_dt_update(c, counter))) return rc;
        }
        return SKG_OK;
    }
    auto run_pass = [&](int pass, int st, int next) -> int {
        for (const Part& p : c->parts) {
            skg::Ns2dArgs a = args2d_part(c, dt, p);
            a.lead = p.r == 0 ? 1 : 0;
            CUDA_TRY(skg::ns2d_fast_pass(a, pass, st, c->stream, counter, hook, next));
        }
        return SKG_OK;
    };
    if (first) {
        if ((rc = run_pass(0, 1, 0)) || (rc = exchange(c, 0))) return rc;
    }
    for (int st = 1; st <= nst; ++st) {
        if ((rc = run_pass(1, st, 0)) || (rc = exchange(c, 1))) return rc;
        if (st == 1 && c->adaptive && (rc = dist_dt_update(c, counter))) return rc;
        const int next = st < nst || !last;
        if ((rc = run_pass(3, st, next))) return rc;
        if (next && (rc = exchange(c, 0))) return rc;
    }
    return SKG_OK;
}

int enqueue_steps(skg_ctx* c, double dt, long nsteps) {
    if (c->adaptive) dt = -1.0;  // device-resident: compute_dt per step
    else if (!(dt > 0.0)) return fail(SKG_ECONFIG, "step: nonpositive dt");
    if (nsteps < 0) return fail(SKG_ECONFIG, "step: negative step count");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->adaptive) {
        skg::DynStep d{};
        d.t = c->t;
        d.t_end = c->t_end;
        d.cfl = c->cfl;
        d.dt_max = c->dt_max;
        for (int k = 0; k < c->dims; ++k) d.dx[k] = c->L[k] / c->n[k];  // grid.cpp:50
        d.last_dt = c->last_dt;
        CUDA_TRY(cudaMemcpyAsync(c->d_dyn, &d, sizeof(d), cudaMemcpyHostToDevice, c->stream));
        c->cached_dt = -1.0;  // the device owns the factor tables now
    } else {
        int rc = refresh_exp(c, dt);
        if (rc) return rc;
    }
    skg::DevFlags init{0, std::numeric_limits<int>::max(), 0, 0};
    CUDA_TRY(cudaMemcpyAsync(c->flags, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    const int nst = c->scheme == SKG_RK2 ? 2 : 4;
    const skg::LaunchHook hook = hook_of(c);
    if (c->dist) {
        for (long s = 0; s < nsteps; ++s) {
            int rc2 = enqueue_dist_step(c, dt, &c->launches, s == 0, s == nsteps - 1);
            if (rc2) return rc2;
        }
        return SKG_OK;
    }
    // first: the step opens the batch; last: it closes it.  On the ns2d fast
    // path the x-forward of each stage is fused with the next stage's
    // x-inverse (across the step boundary too), so only the batch's first
    // step runs a standalone x-inverse and the last one no trailing one.
    auto one_step = [&](long* counter, bool first, bool last) -> cudaError_t {
        cudaError_t e = cudaSuccess;
        bool fused = false;
        auto dt_update = [&]() {
            return skg::launch_dt_update(c->d_dyn, c->flags, c->etab, c->dims, c->n, c->kscale, c->nu,
                                         c->stream, counter);
        };
        if (c->generic) {
            skg::GenArgs a = args_gen(c, dt);
            for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                e = skg::generic_stage(a, st, c->gs, c->stream, counter);
                if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
            }
        } else if (c->solver == 2) {
            skg::Ns2dArgs a = args2d(c, dt);
            fused = skg::ns2d_fast_ok(a);
            if (!fused) a.diag = nullptr;
            if (fused) {
                if (first) e = skg::ns2d_fast_pass(a, 0, 1, c->stream, counter, hook);
                for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                    e = skg::ns2d_fast_pass(a, 1, st, c->stream, counter, hook);
                    if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
                    if (e == cudaSuccess)
                        e = skg::ns2d_fast_pass(a, 3, st, c->stream, counter, hook, st < nst || !last);
                }
            } else {
                for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                    e = skg::ns2d_launch_stage(a, st, c->stream, counter, hook);
                    if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
                }
            }
        } else {
            skg::Ns3dArgs a = args3d(c, dt);
            fused = c->pruned;
            if (!fused) a.diag = nullptr;
            for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                e = skg::ns3d_launch_stage(a, st, c->stream, counter, hook);
                if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
            }
        }
        if (e == cudaSuccess && c->diag && !fused)  // unfused paths: one reduction per step
            e = skg::launch_energy(c->u, c->dims, c->n, c->kscale, c->nvars, energy_mode(c),
                                   c->diag, c->stream, counter, c->nu, &c->flags->steps, false);
        return e;
    };
    long s = 0;
    if (c->forcing) {  // host noise every step: no graph replay
        for (; s < nsteps; ++s) {
            int rc2 = refresh_forcing(c);
            if (rc2) return rc2;
            CUDA_TRY(one_step(&c->launches, s == 0, s == nsteps - 1));
        }
        return SKG_OK;
    }
    if (nsteps > 0) {  // first step eagerly (also sets kernel attributes)
        CUDA_TRY(one_step(&c->launches, true, nsteps == 1));
        s = 1;
    }
    // middle steps: replay of a captured step; the last step eagerly
    if (nsteps - s >= 3 && !c->timing && c->stream != nullptr) {
        if (c->gexec && (c->g_dt != dt || c->g_pruned != c->pruned || c->g_stream != c->stream ||
                         c->g_diag != c->diag)) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        if (!c->gexec) {
            cudaGraph_t graph;
            long dummy = 0;
            CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = one_step(&dummy, false, false);
            cudaError_t e2 = cudaStreamEndCapture(c->stream, &graph);
            CUDA_TRY(e);
            CUDA_TRY(e2);
            CUDA_TRY(cudaGraphInstantiate(&c->gexec, graph, 0));
            cudaGraphDestroy(graph);
            c->g_launches = dummy;
            c->g_dt = dt;
            c->g_diag = c->diag;
            c->g_pruned = c->pruned;
            c->g_stream = c->stream;
        }
        for (; s < nsteps - 1; ++s) {
            CUDA_TRY(cudaGraphLaunch(c->gexec, c->stream));
            c->launches += c->g_launches;
        }
    }
    for (; s < nsteps; ++s) CUDA_TRY(one_step(&c->launches, false, s == nsteps - 1));
    return SKG_OK;
}

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
    const size_t nh = (size_t)c->nh, kzc = (size_t)c->kc[2] + 1;
    const int runs[2][2] = {{0, kcy + 1}, {kcy + 1, 2 * kcy + 1}};  // compact ranges
    for (int b = 0; b < 2; ++b) {
        const int lo = std::max(runs[b][0], p.c0), hi = std::min(runs[b][1], p.c0 + p.ncols);
        if (lo >= hi) continue;
        const int gy = b == 0 ? lo : lo + ny - (2 * kcy + 1);
        for (int v = 0; v < 3; ++v) {
            // kept kz of lines [gy, gy + hi - lo) for every kx: (kz, line, kx) boxes
            cd* io = c->io + (size_t)v * c->S + (size_t)gy * nh;
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
    CUDA_TRY(cudaMalloc(&c->phys, sizeof(double) * (size_t)c->P));
    CUDA_TRY(cudaMalloc(&c->work, sizeof(cd) * (size_t)c->S));
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
    if (cudaMalloc(&d, sizeof(cd) * n) != cudaSuccess) return nullptr;
    cudaMemcpy(d, w.data(), sizeof(cd) * n, cudaMemcpyHostToDevice);
    g_tw.tabs[key] = d;
    return d;
}

}  // namespace

extern "C" {

const char* skg_version(void) { return "skgpu 0.1.0 sm_100a"; }

const char* skg_last_error(void) { return g_err.c_str(); }

static int create_impl(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                       double dealias_coef, double nu, int scheme, int device, int rank, int world,
                       const char* nccl_id, bool slab_one);

int skg_create(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
               double dealias_coef, double nu, int scheme, int device) {
    return create_impl(out, solver, dims, n, L, dealias_coef, nu, scheme, device, 0, 1, nullptr, false);
}

int skg_create_dist(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                    double dealias_coef, double nu, int scheme, int device, int rank, int world,
                    const char* nccl_id) {
    return create_impl(out, solver, dims, n, L, dealias_coef, nu, scheme, device, rank, world, nccl_id,
                       world == 1);
}

int skg_nccl_unique_id(char* out128) {
    ncclUniqueId id;
    if (!nccl().ok) return fail(SKG_ENCCL, nccl().why);
    const ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
    return SKG_OK;
}

static int create_impl(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                       double dealias_coef, double nu, int scheme, int device, int rank, int world,
                       const char* nccl_id, bool slab_one) {
    if (!out) return fail(SKG_ECONFIG, "create: null output pointer");
    *out = nullptr;
    std::string s = solver ? solver : "";
    int sid = s == "ns2d" ? 2 : s == "ns3d" ? 3 : 0;
    if (!sid) return fail(SKG_ECONFIG, "unknown solver '" + s + "' (registered: ns2d, ns3d)");
    if (dims != sid) return fail(SKG_ECONFIG, "solver " + s + " needs " + std::to_string(sid) + " extents");
    for (int d = 0; d < dims; ++d) {
        if (n[d] < 4) return fail(SKG_ECONFIG, "extent " + std::to_string(n[d]) + " too small (min 4)");
        if (n[d] % 2) return fail(SKG_ECONFIG, "extent " + std::to_string(n[d]) + " is odd");
        if (L && !(L[d] > 0)) return fail(SKG_ECONFIG, "domain length must be positive");
    }
    if (!(dealias_coef > 0.0) || dealias_coef > 1.0)
        return fail(SKG_ECONFIG, "dealias_coef must be in (0, 1]");
    if (!(nu >= 0.0)) return fail(SKG_ECONFIG, "viscosity must be >= 0");
    if (scheme != SKG_RK4 && scheme != SKG_RK2) return fail(SKG_ECONFIG, "unknown time scheme");
    // extents outside the fused kernels' range run the generic step
    const bool generic = sid == 2 ? !skg::ns2d_supported(n[0], n[1]) : !skg::ns3d_supported(n[0], n[1], n[2]);
    if (generic && (world > 1 || (sid == 3 && slab_one)))
        return fail(SKG_EUNSUPPORTED,
                    "slab and compact layouts need the fused kernels' extents (powers of two)");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SKG_ECUDA, "no CUDA device visible (the library has no CPU path)");
    if (device < 0 || device >= ndev) return fail(SKG_ECONFIG, "device ordinal out of range");
    if (world < 1 || rank < 0 || rank >= world) return fail(SKG_ECONFIG, "bad rank / world size");
    if (world > 1 && sid == 3 && n[0] % world)
        return fail(SKG_ECONFIG, "nx must be divisible by world for the slab decomposition");
    if (world > 1 && sid == 2 && n[0] % (4 * world))
        return fail(SKG_ECONFIG, "nx must be divisible by 4 * world for the slab decomposition");

    auto c = new skg_ctx();
    c->device = device;
    c->solver = sid;
    c->dims = dims;
    c->coef = dealias_coef;
    c->nu = nu;
    c->scheme = scheme;
    c->nvars = sid == 2 ? 1 : 3;
    for (int d = 0; d < dims; ++d) {
        c->n[d] = n[d];
        c->L[d] = L ? L[d] : kTwoPi;
        c->kscale[d] = kTwoPi / c->L[d];
        c->kc[d] = cut_index(n[d], c->L[d], dealias_coef, d == dims - 1);
    }
    c->generic = generic;
    c->nh = n[dims - 1] / 2 + 1;
    c->S = c->nh;
    c->P = 1;
    for (int d = 0; d < dims - 1; ++d) c->S *= n[d];
    for (int d = 0; d < dims; ++d) c->P *= n[d];

    auto cleanup = [&](int code, const std::string& msg) {
        skg_destroy(c);
        return fail(code, msg);
    };
    if (cudaSetDevice(device) != cudaSuccess) return cleanup(SKG_ECUDA, "cudaSetDevice failed");
    c->nsm = sm_count(device);
    if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(SKG_ECUDA, "stream creation failed");
    c->stream = c->own;
    const size_t S = (size_t)c->S;
    auto alloc = [&](void** p, size_t bytes) {
        if (cudaMalloc(p, bytes < 16 ? 16 : bytes) != cudaSuccess) return false;
        return cudaMemset(*p, 0, bytes < 16 ? 16 : bytes) == cudaSuccess;
    };
    bool ok = true;
    // slab layout: several partitions, or the compact one-partition ns3d
    // layout requested through skg_create_dist(world = 1)
    // ns3d on one GPU: the compact layout when the full one would not fit
    // (1024^3: ~220 GB full vs ~135 GB compact); it needs dealiased states
    if (sid == 3 && world == 1 && !slab_one && !generic) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const double full = 16.0 * (double)c->S * (3.0 * 4 + 3.0) +
                            16.0 * 11.0 * (double)n[0] * n[1] * c->nh;
        if (full > 0.92 * (double)fr) slab_one = true;
    }
    c->dist = world > 1 || (sid == 3 && slab_one);
    c->G = world;
    c->grank = rank;
    if (sid == 2) {  // column partition of the kept ky columns, row partition of x
        const int Kc = c->kc[1] + 1, PP = (Kc + 1) / 2;
        if (PP < world) return cleanup(SKG_ECONFIG, "more ranks than kept ky column pairs");
        c->cstart.resize(world + 1);
        for (int q = 0; q < world; ++q) c->cstart[q] = 2 * (int)((long long)q * PP / world);
        c->cstart[world] = Kc;
        c->nrl = n[0] / world;
        std::vector<int> owner(Kc);
        for (int q = 0; q < world; ++q)
            for (int k = c->cstart[q]; k < c->cstart[q + 1]; ++k) owner[k] = q;
        ok = ok && alloc((void**)&c->d_kowner, sizeof(int) * Kc);
        ok = ok && alloc((void**)&c->d_cstart, sizeof(int) * (world + 1));
        if (ok) {
            cudaMemcpy(c->d_kowner, owner.data(), sizeof(int) * Kc, cudaMemcpyHostToDevice);
            cudaMemcpy(c->d_cstart, c->cstart.data(), sizeof(int) * (world + 1), cudaMemcpyHostToDevice);
        }
    }
    if (sid == 3 && c->dist) {  // contiguous runs of compact kept ky lines, x rows
        const int Kyc = 2 * c->kc[1] + 1;
        if (Kyc < world) return cleanup(SKG_ECONFIG, "more ranks than kept ky lines");
        c->cstart.resize(world + 1);
        for (int q = 0; q <= world; ++q) c->cstart[q] = (int)((long long)q * Kyc / world);
        c->nrl = n[0] / world;
        std::vector<int> owner(Kyc);
        for (int q = 0; q < world; ++q)
            for (int k = c->cstart[q]; k < c->cstart[q + 1]; ++k) owner[k] = q;
        ok = ok && alloc((void**)&c->d_kowner, sizeof(int) * Kyc);
        ok = ok && alloc((void**)&c->d_cstart, sizeof(int) * (world + 1));
        if (ok) {
            cudaMemcpy(c->d_kowner, owner.data(), sizeof(int) * Kyc, cudaMemcpyHostToDevice);
            cudaMemcpy(c->d_cstart, c->cstart.data(), sizeof(int) * (world + 1), cudaMemcpyHostToDevice);
        }
        // state lines and intermediates hold only the kept kz (slab layouts
        // need a dealiased state); one partition: no exchange buffers
        const size_t nx = n[0], ny = n[1], kzc = (size_t)c->kc[2] + 1, nrl = c->nrl;
        for (int q = 0; q < world; ++q) {
            if (nccl_id && q != rank) continue;
            Part p;
            p.r = q;
            p.c0 = c->cstart[q];
            p.ncols = c->cstart[q + 1] - c->cstart[q];
            p.vs = nx * p.ncols * kzc;
            p.fs = std::max(p.vs, nrl * ny * kzc);
            p.rfs = nrl * Kyc * kzc;
            ok = ok && alloc((void**)&p.u, sizeof(cd) * 3 * p.vs);
            for (int i = 0; i < 3; ++i) ok = ok && alloc((void**)&p.k[i], sizeof(cd) * 3 * p.vs);
            ok = ok && alloc((void**)&p.A3, sizeof(cd) * 5 * p.fs);
            ok = ok && alloc((void**)&p.B3, sizeof(cd) * 6 * p.fs);
            if (world > 1) {
                ok = ok && alloc((void**)&p.rA3, sizeof(cd) * 5 * p.rfs);
                ok = ok && alloc((void**)&p.sD3, sizeof(cd) * 3 * p.rfs);
            } else {
                p.rA3 = p.A3;
                p.rfs = p.fs;
                p.sD3 = p.B3;
            }
            c->parts.push_back(p);
        }
        if (ok && nccl_id) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            if (!nccl().ok) return cleanup(SKG_ENCCL, nccl().why);
            const ncclResult_t nr = nccl().CommInitRank(&c->comm, world, id, rank);
            if (nr != ncclSuccess) return cleanup(SKG_ENCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(nr));
        }
    } else if (c->dist) {
        const int Kc = c->kc[1] + 1, PP = (Kc + 1) / 2;
        const size_t nx = n[0], nrl = c->nrl;
        for (int q = 0; q < world; ++q) {
            if (nccl_id && q != rank) continue;  // NCCL: only this process's slab
            Part p;
            p.r = q;
            p.c0 = c->cstart[q];
            p.ncols = c->cstart[q + 1] - c->cstart[q];
            const size_t npairs = (p.ncols + 1) / 2;
            ok = ok && alloc((void**)&p.u, sizeof(cd) * p.ncols * nx);
            for (int i = 0; i < 3; ++i) ok = ok && alloc((void**)&p.k[i], sizeof(cd) * p.ncols * nx);
            for (int f = 0; f < 2; ++f) {
                ok = ok && alloc((void**)&p.sI[f], sizeof(cd) * nx * p.ncols);
                ok = ok && alloc((void**)&p.rI[f], sizeof(cd) * nrl * Kc);
                ok = ok && alloc((void**)&p.sA[f], sizeof(cd) * 2 * PP * nrl);
                ok = ok && alloc((void**)&p.rA[f], sizeof(cd) * world * 2 * npairs * nrl);
            }
            c->parts.push_back(p);
        }
        ok = ok && alloc((void**)&c->cmfull, sizeof(cd) * S);
        if (ok && nccl_id) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            if (!nccl().ok) return cleanup(SKG_ENCCL, nccl().why);
            const ncclResult_t nr = nccl().CommInitRank(&c->comm, world, id, rank);
            if (nr != ncclSuccess) return cleanup(SKG_ENCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(nr));
        }
    } else {
        ok = ok && alloc((void**)&c->u, sizeof(cd) * S * c->nvars);
        for (int i = 0; i < 3 && ok; ++i) ok = alloc((void**)&c->k[i], sizeof(cd) * S * c->nvars);
        if (sid == 2) c->inter_elems = 5 * S;  // 4 intermediates + tendency rows
        else c->inter_elems = 11 * (size_t)n[0] * n[1] * c->nh;  // A[5] (C aliases) + B[6] (D aliases)
        if (c->generic) c->inter_elems = 1;
        ok = ok && alloc((void**)&c->inter, sizeof(cd) * c->inter_elems);
        if (c->generic) {
            const size_t P = (size_t)c->P;
            ok = ok && alloc((void**)&c->gs.w, sizeof(cd) * S * c->nvars);
            ok = ok && alloc((void**)&c->gs.spec, sizeof(cd) * S * (sid == 2 ? 4 : 3));
            ok = ok && alloc((void**)&c->gs.nl, sizeof(cd) * S * c->nvars);
            ok = ok && alloc((void**)&c->gs.phys, sizeof(double) * P * (sid == 2 ? 4 : 6));
            ok = ok && alloc((void**)&c->gs.work, sizeof(cd) * S);
        }
    }
    ok = ok && alloc((void**)&c->io, sizeof(cd) * S * c->nvars);
    int ext_total = 0;
    for (int d = 0; d < dims; ++d) ext_total += d == dims - 1 ? c->nh : n[d];
    ok = ok && alloc((void**)&c->etab, sizeof(double) * 2 * ext_total);
    ok = ok && alloc((void**)&c->flags, sizeof(skg::DevFlags));
    ok = ok && alloc((void**)&c->d_count, sizeof(unsigned long long));
    ok = ok && alloc((void**)&c->d_red, 3 * sizeof(double));
    ok = ok && alloc((void**)&c->d_dyn, sizeof(skg::DynStep));
    if (!ok) return cleanup(SKG_ECUDA, "device allocation failed (grid too large for this GPU?)");
    for (int d = 0; d < dims; ++d) {
        c->tw[d] = twiddle_table(device, n[d]);
        if (!c->tw[d]) return cleanup(SKG_ECUDA, "twiddle table allocation failed");
        c->gs.tw[d] = c->tw[d];
    }
    // cudaMemset above runs on the legacy default stream, which does not order
    // against the context's non-blocking stream: finish it before any kernel.
    if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(SKG_ECUDA, "device synchronize failed");
    c->pruned = true;  // zero state is dealiased
    *out = c;
    return SKG_OK;
}

int skg_destroy(skg_ctx* c) {
    if (!c) return SKG_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->u);
    for (auto p : c->k) cudaFree(p);
    cudaFree(c->inter);
    cudaFree(c->io);
    cudaFree(c->phys);
    cudaFree(c->work);
    cudaFree(c->etab);
    cudaFree(c->flags);
    cudaFree(c->d_count);
    cudaFree(c->d_red);
    cudaFree(c->d_dyn);
    cudaFree(c->f_ref);
    cudaFree(c->f_cm);
    cudaFree(c->f_red);
    if (c->f_noise) cudaFreeHost(c->f_noise);
    cudaFree(c->gs.w);
    cudaFree(c->gs.spec);
    cudaFree(c->gs.nl);
    cudaFree(c->gs.phys);
    cudaFree(c->gs.work);
    harvest(c);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (Part& p : c->parts) {
        cudaFree(p.u);
        for (auto q : p.k) cudaFree(q);
        for (int f = 0; f < 2; ++f) {
            cudaFree(p.sI[f]);
            cudaFree(p.rI[f]);
            cudaFree(p.sA[f]);
            cudaFree(p.rA[f]);
        }
        if (p.rA3 != p.A3) cudaFree(p.rA3);
        if (p.sD3 != p.B3) cudaFree(p.sD3);
        cudaFree(p.A3);
        cudaFree(p.B3);
    }
    cudaFree(c->cmfull);
    cudaFree(c->d_kowner);
    cudaFree(c->d_cstart);
    if (c->comm) nccl().CommDestroy(c->comm);
    for (auto e : c->pool) cudaEventDestroy(e);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
    return SKG_OK;
}

int skg_set_stream(skg_ctx* c, void* stream) {
    c->stream = stream ? (cudaStream_t)stream : c->own;
    return SKG_OK;
}

long skg_spect_size(const skg_ctx* c) { return (long)c->S; }
long skg_phys_size(const skg_ctx* c) { return (long)c->P; }
int skg_nvars(const skg_ctx* c) { return c->nvars; }
long skg_iteration(const skg_ctx* c) { return c->it; }
double skg_time(const skg_ctx* c) { return c->t; }
int skg_pruned(const skg_ctx* c) { return c->pruned ? 1 : 0; }
long skg_launch_count(const skg_ctx* c) { return c->launches; }

int skg_set_state(skg_ctx* c, const double* spect) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemcpyAsync(c->io, spect, sizeof(cd) * c->S * c->nvars, cudaMemcpyHostToDevice,
                             c->stream));
    int rc = load_state_from_io(c);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

int skg_set_state_device(skg_ctx* c, const double* d_spect) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemcpyAsync(c->io, d_spect, sizeof(cd) * c->S * c->nvars,
                             cudaMemcpyDeviceToDevice, c->stream));
    return load_state_from_io(c);
}

int skg_get_state(skg_ctx* c, double* spect_out) {
    CUDA_TRY(cudaSetDevice(c->device));
    int rc = store_state_to_io(c, c->u);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(spect_out, c->io, sizeof(cd) * c->S * c->nvars,
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

int skg_get_state_device(skg_ctx* c, double* d_out) {
    CUDA_TRY(cudaSetDevice(c->device));
    int rc = store_state_to_io(c, c->u);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(d_out, c->io, sizeof(cd) * c->S * c->nvars,
                             cudaMemcpyDeviceToDevice, c->stream));
    return SKG_OK;
}

int skg_step_async(skg_ctx* c, double dt, long nsteps) {
    int rc = enqueue_steps(c, dt, nsteps);
    if (rc) return rc;
    c->pending_steps += nsteps;
    c->pending_dt = dt;
    return SKG_OK;
}

int skg_sync(skg_ctx* c) {
    CUDA_TRY(cudaSetDevice(c->device));
    long n = c->pending_steps;
    c->pending_steps = 0;
    return sync_and_check(c, n, c->pending_dt);
}

int skg_step(skg_ctx* c, double dt, long nsteps) {
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    int rc = enqueue_steps(c, dt, nsteps);
    if (rc) return rc;
    return sync_and_check(c, nsteps, dt);
}

int skg_run(skg_ctx* c, double dt, long nsteps, double* series) {
    if (!series) return skg_step(c, dt, nsteps);
    if (c->comm) return fail(SKG_EUNSUPPORTED, "skg_run series on a multi-process context");
    if (nsteps <= 0) return skg_step(c, dt, nsteps);
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    double* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, sizeof(double) * 3 * nsteps));
    CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(double) * 3 * nsteps, c->stream));
    c->diag = d;
    int rc = enqueue_steps(c, dt, nsteps);
    c->diag = nullptr;
    if (rc == SKG_OK) rc = sync_and_check(c, nsteps, dt);
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(series, d, sizeof(double) * 3 * nsteps, cudaMemcpyDeviceToHost);
    if (c->gexec && c->g_diag == d) {  // the graph baked this buffer in
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    cudaFree(d);
    return rc;
}

static int tendency_impl(skg_ctx* c, const double* in, double* out, double* umax);

int skg_tendency(skg_ctx* c, const double* in, double* out) {
    return tendency_impl(c, in, out, nullptr);
}

int skg_max_velocity(skg_ctx* c, const double* in, double* umax) {
    if (!umax) return fail(SKG_ECONFIG, "skg_max_velocity: null output");
    return tendency_impl(c, in, nullptr, umax);
}

// Solver::tendency of `in` (host, reference layout) into `out` (or not, when
// null); with umax, also max |u_d| of `in` (Solver::max_velocity_per_axis)
// from the same physical pass.
static int tendency_impl(skg_ctx* c, const double* in, double* out, double* umax) {
    if (c->dist) return fail(SKG_EUNSUPPORTED, "skg_tendency on a slab-decomposed context");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(c->io, in, sizeof(cd) * c->S * c->nvars, cudaMemcpyHostToDevice,
                             c->stream));
    const bool keep_pruned = c->pruned;
    int rc = decide_pruned(c, c->io);
    if (rc) return rc;
    if (c->generic) {  // reference layout throughout; tendency into gs.nl
        skg::GenArgs a = args_gen(c, 1.0);
        a.dyn = umax ? c->d_dyn : nullptr;
        a.force = nullptr;  // Solver::tendency has no forcing addend
        skg::DevFlags init{0, std::numeric_limits<int>::max(), 0, 0};
        CUDA_TRY(cudaMemcpyAsync(c->flags, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
        if (umax) CUDA_TRY(cudaMemsetAsync(c->d_dyn, 0, sizeof(skg::DynStep), c->stream));
        CUDA_TRY(skg::generic_tendency(a, c->io, 1, nullptr, c->gs, c->stream, &c->launches));
        CUDA_TRY(cudaMemcpyAsync(c->io, c->gs.nl, sizeof(cd) * c->S * c->nvars, cudaMemcpyDeviceToDevice,
                                 c->stream));
    } else if (c->solver == 2) {
        // input (CM) in k[2], tendency into k[0]
        CUDA_TRY(skg::launch_transpose_c(c->io, c->k[2], c->n[0], c->nh, 0, c->stream, &c->launches));
        rc = refresh_exp(c, c->cached_dt > 0 ? c->cached_dt : 1.0);
        if (rc) return rc;
        skg::Ns2dArgs a = args2d(c, c->cached_dt);
        a.u = c->k[2];
        a.dyn = umax ? c->d_dyn : nullptr;
        a.force = nullptr;
        skg::DevFlags init{0, std::numeric_limits<int>::max(), 0, 0};
        CUDA_TRY(cudaMemcpyAsync(c->flags, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
        if (umax) CUDA_TRY(cudaMemsetAsync(c->d_dyn, 0, sizeof(skg::DynStep), c->stream));
        CUDA_TRY(skg::ns2d_launch_stage(a, 1, c->stream, &c->launches, hook_of(c)));
        rc = store_state_to_io(c, c->k[0]);
        if (rc) return rc;
    } else {
        CUDA_TRY(cudaMemcpyAsync(c->k[2], c->io, sizeof(cd) * c->S * c->nvars,
                                 cudaMemcpyDeviceToDevice, c->stream));
        rc = refresh_exp(c, c->cached_dt > 0 ? c->cached_dt : 1.0);
        if (rc) return rc;
        skg::Ns3dArgs a = args3d(c, c->cached_dt);
        a.u = c->k[2];
        a.dyn = umax ? c->d_dyn : nullptr;
        a.force = nullptr;
        skg::DevFlags init{0, std::numeric_limits<int>::max(), 0, 0};
        CUDA_TRY(cudaMemcpyAsync(c->flags, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
        if (umax) CUDA_TRY(cudaMemsetAsync(c->d_dyn, 0, sizeof(skg::DynStep), c->stream));
        CUDA_TRY(skg::ns3d_launch_stage(a, 1, c->stream, &c->launches, hook_of(c)));
        rc = store_state_to_io(c, c->k[0]);
        if (rc) return rc;
    }
    if (out)
        CUDA_TRY(cudaMemcpyAsync(out, c->io, sizeof(cd) * c->S * c->nvars, cudaMemcpyDeviceToHost,
                                 c->stream));
    if (umax) {
        skg::DynStep d;
        CUDA_TRY(cudaMemcpyAsync(&d, c->d_dyn, sizeof(d), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < c->dims; ++k) umax[k] = d.umax[k];
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->pruned = keep_pruned;
    return SKG_OK;
}

int skg_fft_forward(skg_ctx* c, const double* u, double* uhat) {
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_fft_bufs(c)) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->phys, u, sizeof(double) * c->P, cudaMemcpyHostToDevice, c->stream));
    const cd* tw[3] = {c->tw[0], c->tw[1], c->tw[2]};
    CUDA_TRY(skg::fft_forward_dev(c->dims, c->n, c->phys, c->io, c->work, tw, c->stream, &c->launches));
    CUDA_TRY(cudaMemcpyAsync(uhat, c->io, sizeof(cd) * c->S, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

int skg_fft_inverse(skg_ctx* c, const double* uhat, double* u) {
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_fft_bufs(c)) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->io, uhat, sizeof(cd) * c->S, cudaMemcpyHostToDevice, c->stream));
    const cd* tw[3] = {c->tw[0], c->tw[1], c->tw[2]};
    CUDA_TRY(skg::fft_inverse_dev(c->dims, c->n, c->io, c->phys, c->work, tw, c->stream, &c->launches));
    CUDA_TRY(cudaMemcpyAsync(u, c->phys, sizeof(double) * c->P, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

static int plan_common(int rank, const int* shape, long long* P, long long* S) {
    if (rank < 1 || rank > 3)
        return fail(SKG_ESHAPE, "transform rank must be 1..3, got " + std::to_string(rank));
    *P = 1;
    *S = 1;
    for (int d = 0; d < rank; ++d) {
        if (shape[d] < 4) return fail(SKG_ESHAPE, "extent " + std::to_string(shape[d]) + " too small (min 4)");
        if (shape[d] % 2) return fail(SKG_ESHAPE, "extent " + std::to_string(shape[d]) + " is odd");
        *P *= shape[d];
        *S *= d == rank - 1 ? shape[d] / 2 + 1 : shape[d];
    }
    return SKG_OK;
}

// Device buffers of the shape-level transforms, reused across calls (the
// reference calls FftPlan::forward/inverse many times per step).
struct PlanBufs {
    double* u = nullptr;
    cd* h = nullptr;
    cd* w = nullptr;
    long long P = 0, S = 0;
};
std::mutex g_plan_mu;
std::map<int, PlanBufs> g_plan_bufs;

static int plan_run(int rank, const int* shape, const double* in, double* out, int device, bool forward,
                    bool normalize) {
    long long P, S;
    int rc = plan_common(rank, shape, &P, &S);
    if (rc) return rc;
    CUDA_TRY(cudaSetDevice(device));
    std::lock_guard<std::mutex> lk(g_plan_mu);
    PlanBufs& b = g_plan_bufs[device];
    if (b.P < P || b.S < S) {
        cudaFree(b.u);
        cudaFree(b.h);
        cudaFree(b.w);
        b = PlanBufs{};
        CUDA_TRY(cudaMalloc(&b.u, sizeof(double) * P));
        CUDA_TRY(cudaMalloc(&b.h, sizeof(cd) * S));
        CUDA_TRY(cudaMalloc(&b.w, sizeof(cd) * S));
        b.P = P;
        b.S = S;
    }
    const cd* tw[3] = {nullptr, nullptr, nullptr};
    for (int d = 0; d < rank; ++d) tw[d] = twiddle_table(device, shape[d]);
    long l = 0;
    cudaError_t e;
    if (forward) {
        e = cudaMemcpy(b.u, in, sizeof(double) * P, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = skg::fft_forward_dev(rank, shape, b.u, b.h, nullptr, tw, 0, &l, normalize);
        if (e == cudaSuccess) e = cudaMemcpy(out, b.h, sizeof(cd) * S, cudaMemcpyDeviceToHost);
    } else {
        e = cudaMemcpy(b.h, in, sizeof(cd) * S, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = skg::fft_inverse_dev(rank, shape, b.h, b.u, b.w, tw, 0, &l);
        if (e == cudaSuccess) e = cudaMemcpy(out, b.u, sizeof(double) * P, cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess) return fail(SKG_ECUDA, cudaGetErrorString(e));
    return SKG_OK;
}

int skg_plan_forward(int rank, const int* shape, const double* u, double* uhat, int device) {
    return plan_run(rank, shape, u, uhat, device, true, true);
}

int skg_plan_inverse(int rank, const int* shape, const double* uhat, double* u, int device) {
    return plan_run(rank, shape, uhat, u, device, false, false);
}

int skg_dft_r2c(int rank, const int* shape, const double* in, double* out, int device) {
    return plan_run(rank, shape, in, out, device, true, false);
}

int skg_dft_c2r(int rank, const int* shape, const double* in, double* out, int device) {
    return plan_run(rank, shape, in, out, device, false, false);
}

int skg_get_grid(skg_ctx* c, int axis, double* k_axis, unsigned char* mask) {
    if (axis < 0 || axis >= c->dims) return fail(SKG_ESHAPE, "axis out of range");
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_fft_bufs(c)) return rc;
    double* dk = reinterpret_cast<double*>(c->work);  // >= nh doubles
    unsigned char* dm = mask ? reinterpret_cast<unsigned char*>(c->io) : nullptr;
    CUDA_TRY(skg::launch_grid_dump(c->dims, c->n, c->kc, c->kscale, axis, dk, dm, c->stream, &c->launches));
    const int ext = axis == c->dims - 1 ? c->nh : c->n[axis];
    CUDA_TRY(cudaMemcpyAsync(k_axis, dk, sizeof(double) * ext, cudaMemcpyDeviceToHost, c->stream));
    if (mask) CUDA_TRY(cudaMemcpyAsync(mask, dm, (size_t)c->S, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

int skg_last_divergence(const skg_ctx* c, long* iteration, int* var) {
    *iteration = c->div_it;
    *var = c->div_var;
    return SKG_OK;
}

int skg_set_cfl(skg_ctx* c, double cfl_coef, double dt_max, double t_end) {
    if (cfl_coef <= 0.0) {
        c->adaptive = false;
        return SKG_OK;
    }
    if (!(dt_max > 0.0)) return fail(SKG_ECONFIG, "dt_max must be > 0");  // simulation.cpp:253-256
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    c->adaptive = true;
    c->cfl = cfl_coef;
    c->dt_max = dt_max;
    c->t_end = t_end;
    return SKG_OK;
}

double skg_last_dt(const skg_ctx* c) { return c->last_dt; }

int skg_set_forcing(skg_ctx* c, int enable, double k_lo, double k_hi, double rate, long seed) {
    if (!enable) {
        c->forcing = false;
        return SKG_OK;
    }
    // simulation.cpp:269-273 and random_field's checks (grid.cpp:277-280)
    if (k_lo > k_hi) return fail(SKG_ECONFIG, "forcing band: k_lo must be <= k_hi");
    if (!std::isfinite(rate)) return fail(SKG_ECONFIG, "forcing.rate must be finite");
    if (!(k_lo >= 0) || !(k_hi > k_lo)) return fail(SKG_ECONFIG, "random_field: need 0 <= k_lo < k_hi");
    if (c->dist) return fail(SKG_EUNSUPPORTED, "forcing on a slab-decomposed context");
    double Lmax = 0.0, kmax2 = 0.0, kcut = 1e300;
    for (int d = 0; d < c->dims; ++d) {
        Lmax = std::max(Lmax, c->L[d]);
        const double km = c->kscale[d] * (d == c->dims - 1 ? c->n[d] / 2 : c->n[d] / 2);
        kmax2 += km * km;
        kcut = std::min(kcut, c->coef * (kTwoPi / c->L[d]) * (c->n[d] / 2));  // grid.cpp:83-84
    }
    const double dk = kTwoPi / Lmax;
    if (k_lo > std::sqrt(kmax2))
        return fail(SKG_ECONFIG, "random_field: band lies above the largest resolved |k|");
    if (k_lo < 0.5 * dk || k_hi + 0.5 * dk > kcut)
        return fail(SKG_EUNSUPPORTED,
                    "forcing band must exclude the mean shell and lie inside the dealiasing cut");
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_fft_bufs(c)) return rc;
    if (!c->f_ref) {
        CUDA_TRY(cudaMalloc(&c->f_ref, sizeof(cd) * c->S * c->nvars));
        CUDA_TRY(cudaMalloc(&c->f_red, 8 * sizeof(double)));
        CUDA_TRY(cudaMallocHost(&c->f_noise, sizeof(double) * c->P * c->nvars));
        if (c->solver == 2 && !c->generic) CUDA_TRY(cudaMalloc(&c->f_cm, sizeof(cd) * c->S));
    }
    c->forcing = true;
    c->f_klo = k_lo;
    c->f_khi = k_hi;
    c->f_rate = rate;
    c->f_rng.seed(static_cast<std::uint64_t>(seed));  // simulation.cpp:338-339
    c->last_injection = 0.0;
    return SKG_OK;
}

double skg_last_injection(const skg_ctx* c) { return c->last_injection; }

int skg_sanitize_state(skg_ctx* c) {
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    int rc = store_state_to_io(c, c->u);
    if (rc) return rc;
    CUDA_TRY(skg::sanitize_dev(force_geo(c), c->io, c->stream, &c->launches));
    rc = load_state_from_io(c);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

int skg_set_time(skg_ctx* c, double t) {
    c->t = t;
    return SKG_OK;
}

int skg_set_timing(skg_ctx* c, int enable) {
    c->timing = enable != 0;
    return SKG_OK;
}

int skg_reset_stats(skg_ctx* c) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    harvest(c);
    for (int i = 0; i < 6; ++i) {
        c->st_ms[i] = 0;
        c->st_n[i] = 0;
        c->st_bytes[i] = 0;
    }
    return SKG_OK;
}

int skg_kernel_stats(skg_ctx* c, int cls, double* total_ms, long* launches, double* bytes) {
    if (cls < 0 || cls > 5) return fail(SKG_ESHAPE, "kernel class out of range");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    harvest(c);
    if (total_ms) *total_ms = c->st_ms[cls];
    if (launches) *launches = c->st_n[cls];
    if (bytes) *bytes = c->st_bytes[cls];
    return SKG_OK;
}

int skg_energy(skg_ctx* c, double* energy, double* enstrophy) {
    double d[3];
    int rc = skg_diagnostics(c, d);
    if (rc) return rc;
    if (energy) *energy = d[0];
    if (enstrophy) *enstrophy = d[1];
    return SKG_OK;
}

int skg_diagnostics(skg_ctx* c, double* out3) {
    if (!out3) return fail(SKG_ECONFIG, "skg_diagnostics: null output");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->dist) {  // gather the slabs into the reference layout (io), reduce there
        int rc = store_state_to_io(c, c->u);
        if (rc) return rc;
        CUDA_TRY(skg::launch_energy(c->io, c->dims, c->n, c->kscale, c->nvars, c->solver == 2 ? 2 : 0,
                                    c->d_red, c->stream, &c->launches, c->nu));
    } else {
        CUDA_TRY(skg::launch_energy(c->u, c->dims, c->n, c->kscale, c->nvars, energy_mode(c),
                                    c->d_red, c->stream, &c->launches, c->nu));
    }
    double h[3];
    CUDA_TRY(cudaMemcpyAsync(h, c->d_red, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    out3[0] = h[0];
    out3[1] = c->solver == 2 ? h[1] : 0.0;  // ns3d: no enstrophy (simulation.cpp:599-606)
    out3[2] = h[2];
    return SKG_OK;
}

}  // extern "C"
