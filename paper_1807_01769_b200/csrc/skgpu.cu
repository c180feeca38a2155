// skgpu.cu -- the extern "C" boundary of libskgpu (include/skgpu.h).
//
// Mirrors the reference's Simulation / ExactLinStepper / Solver contract
// (proj/src/simulation.cpp:297-590, proj/src/time_stepping.cpp:72-194) for a
// device-resident state.  The host side only validates arguments, builds the
// small per-axis tables (twiddles, exp factors, dealias cut indices) and
// enqueues kernels; every per-mode operation runs in sm_100a kernels.  There is
// no CPU fallback: a missing device or an unsupported extent is an error.
// Context helpers: host_ctx.cu; step enqueueing: host_step.cu.
#include "host_ctx.h"

using namespace skh;

extern "C" {

const char* skg_version(void) { return "skgpu 0.1.0 sm_100a"; }

const char* skg_last_error(void) { return g_err.c_str(); }

static int create_impl(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                       double dealias_coef, double nu, int scheme, int device, int rank, int world,
                       const char* nccl_id, bool slab_one, int Pz = 1);

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

// 3D pencil decomposition (BASELINE configs[4]): py ranks along
// the kept ky lines / x rows (the slab split) times pz ranks along the kept kz
// modes / y rows; global rank = r_y * pz + r_z.
int skg_create_pencil(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                      double dealias_coef, double nu, int scheme, int device, int rank, int py, int pz,
                      const char* nccl_id) {
    if (py < 1 || pz < 1) return fail(SKG_ECONFIG, "pencil: process grid extents must be >= 1");
    if (std::string(solver ? solver : "") != "ns3d")
        return fail(SKG_EUNSUPPORTED, "pencil decomposition: ns3d only");
    return create_impl(out, solver, dims, n, L, dealias_coef, nu, scheme, device, rank, py, nccl_id, true,
                       pz);
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
                       const char* nccl_id, bool slab_one, int Pz) {
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
    if (generic && (world > 1 || Pz > 1 || (sid == 3 && slab_one)))
        return fail(SKG_EUNSUPPORTED,
                    "slab and compact layouts need the fused kernels' extents (powers of two)");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SKG_ECUDA, "no CUDA device visible (the library has no CPU path)");
    if (device < 0 || device >= ndev) return fail(SKG_ECONFIG, "device ordinal out of range");
    if (world < 1 || rank < 0 || rank >= world * Pz) return fail(SKG_ECONFIG, "bad rank / world size");
    if (Pz > 1 && (n[1] % (2 * Pz) || world * Pz > SKG_MAX_RANKS))
        return fail(SKG_ECONFIG, "pencil: ny must be divisible by 2 * pz and py * pz <= " +
                                     std::to_string(SKG_MAX_RANKS));
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
        c->L[d] = L ? L[d] : skh::kTwoPi;
        c->kscale[d] = skh::kTwoPi / c->L[d];
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
        if (skg::dmalloc(p, bytes < 16 ? 16 : bytes) != cudaSuccess) return false;
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
    c->Pz = Pz;
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
        // need a dealiased state); one partition: no exchange buffers.
        // Pencil (Pz > 1): the kept kz modes split in Pz contiguous ranges.
        const size_t nx = n[0], ny = n[1], kzc = (size_t)c->kc[2] + 1, nrl = c->nrl;
        if ((int)kzc < Pz) return cleanup(SKG_ECONFIG, "more ranks than kept kz modes");
        c->nyl = n[1] / Pz;
        c->zstart.resize(Pz + 1);
        for (int z = 0; z <= Pz; ++z) c->zstart[z] = (int)((long long)z * (long long)kzc / Pz);
        size_t maxcols = 0, maxkz = 0;  // B's field stride is uniform over the ranks (peer exchange)
        for (int q = 0; q < world; ++q) maxcols = std::max(maxcols, (size_t)(c->cstart[q + 1] - c->cstart[q]));
        for (int z = 0; z < Pz; ++z) maxkz = std::max(maxkz, (size_t)(c->zstart[z + 1] - c->zstart[z]));
        for (int q = 0; q < world; ++q)
            for (int z = 0; z < Pz; ++z) {
                if (nccl_id && q * Pz + z != rank) continue;
                Part p;
                p.r = q;
                p.pz = z;
                p.kz0 = c->zstart[z];
                p.nkz = c->zstart[z + 1] - c->zstart[z];
                p.c0 = c->cstart[q];
                p.ncols = c->cstart[q + 1] - c->cstart[q];
                p.vs = nx * p.ncols * p.nkz;
                p.fsz = Pz > 1 ? nrl * (size_t)c->nyl * kzc : 0;
                p.fs = std::max(std::max(nx * maxcols * maxkz, nrl * ny * maxkz), p.fsz);
                p.rfs = nrl * Kyc * p.nkz;
                ok = ok && alloc((void**)&p.u, sizeof(cd) * 3 * p.vs);
                for (int i = 0; i < 3; ++i) ok = ok && alloc((void**)&p.k[i], sizeof(cd) * 3 * p.vs);
                ok = ok && alloc((void**)&p.A3, sizeof(cd) * 5 * p.fs);
                ok = ok && alloc((void**)&p.B3, sizeof(cd) * 6 * p.fs);
                if (Pz > 1) ok = ok && alloc((void**)&p.Z3, sizeof(cd) * 6 * p.fsz);
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
            const ncclResult_t nr = nccl().CommInitRank(&c->comm, world * Pz, id, rank);
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
    // x-forward scratch slots (ns3d.cu k4_3d): measured 512^3 28.95 -> 28.68,
    // 256^3 3.77 -> 3.74 ms/step, 128^3 0.567 -> 0.580 (the claim's atomic and
    // barrier cost more than the write-back there), so from 256 on;
    // SKG_XSCR=0 / 1 forces it off / on
    const char* xs = std::getenv("SKG_XSCR");
    const bool xscr = xs ? std::atoi(xs) != 0 : n[0] >= 256;
    if (sid == 3 && !c->generic && xscr && std::getenv("SKG_NO_XSCR") == nullptr) {
        c->xscr_nsm = skg::max_smid(device);
        ok = ok && alloc((void**)&c->xscr_mask, sizeof(unsigned) * c->xscr_nsm);
        ok = ok && skg::dmalloc(&c->xscr, sizeof(cd) * (size_t)skg::SKG_XSCR_SM * c->xscr_nsm) == cudaSuccess;
    }
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
    skg::dfree(c->u);
    for (auto p : c->k) skg::dfree(p);
    skg::dfree(c->inter);
    skg::dfree(c->io);
    skg::dfree(c->phys);
    skg::dfree(c->work);
    skg::dfree(c->etab);
    skg::dfree(c->flags);
    skg::dfree(c->xscr);
    skg::dfree(c->xscr_mask);
    skg::dfree(c->d_count);
    skg::dfree(c->d_red);
    skg::dfree(c->d_dyn);
    for (void* d : c->ipc_opened) cudaIpcCloseMemHandle(d);
    skg::dfree(c->d_barrier);
    skg::dfree(c->f_ref);
    skg::dfree(c->f_cm);
    skg::dfree(c->f_red);
    if (c->f_noise) cudaFreeHost(c->f_noise);
    skg::dfree(c->gs.w);
    skg::dfree(c->gs.spec);
    skg::dfree(c->gs.nl);
    skg::dfree(c->gs.phys);
    skg::dfree(c->gs.work);
    harvest(c);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (cudaEvent_t e : c->xev)
        if (e) cudaEventDestroy(e);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    for (Part& p : c->parts) {
        skg::dfree(p.u);
        for (auto q : p.k) skg::dfree(q);
        for (int f = 0; f < 2; ++f) {
            skg::dfree(p.sI[f]);
            skg::dfree(p.rI[f]);
            skg::dfree(p.sA[f]);
            skg::dfree(p.rA[f]);
        }
        skg::dfree(p.rD3);
        skg::dfree(p.Z3);
        skg::dfree(p.sZ);
        skg::dfree(p.rZ);
        if (p.rA3 != p.A3) skg::dfree(p.rA3);
        if (p.sD3 != p.B3) skg::dfree(p.sD3);
        skg::dfree(p.A3);
        skg::dfree(p.B3);
    }
    skg::dfree(c->cmfull);
    skg::dfree(c->d_kowner);
    skg::dfree(c->d_cstart);
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
    // one batch in flight: every batch resets the device flags and (CFL) the
    // device time, and sync_and_check accounts one dt per batch, so an
    // earlier batch is checked first (as skg_step does)
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
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
    CUDA_TRY(skg::dmalloc(&d, sizeof(double) * 3 * nsteps));
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
    skg::dfree(d);
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
// Solver::tendency of the reference-layout state in c->io, left in c->io
// (with umax: max |u_d| of it as well, from the same physical pass).
static int tendency_dev(skg_ctx* c, double* umax) {
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
    if (umax) {
        skg::DynStep d;
        CUDA_TRY(cudaMemcpyAsync(&d, c->d_dyn, sizeof(d), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < c->dims; ++k) umax[k] = d.umax[k];
    }
    c->pruned = keep_pruned;
    return SKG_OK;
}

static int tendency_impl(skg_ctx* c, const double* in, double* out, double* umax) {
    if (c->dist) return fail(SKG_EUNSUPPORTED, "skg_tendency on a slab-decomposed context");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(c->io, in, sizeof(cd) * c->S * c->nvars, cudaMemcpyHostToDevice,
                             c->stream));
    if (int rc = tendency_dev(c, umax)) return rc;
    if (out)
        CUDA_TRY(cudaMemcpyAsync(out, c->io, sizeof(cd) * c->S * c->nvars, cudaMemcpyDeviceToHost,
                                 c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SKG_OK;
}

int skg_spectra(skg_ctx* c, int cap, double* k, double* E, double* T, double* D, int* n_shells) {
    // n_shells = round(k_norm_max / delta_k) + 1 (grid.cpp:95, 108)
    double kmax2 = 0.0, Lmax = 0.0;
    for (int d = 0; d < c->dims; ++d) {
        const double km = c->kscale[d] * (c->n[d] / 2);
        kmax2 += km * km;
        Lmax = std::max(Lmax, c->L[d]);
    }
    const double dk = skh::kTwoPi / Lmax;
    const int nsh = (int)std::llround(std::sqrt(kmax2) / dk) + 1;
    if (n_shells) *n_shells = nsh;
    if (!k || !E || !T || !D) return SKG_OK;  // size query
    if (cap < nsh) return fail(SKG_ESHAPE, "skg_spectra: arrays shorter than n_shells");
    if (c->dist) return fail(SKG_EUNSUPPORTED, "skg_spectra on a slab-decomposed context");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->pending_steps) {
        int rc = skg_sync(c);
        if (rc) return rc;
    }
    // state (reference layout) kept in work buffers while io receives the tendency
    if (int rc = ensure_fft_bufs(c)) return rc;
    cd* st = nullptr;
    double* d3 = nullptr;
    CUDA_TRY(skg::dmalloc(&st, sizeof(cd) * c->S * c->nvars));
    CUDA_TRY(skg::dmalloc(&d3, sizeof(double) * 3 * nsh));
    int rc = store_state_to_io(c, c->u);
    if (!rc) {
        cudaMemcpyAsync(st, c->io, sizeof(cd) * c->S * c->nvars, cudaMemcpyDeviceToDevice, c->stream);
        rc = tendency_dev(c, nullptr);
    }
    if (!rc) {
        cudaError_t e = skg::spectra_dev(force_geo(c), st, c->io, c->nu, nsh, d3, c->stream, &c->launches);
        std::vector<double> h(3 * (size_t)nsh);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d3, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                                                  c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) {
            rc = fail(SKG_ECUDA, cudaGetErrorString(e));
        } else {
            for (int s = 0; s < nsh; ++s) {
                k[s] = s * dk;
                E[s] = h[s] / dk;  // bin_shells(..., density = true)
                T[s] = h[nsh + s];
                D[s] = h[2 * nsh + s];
            }
        }
    }
    skg::dfree(st);
    skg::dfree(d3);
    return rc;
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
        skg::dfree(b.u);
        skg::dfree(b.h);
        skg::dfree(b.w);
        b = PlanBufs{};
        CUDA_TRY(skg::dmalloc(&b.u, sizeof(double) * P));
        CUDA_TRY(skg::dmalloc(&b.h, sizeof(cd) * S));
        CUDA_TRY(skg::dmalloc(&b.w, sizeof(cd) * S));
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
        kcut = std::min(kcut, c->coef * (skh::kTwoPi / c->L[d]) * (c->n[d] / 2));  // grid.cpp:83-84
    }
    const double dk = skh::kTwoPi / Lmax;
    if (k_lo > std::sqrt(kmax2))
        return fail(SKG_ECONFIG, "random_field: band lies above the largest resolved |k|");
    if (k_lo < 0.5 * dk || k_hi + 0.5 * dk > kcut)
        return fail(SKG_EUNSUPPORTED,
                    "forcing band must exclude the mean shell and lie inside the dealiasing cut");
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_fft_bufs(c)) return rc;
    if (!c->f_ref) {
        CUDA_TRY(skg::dmalloc(&c->f_ref, sizeof(cd) * c->S * c->nvars));
        CUDA_TRY(skg::dmalloc(&c->f_red, 8 * sizeof(double)));
        CUDA_TRY(cudaMallocHost(&c->f_noise, sizeof(double) * c->P * c->nvars));
        if (c->solver == 2 && !c->generic) CUDA_TRY(skg::dmalloc(&c->f_cm, sizeof(cd) * c->S));
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

// ---- peer-memory exchange for the ns2d slab (include/skgpu.h)
static const int kIpcBytes = 4 * (int)sizeof(cudaIpcMemHandle_t);

int skg_dist_ipc_handle(skg_ctx* c, char* out) {
    if (!c->dist || c->G * c->Pz < 2 || c->parts.size() != 1)
        return fail(SKG_EUNSUPPORTED, "IPC handles: one slab partition per process");
    if (skg::guards_enabled()) return fail(SKG_EUNSUPPORTED, "IPC handles: not with SKG_GUARD=1 (offset allocations)");
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_p2p_bufs(c)) return rc;
    const Part& p = c->parts[0];
    cd* bufs[4] = {p.rI[0], p.rI[1], p.rA[0], p.rA[1]};
    if (c->solver == 3) {  // pencil: + the z-pass input and the y-pass buffer
        bufs[0] = p.rA3;
        bufs[1] = p.rD3;
        bufs[2] = p.Z3;
        bufs[3] = p.B3;
    }
    const int nb = c->solver == 3 ? (c->Pz > 1 ? 4 : 2) : 4;
    std::memset(out, 0, kIpcBytes);
    for (int b = 0; b < nb; ++b) {
        cudaIpcMemHandle_t h;
        CUDA_TRY(cudaIpcGetMemHandle(&h, bufs[b]));
        std::memcpy(out + b * sizeof(h), &h, sizeof(h));
    }
    return SKG_OK;
}

int skg_dist_open_peers(skg_ctx* c, const char* all) {
    const int W = c->G * c->Pz;  // global ranks (pencil: r Pz + pz)
    if (!c->dist || W < 2 || c->parts.size() != 1 || !c->comm)
        return fail(SKG_EUNSUPPORTED, "peer exchange across processes: NCCL slab contexts");
    if (W > SKG_MAX_RANKS) return fail(SKG_EUNSUPPORTED, "peer exchange: too many ranks");
    CUDA_TRY(cudaSetDevice(c->device));
    const Part& me = c->parts[0];
    const int nb = c->solver == 3 ? (c->Pz > 1 ? 4 : 2) : 4;
    for (int q = 0; q < W; ++q) {
        cd* ptr[4] = {nullptr, nullptr, nullptr, nullptr};
        if (q == c->grank) {
            ptr[0] = c->solver == 3 ? me.rA3 : me.rI[0];
            ptr[1] = c->solver == 3 ? me.rD3 : me.rI[1];
            ptr[2] = c->solver == 3 ? me.Z3 : me.rA[0];
            ptr[3] = c->solver == 3 ? me.B3 : me.rA[1];
        } else {
            for (int b = 0; b < nb; ++b) {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, all + (size_t)q * kIpcBytes + b * sizeof(h), sizeof(h));
                void* d = nullptr;
                CUDA_TRY(cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess));
                c->ipc_opened.push_back(d);
                ptr[b] = static_cast<cd*>(d);
            }
        }
        if (c->solver == 3) {
            c->peer_rA3[q] = ptr[0];
            c->peer_D3[q] = ptr[1];
            c->peer_Z3[q] = ptr[2];
            c->peer_B3[q] = ptr[3];
            continue;
        }
        c->peer_rI[q][0] = ptr[0];
        c->peer_rI[q][1] = ptr[1];
        c->peer_rA[q][0] = ptr[2];
        c->peer_rA[q][1] = ptr[3];
    }
    if (!c->d_barrier) CUDA_TRY(skg::dmalloc(&c->d_barrier, sizeof(double)));
    c->p2p = true;
    return SKG_OK;
}

long skg_guard_violations(void) { return skg::guard_violations(); }

int skg_dist_overlap(skg_ctx* c, int enable) {
    if (!c->dist) return fail(SKG_EUNSUPPORTED, "exchange overlap: slab-decomposed contexts");
    if (c->gexec) {  // the captured step holds the old exchange sequence
        CUDA_TRY(cudaSetDevice(c->device));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    c->no_overlap = !enable;
    c->zpack = enable == 2;  // pencil, single process: the NCCL route's pack / unpack blocks
    c->zfuse = enable != 3;  // 3: the kz -> y transpose as a separate strided-copy kernel
    return SKG_OK;
}

int skg_dist_p2p(skg_ctx* c, int enable) {
    if (!enable) {
        c->p2p = false;
        return SKG_OK;
    }
    if (!c->dist || c->G * c->Pz < 2) return fail(SKG_EUNSUPPORTED, "peer exchange: slab-decomposed contexts");
    if (c->comm) return fail(SKG_ECONFIG, "multi-process contexts: skg_dist_open_peers");
    if (c->G * c->Pz > SKG_MAX_RANKS) return fail(SKG_EUNSUPPORTED, "peer exchange: too many ranks");
    if (c->G < 2) return SKG_OK;  // 1 x Pz pencil: the kz <-> y transposes store into the parts already
    if (int rc = ensure_p2p_bufs(c)) return rc;
    for (const Part& p : c->parts) {
        if (c->solver == 3) {
            c->peer_rA3[p.r * c->Pz + p.pz] = p.rA3;
            c->peer_D3[p.r * c->Pz + p.pz] = p.rD3;
            c->peer_Z3[p.r * c->Pz + p.pz] = p.Z3;
            c->peer_B3[p.r * c->Pz + p.pz] = p.B3;
            continue;
        }
        for (int f = 0; f < 2; ++f) {
            c->peer_rI[p.r][f] = p.rI[f];
            c->peer_rA[p.r][f] = p.rA[f];
        }
    }
    c->p2p = true;
    return SKG_OK;
}

int skg_set_timing(skg_ctx* c, int enable) {
    c->timing = enable != 0;
    return SKG_OK;
}

int skg_fp64_peak(int device, double* dfma_per_s) {
    if (!dfma_per_s) return fail(SKG_ECONFIG, "fp64_peak: null output pointer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SKG_ECUDA, "no CUDA device visible (the library has no CPU path)");
    if (device < 0 || device >= ndev) return fail(SKG_ECONFIG, "device ordinal out of range");
    CUDA_TRY(skg::fp64_peak(device, dfma_per_s));
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
