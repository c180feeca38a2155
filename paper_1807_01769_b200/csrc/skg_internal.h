// skg_internal.h -- shared host/device declarations of the skgpu library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "fft_block.cuh"

#define SKG_MAX_RANKS 16  // slab partitions addressable by the peer-memory path

namespace skg {

// Device flags shared by every kernel of a context (one allocation).
struct DevFlags {
    int diverged;   // set by the final RK update on a non-finite value
    int div_var;    // variable index of the first non-finite value
    int div_step;   // step counter value (1-based within the launch batch)
    int steps;      // steps started since the counter was last reset
    int bad_dt;     // adaptive dt: nonpositive dt (past t_end) at step div_step
};

// The divergence flag as one value per CTA: CTAs of the grid that sets it
// (the final RK update) may see it change while they start, and a kernel
// whose threads disagree would leave some of them waiting at a barrier.
// All threads of the CTA must call it (kernel entry, before any return).
__device__ __forceinline__ bool cta_diverged(const DevFlags* f) {
    return __syncthreads_or(*reinterpret_cast<const volatile int*>(&f->diverged)) != 0;
}

// Adaptive (CFL) time step, device-resident so replayed graphs follow it
// (Simulation::compute_dt + compute_cfl_dt, simulation.cpp:463-476,
// time_stepping.cpp:15-26).  The stage-1 physical pass of every step reduces
// max |u_d| of the step's initial state (Solver::max_velocity_per_axis,
// solvers.cpp:176-194, 341-357) into umax; dt_update then sets dt and the
// integrating-factor tables before stage 2.
struct DynStep {
    double dt, hdt, sdt;
    double umax[3];      // non-negative: ordered like their bit patterns
    double t;            // time at the start of the current step
    double t_end;        // < 0: no clamp
    double cfl, dt_max;
    double dx[3];
    double last_dt;
};

template <class A>
__device__ __forceinline__ double dt_of(const A& a) { return a.dyn ? a.dyn->dt : a.dt; }
template <class A>
__device__ __forceinline__ double hdt_of(const A& a) { return a.dyn ? a.dyn->hdt : a.hdt; }
template <class A>
__device__ __forceinline__ double sdt_of(const A& a) { return a.dyn ? a.dyn->sdt : a.sdt; }

// max(|a|, |b|, |c|) of one thread's points into dyn->umax (warp max, then one
// atomic per warp and axis).
__device__ __forceinline__ void umax_accumulate(DynStep* dyn, int naxes, double a, double b, double c) {
    for (int o = 16; o > 0; o >>= 1) {
        a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* u = reinterpret_cast<unsigned long long*>(dyn->umax);
        atomicMax(u + 0, (unsigned long long)__double_as_longlong(a));
        atomicMax(u + 1, (unsigned long long)__double_as_longlong(b));
        if (naxes > 2) atomicMax(u + 2, (unsigned long long)__double_as_longlong(c));
    }
}

// Grid description shared by the 2D and 3D solvers.  Axis 0 is the slowest
// (row-major), the last axis is the half-stored Hermitian one.
struct GridDesc {
    int dims;
    int n[3];        // physical extents (padded with 1 on the left for 2D: NOT used)
    int nh;          // n[dims-1]/2 + 1
    int kc[3];       // keep iff |signed index| <= kc[d]  (bit-exact dealias rule)
    double kscale[3];  // 2 pi / L_d: k = kscale * signed index
};

__host__ __device__ __forceinline__ int signed_index(int i, int n) { return i <= n / 2 ? i : i - n; }

// ---------------------------------------------------------------- ns2d
// Internal spectral layout "CM": [ky][kx] (each ky column contiguous over
// kx), nh columns of nx complex.  Intermediates between the x and y passes
// are row-major [x][ky] with row stride ld (only the ky columns that can be
// non-zero are stored).
struct Ns2dArgs {
    int opt;            // tuning bits (SKG_OPT, read once on the host)
    int wave;           // resident CTAs of the x passes (next-wave prefetch)
    int nx, ny, nh;
    int kcx, kcy;       // dealias: keep |kx_i| <= kcx and ky_i <= kcy
    int ky_in;          // columns read by the x-inverse pass (kcy+1 pruned, nh full)
    int ld_i;           // row stride of the four intermediates (= ky_in)
    int ld_o;           // row stride of the tendency rows (= kcy+1)
    int pruned;         // 1: state is dealiased, skip masked modes
    int has_sigma;      // nu != 0
    int rk2;            // scheme
    double kx_scale, ky_scale;
    double inv_n;       // 1 / (nx ny)
    double dt, hdt, sdt;
    DynStep* dyn;       // adaptive dt (nullptr: the fixed dt above)
    int ystage;         // RK stage of the physical pass (stage 1 feeds the CFL max)
    const cd* force;    // forcing addend in the state layout (nullptr: off)
    const double* e1x;  // exp(0.5 dt (-nu kx^2)) per kx index (nx)
    const double* e1y;  // exp(0.5 dt (-nu ky^2)) per ky index (nh)
    const double* e2x;  // exp(dt (-nu kx^2))
    const double* e2y;
    cd* u;              // state (CM)
    cd* k1;
    cd* k2;
    cd* k3;
    cd* I[4];           // X[psi], X[kx psi], X[kx w], X[w]  ([x][ld_i])
    cd* nl;             // tendency rows [x][ld_o] (x-space, ky spectral)
    const cd* twx;      // W_nx table
    const cd* twy;      // W_ny table
    DevFlags* flags;
    double* diag;       // per-step (E, Z, eps) series, slot steps-1; nullptr = off
    double nu;
    // Slab decomposition of the dealiased fast path (G = 1 on one GPU):
    // this partition owns the kept ky columns [c0, c0 + ncols) (c0 even) of
    // the state and the x rows [r nrl, (r + 1) nrl) of physical space.
    //   sI/rI: x-inverse outputs X[psi], X[kx psi]; send block for rank q =
    //          rows(q) x own columns, row-quad interleaved ((xl/4) ncols + kyl) 4 + xl%4;
    //          receive block from r' at nrl * cstart[r'] with r's layout.
    //   sA/rA: product spectra; send layout ((k/2) nrl + xl) 2 + k%2 (blocks in
    //          pair order), receive block from r' at r' * 2 npairs nrl.
    // With G = 1 send and receive alias and the layouts reduce to the
    // single-GPU ones.
    int G, r, c0, ncols, nrl;
    int lg_nrl;         // log2(nrl) (nx and G are powers of two)
    int lead;           // this partition advances the step counter
    const int* kowner;  // owning rank of each kept column (kcy + 1 entries)
    const int* cstart;  // first column of each rank (G + 1 entries)
    cd* sI[2];
    cd* rI[2];
    cd* sA[2];
    cd* rA[2];
    // Peer-memory exchange (p2p = 1): the x-inverse and y-pass epilogues store
    // straight into the destination partition's receive buffers -- the same
    // GPU in the single-process mode, CUDA-IPC-mapped peer memory over NVLink
    // across processes -- so the all-to-all copies disappear (the transfer
    // overlaps the FFTs tile by tile) and only a barrier remains.
    int p2p;
    cd* peer_rI[SKG_MAX_RANKS][2];
    cd* peer_rA[SKG_MAX_RANKS][2];
};

// Optional per-launch instrumentation: hook(user, cls, 0, 0) before a launch
// and hook(user, cls, 1, algorithmic_bytes) after it.
struct LaunchHook {
    void (*fn)(void* user, int cls, int phase, double bytes) = nullptr;
    void* user = nullptr;
    void begin(int cls) const {
        if (fn) fn(user, cls, 0, 0.0);
    }
    void end(int cls, double bytes) const {
        if (fn) fn(user, cls, 1, bytes);
    }
};

// Launchers (ns2d.cu).  stage in 1..4 (RK4) or 1..2 (RK2); stage 0 = plain
// tendency evaluation of u into k1 (no RK arithmetic).
cudaError_t ns2d_launch_stage(const Ns2dArgs& a, int stage, cudaStream_t s, long* launches,
                              const LaunchHook& hook);
// The three passes of the fast path separately (slab decomposition):
// pass 0 x-inverse, 1 y pass, 2 x-forward + RK.
bool ns2d_fast_ok(const Ns2dArgs& a);
// Dealiased-path passes: 0 x-inverse, 1 y pass, 2 x-forward + RK,
// 3 x-forward + RK fused with the x-inverse of the next stage (next != 0;
// after the final stage: stage 1 of the next step).
cudaError_t ns2d_fast_pass(const Ns2dArgs& a, int pass, int stage, cudaStream_t s, long* launches,
                           const LaunchHook& hook, int next = 0);
bool ns2d_supported(int nx, int ny);

// ---------------------------------------------------------------- ns3d
// State and RK buffers keep the reference layout [kx][ky][kz] (kz the
// half axis, nh = nz/2 + 1).  Intermediates (all row-major, kz fastest):
//   A[5] after the x-inverse pass  (x, ky, kz)  kz < kz_in   X[vx] X[vy] X[vz] X[kx vy] X[kx vz]
//   B[6] after the y-inverse pass  (x, y, kz)   kz < kz_in   u v w wx wy wz (still kz-spectral)
//   C[3] after the z pass          (x, y, kz)   kz <= kcz    (u x w)^ in kz
//   D[3] after the y-forward pass  (x, ky, kz)  kz <= kcz
// C aliases A and D aliases B (each is dead when the other is produced).
struct Ns3dArgs {
    int opt;                // tuning bits (SKG_OPT)
    int wave;               // resident 256-thread CTAs (2 per SM)
    int nx, ny, nz, nh;
    int kcx, kcy, kcz;
    int pruned, has_sigma, rk2;
    int kz_in;           // kz extent of A/B (kcz+1 pruned, nh full)
    int kz_o;            // kz extent of C/D (= kcz+1)
    int ky_lines;        // ky lines of the x passes (2kcy+1 pruned, ny full)
    double kx_scale, ky_scale, kz_scale;
    double inv_n;
    double dt, hdt, sdt;
    DynStep* dyn;       // adaptive dt (nullptr: the fixed dt above)
    int ystage;         // RK stage of the physical pass (stage 1 feeds the CFL max)
    int comp0 = 0;      // x-inverse / y-forward launches: components [comp0, comp0 + ncomp)
    int ncomp = 3;
    const cd* force;    // forcing addend in the state layout (nullptr: off)
    const double *e1x, *e1y, *e1z, *e2x, *e2y, *e2z;
    cd* u;               // 3 variables, each nx*ny*nh (reference layout)
    cd* k1;
    cd* k2;
    cd* k3;
    size_t vstride;      // elements between variables of u/k1/k2/k3
    cd* A;               // 5 fields, stride fstride
    cd* B;               // 6 fields
    size_t fstride;      // elements per intermediate field (nx*ny*nh)
    const cd *twx, *twy, *twz;
    DevFlags* flags;
    double* diag;           // per-step (E, Z, eps) series, slot steps-1; nullptr = off
    double nu;
    // Slab layout (slab = 1; G partitions, G = 1 is the compact single-GPU
    // layout): this rank owns the kept ky lines [kys, kys + nkyl) (compact
    // kept index kyi: 0..kcy, then the negative ky) of the state and the x
    // rows [r nrl, (r + 1) nrl) of the y/z passes.  The state and the x-pass
    // intermediates are indexed ((x * ystate + ys) * kz + ...) with
    // ystate = ny, ys = ky in the full layout (slab = 0) and ystate = nkyl,
    // ys = kyi - kys in the slab layout (send/receive blocks of the two
    // all-to-alls are then contiguous x ranges; state lines hold only the
    // kept kz).  y-pass reads of A and writes of D go through the owner
    // table of each kept line.
    int G, r, lead, kys, nkyl, nrl;
    int slab;               // 1: partitioned layout (any G, including one partition)
    int ystate;
    int sz;                 // kz extent of a state line (nh; kz_in = kcz + 1 in slab layout)
    const int* kowner;      // owner rank of each compact kept ky line (2 kcy + 1)
    const int* kstart;      // first compact line of each rank (G + 1)
    cd* rA;                 // received x-inverse outputs (5 fields, stride rfs), G > 1
    cd* sD;                 // y-forward outputs to send (3 fields, stride rfs), G > 1
    size_t rfs;
    // peer-memory exchange (see Ns2dArgs): every rank's x-inverse receive
    // buffer (5 fields, stride rfs) and y-forward receive buffer rD (3 fields,
    // stride dfs, uniform over the ranks)
    int p2p;
    cd* peer_rA[SKG_MAX_RANKS];
    cd* peer_D[SKG_MAX_RANKS];
    cd* rD;                 // p2p: this rank's y-forward receive buffer (3 fields, stride dfs);
    size_t dfs;             // B stays the y/z-pass intermediate, which peers must not touch
    // Pencil layout (slab over ky lines / x rows as above, times a split of
    // the kept kz modes over Pz ranks): this rank's x and y passes see the kz
    // modes [kz0, kz0 + kz_in) only (local index kz, global kz0 + kz); the
    // factor tables e1z / e2z are passed already shifted by kz0.
    int kz0 = 0;
    // kz -> y transpose fused into the y-inverse's stores (zfused; all parts
    // in one process or peer memory): output (m, x, y, kz) goes straight to
    // the z-pass input of the pz-group member y / nyl, Z3 [xl][yl][kzf]
    // (field stride fsz), instead of this rank's B.
    int zfused = 0, lg_nyl = 0, nyl = 0, kzf = 0;
    size_t fsz = 0;
    cd* peer_Z[SKG_MAX_RANKS];
    // x-forward scratch: xscr_nsm regions of SKG_XSCR_SM elements, one per
    // %smid, and the per-SM claim masks (nullptr: in-place write-back)
    cd* xscr = nullptr;
    unsigned* xscr_mask = nullptr;
    int xscr_nsm = 0;
};
// per-SM scratch region: 1024 resident threads x 2 components x 16 elements
constexpr int SKG_XSCR_SM = 1024 * 2 * 16;

// Programmatic dependent launch (sm_90+): step kernels are launched with
// programmatic stream serialization and wait (griddepcontrol.wait) for their
// predecessor's completion and memory flush before touching anything it
// wrote, so the next launch is processed while the previous grid drains.  An
// explicit early launch_dependents trigger was measured slower (dependent
// CTAs parked on SMs: 0.146 -> 0.179 ms/step at 1024^2) and is not used.
// The wait is a no-op for a launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// L2 prefetch of [p, p + bytes) (bytes a multiple of 16, p 16-byte aligned),
// split in 4 KB bulk requests over the calling threads.
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes, int t, int nt) {
    const char* c = static_cast<const char*>(p);
    for (size_t off = (size_t)t * 4096; off < bytes; off += (size_t)nt * 4096) {
        const unsigned n = (unsigned)(bytes - off < 4096 ? bytes - off : 4096);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(c + off), "r"(n) : "memory");
    }
}

// Bulk (TMA 1D) global -> shared copies completing on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes)
                 : "memory");
}
// dst, src 16-byte aligned; bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mb) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W;\n"
        "}\n" ::"r"(smem_u32(mb)),
        "r"(parity)
        : "memory");
}

// Warp-sum three doubles and add them to slot[0..2] (all 32 lanes must call).
__device__ __forceinline__ void diag_accumulate(double* slot, double e, double z, double d) {
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_down_sync(0xffffffffu, e, o);
        z += __shfl_down_sync(0xffffffffu, z, o);
        d += __shfl_down_sync(0xffffffffu, d, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (e != 0.0) atomicAdd(&slot[0], e);
        if (z != 0.0) atomicAdd(&slot[1], z);
        if (d != 0.0) atomicAdd(&slot[2], d);
    }
}
cudaError_t ns3d_launch_stage(const Ns3dArgs& a, int stage, cudaStream_t s, long* launches,
                              const LaunchHook& hook);
// Slab pieces: pass 0 x-inverse, 1 y-inverse + z + y-forward, 2 x-forward + RK;
// pass 3 = y-inverse + z alone, 4 = y-forward alone (a.comp0 / a.ncomp pick
// the fields of passes 0 and 4).
cudaError_t ns3d_pass(const Ns3dArgs& a, int pass, int stage, cudaStream_t s, long* launches,
                      const LaunchHook& hook);
bool ns3d_supported(int nx, int ny, int nz);

// ---------------------------------------------------------------- utilities (util.cu)
cudaError_t launch_transpose_c(const cd* in, cd* out, int rows, int cols, int conj_flag,
                               cudaStream_t s, long* launches);  // out[c][r] = in[r][c]
// Strided box copy of complex fields (the pencil decomposition's kz <-> y
// transposes): dst[f df + x dx + y dy + z] = src[f sf + x sx + y sy + z] for
// f < nf, x < nx, y < ny, z < nz (z contiguous on both sides; dst may be peer
// memory).  fence: __threadfence_system after the stores (peer destinations).
struct BoxCopy {
    const cd* src;
    cd* dst;
    int nf, nx, ny, nz;
    size_t sf, sx, sy, df, dx, dy;
};
cudaError_t launch_box_copy(const BoxCopy& b, bool fence, cudaStream_t s, long* launches);
cudaError_t launch_count_masked(const cd* f, int dims, const int* n, const int* kc, int nvars,
                                long long spect_size, unsigned long long* d_count,
                                cudaStream_t s, long* launches);
cudaError_t launch_grid_dump(int dims, const int* n, const int* kc, const double* kscale,
                             int axis, double* d_k, unsigned char* d_mask, cudaStream_t s,
                             long* launches);
cudaError_t fp64_peak(int device, double* dfma_per_s);  // util.cu (skg_fp64_peak)
// Return the error of a CUDA call from a cudaError_t function.
#define SKG_TRY(...)                                \
    do {                                            \
        const cudaError_t skg_e_ = (__VA_ARGS__);   \
        if (skg_e_ != cudaSuccess) return skg_e_;   \
    } while (0)

// Generic (unfused) step for extents outside the fused kernels' range
// (generic.cu): reference layout, one pass per reference operator.
struct GenArgs {
    int dims, n[3], nh, kc[3];
    double ks[3];
    long long S, P;
    int nvars, has_sigma, rk2;
    double dt, hdt, sdt;
    DynStep* dyn;
    const double* e1[3];
    const double* e2[3];
    cd *u, *k1, *k2, *k3;
    DevFlags* flags;
    const cd* force;  // forcing addend (nullptr: off)
};
struct GenScratch {
    cd* w;        // stage state (nvars S)
    cd* spec;     // spectral inputs of the inverse transforms (4 S in 2D, 3 S in 3D)
    cd* nl;       // forward-transformed products (nvars S)
    double* phys; // physical fields (4 P in 2D, 6 P in 3D)
    cd* work;     // transform scratch (S)
    const cd* tw[3];
};
cudaError_t generic_stage(const GenArgs& a, int stage, GenScratch& g, cudaStream_t s, long* launches);
// Tendency of w into g.nl (kout == nullptr) with the stage-1 CFL reduction
// when a.dyn is set.
cudaError_t generic_tendency(const GenArgs& a, const cd* w, int stage, cd* kout, GenScratch& g,
                             cudaStream_t s, long* launches);

// Random band forcing (forcing.cu), reference layout.
struct ForceGeo {
    int dims, n[3], nh, kc[3], nvars;
    double ks[3];
    long long S;
    double delta_k, k_lo, k_hi;
};
// band filter + unit magnitude + prepare_forcing of the transformed noise f
cudaError_t forcing_shape(const ForceGeo& g, cd* f, cudaStream_t s, long* launches);
// per-shell energy, transfer and dissipation into out3 = [E | T | D] (nsh each)
cudaError_t spectra_dev(const ForceGeo& g, const cd* u, const cd* nl, double nu, int nsh, double* out3,
                        cudaStream_t s, long* launches);
// Solver::sanitize_state of a reference-layout state
cudaError_t sanitize_dev(const ForceGeo& g, cd* f, cudaStream_t s, long* launches);
// reductions against the state u, the rate split, f <- alpha f + beta ub;
// red: 8 doubles (red[6] = last injection, red[7] = 1 on the fallback)
cudaError_t forcing_finish(const ForceGeo& g, const cd* u, cd* f, double rate, double* red,
                           cudaStream_t s, long* launches);

// Device allocations of the library.  With SKG_GUARD=1 in the environment
// every allocation gets 64 KB guard zones before and after it, filled with a
// byte pattern; guard_violations() counts the guard bytes that changed (an
// out-of-bounds write by any kernel or copy).  Debug aid where
// compute-sanitizer is unavailable; IPC export is refused in this mode.
cudaError_t dmalloc_raw(void** p, size_t bytes);
void dfree(void* p);
int max_smid(int device);
long guard_violations();
bool guards_enabled();
template <class T>
inline cudaError_t dmalloc(T** p, size_t bytes) {
    return dmalloc_raw(reinterpret_cast<void**>(p), bytes);
}

// Opt a kernel in to `bytes` of dynamic shared memory on the CURRENT device
// (cudaFuncSetAttribute is per device): recorded per (kernel, device) under a
// mutex, so a second device or a second thread gets its own attribute call;
// a no-op up to the 48 KB default.  Returns the attribute call's error.
cudaError_t ensure_smem(const void* kernel, size_t bytes);

// Launch with the programmatic-stream-serialization attribute (PDL).
template <typename... KP, typename... A>
inline cudaError_t launch_pdl(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              A... args) {
    SKG_TRY(ensure_smem(reinterpret_cast<const void*>(k), smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

// dt from umax (CFL), clamp to t_end, integrating-factor tables for it
// (layout of skgpu.cu etab_ptr), umax reset; flags->bad_dt if dt <= 0.
cudaError_t launch_dt_update(DynStep* dyn, DevFlags* flags, double* etab, int dims, const int* n,
                             const double* kscale, double nu, cudaStream_t s, long* launches);
cudaError_t launch_energy(const cd* f, int dims, const int* n, const double* kscale, int nvars,
                          int solver2d, double* d_out, cudaStream_t s, long* launches,
                          double nu = 0.0, const int* steps = nullptr, bool zero_first = true);

// Plain transforms on the context grid / arbitrary shapes (fft_ops.cu).
// u: row-major real (n0..n_{d-1}); uhat: row-major half spectrum.
cudaError_t fft_forward_dev(int rank, const int* n, const double* d_u, cd* d_uhat, cd* d_work,
                            const cd* const* tw, cudaStream_t s, long* launches, bool normalize = true);
cudaError_t fft_inverse_dev(int rank, const int* n, const cd* d_uhat, double* d_u, cd* d_work,
                            const cd* const* tw, cudaStream_t s, long* launches);
bool fft_pow2(int n);

}  // namespace skg
