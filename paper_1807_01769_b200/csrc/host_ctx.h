// host_ctx.h -- host side of libskgpu: the context (skg_ctx), its device
// buffers and the helpers shared by host_ctx.cu (tables, kernel arguments,
// state I/O), host_step.cu (step enqueueing, slab exchange, forcing) and
// skgpu.cu (the extern "C" boundary).  Not part of the public ABI.
#pragma once
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

namespace skh {

// NCCL, resolved with dlopen on first multi-GPU use (host_ctx.cu)
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
NcclApi& nccl();

// thread-local message of the last failing call (skg_last_error)
extern thread_local std::string g_err;
int fail(int code, const std::string& msg);

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return skh::fail(SKG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr double kTwoPi = 6.283185307179586476925286766559;  // grid.cpp:11

std::vector<cd> twiddles(int n);
int cut_index(int n, double L, double coef, bool half);

}  // namespace skh


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
    cd* rD3 = nullptr;  // p2p: y-forward receive buffer (3 fields, stride dfs3)
    size_t vs = 0, fs = 0, rfs = 0;
    // ns3d pencil layout (skg_create_pencil): r is the rank along the ky-line /
    // x-row split (Py), pz the rank along the kept-kz / y-row split (Pz); the
    // part holds the kept kz modes [kz0, kz0 + nkz) in its x and y passes and
    // the y rows [pz nyl, (pz + 1) nyl) in its z pass.  Z3: the z pass's six
    // input fields [xl][yl][kz] (all kept kz), stride fsz; its three outputs
    // go to A3 with the same stride.  sZ / rZ: pack / unpack blocks of the
    // NCCL route of the two kz <-> y transposes.
    int pz = 0, kz0 = 0, nkz = 0;
    cd* Z3 = nullptr;
    cd* sZ = nullptr;
    cd* rZ = nullptr;
    size_t fsz = 0;
};

struct skg_ctx {
    int device = 0;
    int nsm = 148;
    int solver = 2;  // 2: ns2d, 3: ns3d
    int dims = 2;
    int n[3] = {1, 1, 1};
    double L[3] = {skh::kTwoPi, skh::kTwoPi, skh::kTwoPi};
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
    // ns3d x-forward scratch (k4_3d): per-SM slots for the transformed
    // components 0 and 1 of a CTA, claimed through a per-SM bit mask
    cd* xscr = nullptr;
    unsigned* xscr_mask = nullptr;
    int xscr_nsm = 0;
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
    // ns3d pencil: G ranks along ky lines / x rows times Pz ranks along the
    // kept kz / y rows; global rank = r Pz + pz; zstart: kz ranges (Pz + 1)
    int Pz = 1, nyl = 0;
    bool zfuse = true;   // kz -> y transpose from the y-inverse's stores (skg_dist_overlap(ctx, 3): off)
    bool zpack = false;  // single process: run the NCCL route's pack / unpack (skg_dist_overlap(ctx, 2))
    std::vector<int> zstart;
    cd* peer_Z3[SKG_MAX_RANKS] = {};   // pencil: z-pass input buffers (Z3) by global rank
    cd* peer_B3[SKG_MAX_RANKS] = {};   // pencil: y-pass buffers (B3) by global rank
    std::vector<Part> parts;
    int* d_kowner = nullptr;
    int* d_cstart = nullptr;
    cd* cmfull = nullptr;     // full CM staging for set/get_state
    ncclComm_t comm = nullptr;
    double* diag = nullptr;   // per-step (E, Z, eps) series of skg_run (device)
    // peer-memory exchange (ns2d slab): receive buffers of every partition
    // (local parts, or CUDA-IPC-mapped peers); p2p replaces the copies
    bool p2p = false;
    cd* peer_rI[SKG_MAX_RANKS][2] = {};
    cd* peer_rA[SKG_MAX_RANKS][2] = {};
    cd* peer_rA3[SKG_MAX_RANKS] = {};  // ns3d: x-inverse receive buffers
    cd* peer_D3[SKG_MAX_RANKS] = {};   // ns3d: y-forward receive buffers (rD3)
    size_t dfs3 = 0;                   // ns3d: their field stride (uniform)
    std::vector<void*> ipc_opened;  // cudaIpcOpenMemHandle mappings to close
    double* d_barrier = nullptr;    // one double all-reduced as the cross-rank barrier
    // ns3d copy / NCCL exchange chunked per field on a second stream
    // (enqueue_dist_step3_chunked); no_overlap keeps it on the context stream
    cudaStream_t cstream = nullptr;
    cudaEvent_t xev[7] = {};
    bool no_overlap = false;

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
    bool g_p2p = false;  // exchange mode the graph was captured with
    cudaStream_t g_stream = nullptr;
};


namespace skh {

// kernel-class timing (skg_set_timing)
skg::LaunchHook hook_of(skg_ctx* c);
void harvest(skg_ctx* c);
// integrating-factor tables and kernel arguments
int refresh_exp(skg_ctx* c, double dt);
const double* etab_ptr(const skg_ctx* c, int which, int axis);
int env_opt();
int sm_count(int device);
skg::Ns2dArgs args2d(skg_ctx* c, double dt);
skg::Ns2dArgs args2d_part(skg_ctx* c, double dt, const Part& p);
skg::Ns3dArgs args3d(skg_ctx* c, double dt);
skg::Ns3dArgs args3d_part(skg_ctx* c, double dt, const Part& p);
int energy_mode(const skg_ctx* c);
skg::GenArgs args_gen(skg_ctx* c, double dt);
skg::ForceGeo force_geo(const skg_ctx* c);
// state I/O between the reference layout (io) and the internal layouts
int decide_pruned(skg_ctx* c, const cd* d_ref_layout);
int copy_slab3(skg_ctx* c, const Part& p, bool to_part);
int load_state_from_io(skg_ctx* c);
int store_state_to_io(skg_ctx* c, const cd* src);
int ensure_fft_bufs(skg_ctx* c);
int ensure_p2p_bufs(skg_ctx* c);
cd* twiddle_table(int device, int n);
// stepping (host_step.cu)
int refresh_forcing(skg_ctx* c);
int sync_and_check(skg_ctx* c, long nsteps, double dt);
int exchange(skg_ctx* c, int which);
int exchange_z(skg_ctx* c, int dir, cudaStream_t st = nullptr);
int enqueue_steps(skg_ctx* c, double dt, long nsteps);

}  // namespace skh
