/*
 * skgpu.h -- C ABI of the B200-native pseudo-spectral Navier-Stokes step.
 *
 * Drop-in boundary for the reference's hot path (spectralkit, mounted at
 * /root/reference; paths below are relative to /root/reference/proj).
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void*).  Host pointers are borrowed for the
 * duration of a call (copy-in / copy-out); *_device variants take device
 * pointers for zero-copy use.  Spectral arrays use the reference layout:
 * per variable, row-major over (n0, ..., n_{d-1}/2+1), complex128
 * interleaved (re, im) -- include/spectralkit/grid.hpp:18-25,
 * include/spectralkit/state.hpp (StateSet spectral storage).
 *
 * Status codes mirror include/spectralkit/errors.hpp:
 *   SKG_ECONFIG     <- ConfigError / ParamError   (bad extents, nu < 0, dt <= 0)
 *   SKG_ESHAPE      <- ShapeError                 (size mismatch, bad axis)
 *   SKG_EDIVERGENCE <- DivergenceError(iteration, field)  (simulation.cpp:557-563)
 *   SKG_ECUDA       CUDA runtime failure (no reference equivalent)
 *   SKG_EUNSUPPORTED extent outside what the sm_100a kernels implement
 * One context per host thread, as the reference allows one thread per
 * Simulation.  skg_last_error() is thread-local.
 */
#ifndef SKGPU_H
#define SKGPU_H

#ifdef __cplusplus
extern "C" {
#endif

#define SKG_OK 0
#define SKG_ECONFIG 1
#define SKG_ESHAPE 2
#define SKG_EDIVERGENCE 3
#define SKG_ECUDA 4
#define SKG_ENCCL 5
#define SKG_EUNSUPPORTED 6

#define SKG_RK4 0 /* Scheme::RK4, include/spectralkit/time_stepping.hpp:14 */
#define SKG_RK2 1 /* Scheme::RK2 */

typedef struct skg_ctx skg_ctx;

/* Version string of the library ("skgpu <semver> sm_100a"). */
const char* skg_version(void);

/* Thread-local message of the last failing call on this thread. */
const char* skg_last_error(void);

/*
 * Create a solver context on one device.
 *   solver: "ns2d" (vorticity form, 1 variable "rot") or "ns3d" (rotational
 *           form, 3 variables vx, vy, vz) -- replaces resolve_solver +
 *           Solver factory (simulation.cpp:33-70, solvers.cpp:398-427).
 *   dims/n/L: grid extents and box lengths -- replaces make_grid
 *           (grid.cpp:20-110); L == NULL means 2*pi on every axis.
 *   dealias_coef: 2/3 in every BASELINE config (simulation.cpp:91).
 *   nu:     nu_2; sigma = -nu |k|^2 (Solver::linear_coef, simulation.cpp:147-157);
 *           nu == 0 selects the "no linear part" RK branch (time_stepping.cpp:177-185).
 *   scheme: SKG_RK4 or SKG_RK2 (ExactLinStepper, time_stepping.cpp:72-194).
 *   device: CUDA ordinal.
 * The state starts at zero, like init_fields.type = "constant" with value 0.
 * Extents: any even n >= 4, as the reference (grid.cpp:34-44).  Powers of
 * two (ns2d 4..8192, ns3d 8..1024) run the fused kernels; other extents run
 * the generic step (one pass per reference operator, csrc/generic.cu).
 * ns3d grids whose full layout would not fit in free device memory get the
 * compact layout of skg_create_dist(world = 1) (dealiased states only).
 */
int skg_create(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
               double dealias_coef, double nu, int scheme, int device);
int skg_destroy(skg_ctx* ctx);

/*
 * Slab-decomposed context (ns2d, ns3d): the dealiased state is
 * split over the kept ky columns (ns2d) / kept ky lines (ns3d), physical
 * space over x rows; each RK stage runs x-inverse -> all-to-all -> y (and z)
 * passes -> all-to-all -> x-forward, with the transposes as grouped NCCL
 * send/recv (one block per peer) on the context stream.  This process runs
 * partition `rank` of `world` on `device`; nccl_id = the 128 bytes of
 * skg_nccl_unique_id() from rank 0, broadcast by the caller.  nccl_id ==
 * NULL runs ALL `world` partitions in this process on one device with device
 * copies as the exchange (tests).  ns3d with world == 1 is the compact
 * single-GPU layout: state and intermediates hold only the kept (ky, kz)
 * lines (about 2.4x less memory than skg_create; 1024^3 fits one B200).
 * State I/O is the full reference layout on every rank; tendency/energy are
 * not offered; the state must be dealiased (SKG_EUNSUPPORTED otherwise).
 */
/*
 * Peer-memory exchange of the ns2d slab (fused compute + transfer): the
 * x-inverse and y-pass epilogues store directly into the destination
 * partition's receive buffers, so each all-to-all becomes a barrier.
 *   single process (nccl_id == NULL): skg_dist_p2p(ctx, 1);
 *   one process per GPU: every rank calls skg_dist_ipc_handle (256 bytes:
 *   CUDA IPC handles of its receive buffers), the caller all-gathers them in
 *   rank order and every rank calls skg_dist_open_peers(ctx, all) (world x
 *   256 bytes); the NCCL communicator then carries only a 1-double barrier.
 */
int skg_dist_p2p(skg_ctx* ctx, int enable);
/*
 * Copy / NCCL exchange of the ns3d slab: with overlap on (the default) the
 * x-inverse runs one velocity component and the y-forward one field per
 * launch, and each one's all-to-all runs on a second stream while the next
 * one computes (events fork and join the streams; CUDA-graph capturable).
 * Off: one all-to-all per exchange on the context stream.  No effect on the
 * peer-memory exchange (it overlaps by construction) or on ns2d.
 * enable == 2 (pencil contexts with all parts in one process; tests): the kz
 * <-> y transposes run the NCCL route's pack -> block transfer -> unpack
 * instead of direct strided stores, with copies standing in for send / recv.
 * enable == 3 (pencil): the kz -> y transpose as a separate strided-copy
 * kernel instead of the y-inverse kernel's own stores (the default wherever
 * the members' buffers are addressable).
 */
int skg_dist_overlap(skg_ctx* ctx, int enable);

/* Debug aid (no compute-sanitizer on the target pool): with SKG_GUARD=1 in
 * the environment every device allocation of the library is surrounded by
 * 64 KB guard zones holding a byte pattern; this returns how many guard
 * bytes of the live allocations changed (out-of-bounds writes), 0 when the
 * mode is off, -1 on a copy error. */
long skg_guard_violations(void);
int skg_dist_ipc_handle(skg_ctx* ctx, char* out256);
int skg_dist_open_peers(skg_ctx* ctx, const char* all_handles);
int skg_nccl_unique_id(char* out128);
int skg_create_dist(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                    double dealias_coef, double nu, int scheme, int device, int rank, int world,
                    const char* nccl_id);

/*
 * Pencil-decomposed ns3d context (BASELINE configs[4]; the
 * paper's p3dfft-style 2D process grid): py ranks along the
 * kept ky lines / x rows (the slab split above) times pz ranks along the kept
 * kz modes / y rows, global rank = r_y * pz + r_z, two transposes per 3D FFT:
 *   x-inverse on (ky, kz) lines [own ky lines, own kz range]
 *   -> all-to-all inside the py group (ky lines <-> x rows)
 *   -> y-inverse on (x, kz) lines [own x rows, own kz range]
 *   -> all-to-all inside the pz group (kz range <-> y rows)
 *   -> z pass (c2r, u x w, r2c) on (x, y) rows [own x rows, own y rows]
 *   -> the two transposes back around the y-forward -> x-forward + RK.
 * State per rank: [kx][own kept ky lines][own kept kz].  Same kernels as the
 * slab path.  nccl_id == NULL: all py * pz parts live in this process on
 * `device` (copies stand in for the exchanges; tests); otherwise this process
 * runs part `rank` and the transposes are grouped NCCL send/recv -- or, after
 * skg_dist_open_peers, stores straight into the peers' buffers.
 * Needs ny divisible by 2 pz, nx by py, py * pz <= 16, a dealiased state.
 * set_state / get_state / diagnostics take the full reference-layout field
 * on every rank, as for the slab contexts.
 */
int skg_create_pencil(skg_ctx** out, const char* solver, int dims, const int* n, const double* L,
                      double dealias_coef, double nu, int scheme, int device, int rank, int py, int pz,
                      const char* nccl_id);

/* Launch all work on this CUDA stream (cudaStream_t passed as void*);
 * NULL restores the context's own stream. */
int skg_set_stream(skg_ctx* ctx, void* stream);

/* Sizes: spectral modes per variable (S), physical points (P), variables. */
long skg_spect_size(const skg_ctx* ctx);
long skg_phys_size(const skg_ctx* ctx);
int skg_nvars(const skg_ctx* ctx);

/* State I/O, reference layout, nvars * S complex128 -- replaces
 * StateSet::spect()/spect_mut() (state.hpp).  set_state also decides whether
 * the dealiased fast path applies (every masked-out mode exactly zero). */
int skg_set_state(skg_ctx* ctx, const double* spect);
int skg_get_state(skg_ctx* ctx, double* spect_out);
int skg_set_state_device(skg_ctx* ctx, const double* d_spect);
int skg_get_state_device(skg_ctx* ctx, double* d_spect_out);

/* nsteps x Simulation::step_once with fixed dt, forcing off
 * (simulation.cpp:535-555): integrating-factor RK4/RK2 with the nonlinear
 * tendency of the solver, check_finite after every step.  Blocking; returns
 * SKG_EDIVERGENCE with the state frozen after the first non-finite step
 * (see skg_last_divergence). */
/*
 * Adaptive time step (Simulation::compute_dt with fixed_dt = 0,
 * simulation.cpp:463-476): dt = min(dt_max, cfl_coef * min_d dx_d / max|u_d|)
 * per step, clamped to t_end (t_end < 0: no clamp), computed on the device
 * from the max |u_d| of the step's initial state, reduced inside the
 * stage-1 physical pass (no extra transforms).  While enabled, the dt
 * argument of skg_step / skg_step_async / skg_run is ignored; a step whose dt
 * would be <= 0 fails with SKG_ECONFIG ("past t_end") without running.
 * cfl_coef <= 0 returns to the caller's fixed dt.  skg_last_dt = the dt of
 * the last completed step; skg_set_time sets t (restart).
 */
/*
 * Random band forcing (forcing.enable, simulation.cpp:482-548): before each
 * step a unit-magnitude random field in the shell band [k_lo, k_hi]
 * (random_field, grid.cpp:276-306; white noise from the reference's own
 * std::mt19937_64(seed) + std::normal_distribution on the host, the rest on
 * the device) is split so that it injects exactly `rate` (or the unit-energy
 * fallback) and is added to the tendency of every RK stage.  The band must
 * exclude the mean shell and lie inside the dealiasing cut.  Steps with
 * forcing are not graph-replayed (host noise every step).
 * skg_last_injection = Simulation::last_injection of the last step.
 */
/* Solver::sanitize_state on the current state: ns2d dealias + mean 0
 * (solvers.cpp:263-267); ns3d Leray projection + dealias (solvers.cpp:377-381). */
/* Shell spectra of the current state as OutputManager records them
 * (output.cpp:231-257, bin_shells output.cpp:21-39): k = s delta_k, energy
 * density E(k), nonlinear transfer T(k) (from the tendency) and dissipation
 * D(k), s = 0..n_shells-1.  With k == NULL only *n_shells is returned. */
int skg_spectra(skg_ctx* ctx, int cap, double* k, double* E, double* T, double* D, int* n_shells);
int skg_sanitize_state(skg_ctx* ctx);

int skg_set_forcing(skg_ctx* ctx, int enable, double k_lo, double k_hi, double rate, long seed);
double skg_last_injection(const skg_ctx* ctx);

int skg_set_cfl(skg_ctx* ctx, double cfl_coef, double dt_max, double t_end);
double skg_last_dt(const skg_ctx* ctx);
int skg_set_time(skg_ctx* ctx, double t);

int skg_step(skg_ctx* ctx, double dt, long nsteps);
/* Same, enqueued on the context stream without waiting; skg_sync() waits
 * and reports divergence. */
int skg_step_async(skg_ctx* ctx, double dt, long nsteps);
int skg_sync(skg_ctx* ctx);

/* Simulation::run() with n_iters = nsteps (simulation.cpp:565-590): as
 * skg_step, plus the per-step means the reference's OutputManager writes
 * every step (output.cpp:204-214): series[3 i + {0,1,2}] = energy, enstrophy
 * (0 for ns3d) and dissipation rate after step i (simulation.cpp:592-615),
 * reduced on the device (fused into the final RK update on the dealiased
 * path).  series may be NULL.  On divergence the entries after the failing
 * step are 0. */
int skg_run(skg_ctx* ctx, double dt, long nsteps, double* series);

/* Iteration count and time, as Simulation::iteration()/t(). */
long skg_iteration(const skg_ctx* ctx);
double skg_time(const skg_ctx* ctx);

/* == Solver::tendency (solvers.cpp:133-174 ns2d, 299-339 ns3d) on an
 * arbitrary stage state (dealiased output, mean mode 0).  Host buffers,
 * nvars * S complex128 each. */
int skg_tendency(skg_ctx* ctx, const double* in, double* out);
/* Solver::max_velocity_per_axis (solvers.cpp:176-194, 341-357) of the
 * spectral state `spect` (host, reference layout): max |u_d| over the grid,
 * `dims` doubles, from the same fused physical pass as the tendency. */
int skg_max_velocity(skg_ctx* ctx, const double* spect, double* umax);

/* == FftPlan::forward (fft.cpp:92-98: r2c then *= 1/N) and FftPlan::inverse
 * (fft.cpp:100-106: unnormalised c2r, input untouched) on the context grid.
 * u: P doubles; uhat: S complex128. */
int skg_fft_forward(skg_ctx* ctx, const double* u, double* uhat);
int skg_fft_inverse(skg_ctx* ctx, const double* uhat, double* u);

/* Stateless transform operators for any shape (rank 1..3, even extents >= 4,
 * as plan_fft checks in fft.cpp:34-44): FftPlan::forward / inverse. */
int skg_plan_forward(int rank, const int* shape, const double* u, double* uhat, int device);
int skg_plan_inverse(int rank, const int* shape, const double* uhat, double* u, int device);
/* The same transforms in FFTW's conventions, for a GPU-backed FFTW-API shim
 * under the reference's unmodified FftPlan (fft.cpp:67-104):
 * skg_dft_r2c = fftw_execute_dft_r2c (unnormalised, forward sign -1),
 * skg_dft_c2r = fftw_execute_dft_c2r (unnormalised, input left intact). */
int skg_dft_r2c(int rank, const int* shape, const double* in, double* out, int device);
int skg_dft_c2r(int rank, const int* shape, const double* in, double* out, int device);

/* Wavenumbers and dealias mask computed ON THE DEVICE from indices, copied
 * back for a bit-exact comparison with make_grid (grid.cpp:49-100).
 * k_axis: spect_shape[axis] doubles; mask: S bytes or NULL. */
int skg_get_grid(skg_ctx* ctx, int axis, double* k_axis, unsigned char* mask);

/* Divergence report of the last failing step: iteration (as
 * DivergenceError::iteration) and variable index (keys_state_spect order). */
int skg_last_divergence(const skg_ctx* ctx, long* iteration, int* var);

/* Energy / enstrophy of the current state (Simulation::energy/enstrophy,
 * simulation.cpp:592-615), reduced on the device. */
int skg_energy(skg_ctx* ctx, double* energy, double* enstrophy);
/* Simulation::energy, enstrophy and dissipation_rate (simulation.cpp:592-615)
 * of the current state in one device reduction: out3 = {E, Z, eps}. */
int skg_diagnostics(skg_ctx* ctx, double* out3);

/* 1 if the dealiased (pruned) fast path is active for the current state. */
int skg_pruned(const skg_ctx* ctx);

/* Number of kernel launches issued since the context was created. */
long skg_launch_count(const skg_ctx* ctx);

/* Per-kernel-class device timing for the roofline report: when enabled,
 * CUDA events bracket every hot-path launch on the context stream.
 * Classes: 0 x-inverse pass, 1 physical-space pass, 2 x-forward pass + RK,
 * 3 y-inverse pass (3D) and other (decay), 4 all-to-all exchange (bytes =
 * bytes sent to other ranks), 5 y-forward pass (3D).  skg_kernel_stats returns the
 * accumulated device milliseconds, launch count and ALGORITHMIC bytes (the
 * HBM bytes the kernel must move: fields crossing the pass boundary, read or
 * written once) of one class since the last reset. */
int skg_set_timing(skg_ctx* ctx, int enable);
int skg_kernel_stats(skg_ctx* ctx, int cls, double* total_ms, long* launches, double* bytes);
int skg_reset_stats(skg_ctx* ctx);

/* Measurement support (no reference counterpart): the FP64 FMA throughput of
 * `device` measured with a DFMA-only kernel (8 independent chains per thread,
 * every SM filled), in DFMA thread-instructions per second (2 flops each).
 * bench.py's FP64 roofline divides the butterfly kernels' FP64 instruction
 * counts (ncu) by their launch times against this number. */
int skg_fp64_peak(int device, double* dfma_per_s);

#ifdef __cplusplus
}
#endif

#endif
