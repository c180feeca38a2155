// ns2d.cu -- fused RK stage of the 2D vorticity-form solver on sm_100a.
//
// One RK stage = three kernels (SURVEY.md 8(a) GPU mapping, ns2d):
//   k1_xinv : x-inverse c2c on each ky column of the internal CM state
//             ([ky][kx], columns contiguous).  Prologue recomputes the RK
//             stage state from u and the previous k (time_stepping.cpp:
//             128-170) and applies the x-multipliers of the four fields the
//             product needs: psi = w/|k|^2, kx psi, kx w, w
//             (velocity_from_vorticity2d grid.cpp:251-274, gradient_component
//             grid.cpp:124-143).  Writes 4 intermediates [x][ky].
//   k3_phys : y pass per pair of rows: two packed c2r (ux + i dx w,
//             uy + i dy w; the ky factors i*ky are applied here), the product
//             -(ux dx w + uy dy w) (solvers.cpp:160-164), one packed r2c of the
//             two rows, *1/N, ky-dealias (only kept ky stored).
//   k4_xfwd : x-forward c2c per kept ky column, kx-dealias, mean = 0
//             (solvers.cpp:171-172), RK accumulate / final update
//             (time_stepping.cpp:174-193) and the check_finite guard
//             (simulation.cpp:557-563) in the epilogue.
// "pruned": when the state is dealiased every masked-out mode is exactly zero
// and stays zero, so masked columns/rows are never read or
// written.  Otherwise every mode is processed, with identical results.
#include <cstdio>

#include "skg_internal.h"

// Elements per thread of the fast path's x passes below 4096: 8 (twice the
// threads per column; these grids have too few kept columns to fill the GPU
// with 16-element lines -- 1024^2: 0.148 -> 0.118 ms/step, 256^2 0.136 -> 0.064).
// Same for the y pass (1024^2 0.119 -> 0.117, 2048^2 0.448 -> 0.423).
#ifndef SKG_FAST_Y_EM_SMALL
#define SKG_FAST_Y_EM_SMALL 8
#endif
#ifndef SKG_Y8_MINB
#define SKG_Y8_MINB 2
#endif
#ifndef SKG_FAST_Y_EM
#define SKG_FAST_Y_EM 16
#endif
#ifndef SKG_FAST_X_EM_SMALL
#define SKG_FAST_X_EM_SMALL 8
#endif
#ifndef SKG_FAST_X_EM
#define SKG_FAST_X_EM 16
#endif
// 4 elements per thread (four times the threads per line) for the smallest
// grids, 128 registers: x passes up to 512 (ms/step 256^2 0.0599 -> 0.0455,
// 512^2 0.0589 -> 0.0525; 1024^2 slower, 0.1175 -> 0.1334), the y pass up to
// 256 (256^2 -> 0.0432; 512^2 slower).  64 registers spill (slower).
// Paired x-forward (k4p_xfwd) for NX in [SKG_PAIRED_X_MIN, SKG_PAIRED_X_MAX],
// SKG_PAIRED_REGS registers per thread (80: three 256-thread CTAs per SM, no
// spills).  Measured (ms/step): 1024^2 0.1173 -> 0.1119, 512^2 0.0524 ->
// 0.0483; 2048^2 slower (0.420 -> 0.442: 683 columns, more than one wave);
// 128 registers 0.1230 at 1024^2 (two CTAs per SM: two waves).
#ifndef SKG_PAIRED_X_MIN
#define SKG_PAIRED_X_MIN 512
#endif
#ifndef SKG_PAIRED_X_MAX
#define SKG_PAIRED_X_MAX 1024
#endif
#ifndef SKG_PAIRED_REGS
#define SKG_PAIRED_REGS 80
#endif

#ifndef SKG_EM4_REGS
#define SKG_EM4_REGS 128
#endif
#ifndef SKG_X_EM4_MAX
#define SKG_X_EM4_MAX 512
#endif
#ifndef SKG_Y_EM4_MAX
#define SKG_Y_EM4_MAX 256
#endif

namespace skg {

namespace {

// Row-pair interleaved layout of the x-space intermediates and tendency rows:
// element (x, ky) of a [nx][ld] field lives at ((x/2) ld + ky) 2 + (x mod 2).
// The y pass (k3_phys) works on row pairs, so each pair is one contiguous
// block; the strided x passes touch 32-byte chunks (two adjacent x of one
// ky column) instead of 16-byte ones.
__device__ __forceinline__ size_t pidx(int x, int ky, int ld) {
    return ((size_t)(x >> 1) * ld + ky) * 2 + (x & 1);
}

// Column-pair interleaved layout of the fast path's product spectra A, B:
// element (x, ky) at ((ky/2) nx + x) 2 + (ky mod 2).  The y pass writes it
// (strided stores, merged in L2), the x-forward pass reads each ky column
// as one contiguous stream (strided loads would defeat DRAM row locality).
__device__ __forceinline__ size_t cpidx(int x, int ky, int nx) {
    return ((size_t)(ky >> 1) * nx + x) * 2 + (ky & 1);
}

// Rows interleaved per ky in the fast path's x-inverse outputs: the x-inverse
// pass stores RG consecutive x of one column as one 16*RG-byte chunk.
constexpr int RG = 4;

// x-inverse output (x, local column kyl) in the send block of the row's owner
// q: rows(q) x own columns, row-quad interleaved ((xl/4) ncols + kyl) 4 + xl%4.
__device__ __forceinline__ size_t sidx_send(const Ns2dArgs& a, int x, int kyl) {
    const int q = x >> a.lg_nrl, xl = x & (a.nrl - 1);
    return (size_t)q * a.nrl * a.ncols + ((size_t)(xl / RG) * a.ncols + kyl) * RG + (xl % RG);
}

// Where the x-inverse output m of (x, local column kyl) goes: this
// partition's send block for the row's owner, or (p2p) directly the owner's
// receive block (offset nrl * c0, same layout).
__device__ __forceinline__ cd* xinv_dst(const Ns2dArgs& a, int m, int x, int kyl) {
    if (!a.p2p) return a.sI[m] + sidx_send(a, x, kyl);
    const int q = x >> a.lg_nrl, xl = x & (a.nrl - 1);
    return a.peer_rI[q][m] + (size_t)a.nrl * a.c0 + ((size_t)(xl / RG) * a.ncols + kyl) * RG + (xl % RG);
}

// Where the y-pass output f of (local row x, kept column k) goes: the send
// buffer in pair order, or (p2p) the column owner's receive block from this
// partition (offset r * 2 npairs(q) nrl, layout ((k-c_q)/2 nrl + x) 2 + k%2).
__device__ __forceinline__ cd* ypass_dst(const Ns2dArgs& a, int f, int x, int k) {
    if (!a.p2p) return a.sA[f] + cpidx(x, k, a.nrl);
    const int PP = (a.ky_in + 1) >> 1;
    const int q = (((k >> 1) + 1) * a.G - 1) / PP;
    const int cs = 2 * (q * PP / a.G);
    const int nc = (q == a.G - 1 ? a.ky_in : 2 * ((q + 1) * PP / a.G)) - cs;
    const size_t npq = (size_t)(nc + 1) >> 1;
    return a.peer_rA[q][f] + (size_t)a.r * 2 * npq * a.nrl + ((size_t)((k - cs) >> 1) * a.nrl + x) * 2 +
           (k & 1);
}

__device__ __forceinline__ cd* pick(const Ns2dArgs& a, int m) {
    return m == 0 ? a.I[0] : m == 1 ? a.I[1] : m == 2 ? a.I[2] : a.I[3];
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ bool finite2(cd v) { return isfinite(v.x) && isfinite(v.y); }

// RK stage state from already-loaded u and previous k (time_stepping.cpp:128-170).
__device__ __forceinline__ cd stage_combine(const Ns2dArgs& a, int stage, int ky, int i, cd u, cd k) {
    if (stage <= 1) return u;
    if (a.has_sigma) {
        const double e1 = a.e1x[i] * a.e1y[ky];
        if (stage == 2) return scale(add(u, scale(k, hdt_of(a))), e1);
        if (stage == 3) return add(scale(u, e1), scale(k, hdt_of(a)));
        const double e2 = a.e2x[i] * a.e2y[ky];
        return add(scale(u, e2), scale(k, dt_of(a) * e1));
    }
    return add(u, scale(k, stage == 4 ? dt_of(a) : hdt_of(a)));
}

// PZ: the state is dealiased and the kept |kx| <= kcx < 6T, so the elements
// e in [6, 10) of every thread (kx in [6T, 10T)) are exactly zero: they are
// neither loaded nor stored, and the stage-state slots shrink from 16 to 12.
// EM = 8 elements per thread: twice the threads per line, a quarter fewer
// registers, one more shared-memory exchange; the zero band is then e in [3, 5).
// CTW: target CTA width (threads); narrow CTAs (one line each, CTW <= T)
// spread small grids over all SMs.
template <int N, int EM, int CTW = 256>
struct XCfg {
    using F = BFFT<N, false, EM>;
    static constexpr int T = F::T;
    static constexpr int LPC = T >= CTW ? 1 : CTW / T;
    static constexpr int CT = T * LPC;
    // resident CTAs the register budget is sized for: <= 128 registers per
    // thread (512-thread lines of 8192: one CTA, its shared memory is ~224 KB)
    static constexpr int MINB = EM == 4 ? (CT >= 65536 / SKG_EM4_REGS ? 1 : 65536 / SKG_EM4_REGS / CT > 32 ? 32 : 65536 / SKG_EM4_REGS / CT)
                               : CT >= 512 ? 1 : CT >= 256 ? 2 : (512 / CT > 32 ? 32 : 512 / CT);
    // zero band of the dealiased kx (none with 4-element lines)
    static constexpr int ZLO = EM == 16 ? 6 : EM == 8 ? 3 : F::E / 2, ZHI = EM == 16 ? 10 : EM == 8 ? 5 : F::E / 2;
};
// fused x-forward: shared memory per line (exchange + kept slots), cd units
template <int N, int EM, int CTW>
constexpr int xf_slot() {
    using C = XCfg<N, EM, CTW>;
    return C::F::SMEM + (C::F::E - (C::ZHI - C::ZLO)) * C::T;
}

template <int NX, bool PZ, int NM, int EM = 16, int CTW = 256>
__global__ void __launch_bounds__(XCfg<NX, EM, CTW>::CT,
                                  (PZ || EM == 8 || XCfg<NX, EM, CTW>::MINB < 2) ? XCfg<NX, EM, CTW>::MINB
                                                                       : XCfg<NX, EM, CTW>::MINB / 2)
    k1_xinv(Ns2dArgs a, int stage) {
    using F = BFFT<NX, false, EM>;
    constexpr int T = F::T, E = F::E;
    constexpr int LPC = XCfg<NX, EM, CTW>::LPC;
    constexpr int ZLO = PZ ? XCfg<NX, EM>::ZLO : E, ZHI = PZ ? XCfg<NX, EM>::ZHI : E;
    constexpr int NS = E - (ZHI - ZLO);  // stage-state slots per thread
    extern __shared__ cd smem[];
    const int l = threadIdx.x / T, t = threadIdx.x % T;
    // NM == 2 (fast path): local column kyl of this partition; NM == 4: G = 1
    const int kyl = blockIdx.x * LPC + l;
    const int ky = (NM == 2 ? a.c0 : 0) + kyl;
    const bool active = kyl < (NM == 2 ? a.ncols : a.ky_in);
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    // step counter: here on the general path, in the stage-1 y pass on the
    // fast path (whose x-inverse usually runs fused into the previous step)
    if (NM == 4 && stage == 1 && blockIdx.x == 0 && threadIdx.x == 0 && a.lead)
        atomicAdd(&a.flags->steps, 1);
    cd* sm = smem + l * (F::SMEM + NS * T);
    cd* sv = sm + F::SMEM;  // thread-private slots sv[slot * T + t]
    const double kyv = a.ky_scale * (double)ky;
    const typename F::Bases wb = F::bases(t, a.twx);
    // RK stage state w, computed once per column (time_stepping.cpp:128-170),
    // kept as psi = w/|k|^2 (grid.cpp:262-270): the four x-multipliers are then
    // psi, kx psi, kx |k|^2 psi, |k|^2 psi -- no division inside the loop.
    // (|k|^2 psi differs from w in the last bit and is 0 at k = 0, where w
    // only feeds columns multiplied by kx = 0 or ky = 0.)
    // u and k_{j-1} of the column stream into shared memory with cp.async
    // (u into the thread's slots, k into the still idle exchange buffer,
    // same thread-private layout), so all loads are in flight at once.
    const cd* kprev = stage == 2 ? a.k1 : stage == 3 ? a.k2 : a.k3;
    cd* kv = sm;  // exchange buffer as k staging: kv[slot * T + t]
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZLO && e < ZHI) continue;
        const int slot = e < ZLO ? e : e - (ZHI - ZLO);
        const int i = t + T * e;
        const bool keep = active && (!a.pruned || abs(signed_index(i, NX)) <= a.kcx);
        if (keep) {
            const size_t idx = (size_t)kyl * NX + i;
            cp_async16(&sv[slot * T + t], a.u + idx);
            if (stage > 1) cp_async16(&kv[slot * T + t], kprev + idx);
        }
    }
    cp_async_commit();
    cp_async_wait_all();
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZLO && e < ZHI) continue;
        const int slot = e < ZLO ? e : e - (ZHI - ZLO);
        const int i = t + T * e;
        const int si = signed_index(i, NX);
        const bool keep = active && (!a.pruned || abs(si) <= a.kcx);
        cd psi = zero();
        if (keep) {
            const cd s = stage_combine(a, stage, ky, i, sv[slot * T + t],
                                       stage > 1 ? kv[slot * T + t] : zero());
            const double kxv = a.kx_scale * (double)si;
            const double ksq = kxv * kxv + kyv * kyv;
            if (ksq != 0.0) {  // one reciprocal instead of two IEEE divisions
                const double r = __drcp_rn(ksq);
                psi = mk(s.x * r, s.y * r);
            }
        }
        sv[slot * T + t] = psi;
    }
    __syncthreads();  // k staging lived in the exchange buffer
#pragma unroll 1
    for (int m = 0; m < NM; ++m) {
        cd v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= ZLO && e < ZHI) {
                v[e] = zero();
                continue;
            }
            const int slot = e < ZLO ? e : e - (ZHI - ZLO);
            const cd psi = sv[slot * T + t];
            const double kxv = a.kx_scale * (double)signed_index(t + T * e, NX);
            const double ksq = kxv * kxv + kyv * kyv;
            double f = m == 0 ? 1.0 : m == 1 ? kxv : m == 2 ? kxv * ksq : ksq;
            v[e] = scale(psi, f);
        }
        F::template run<+1>(v, sm, t, wb);
        if (active) {
            if constexpr (NM == 2) {
#pragma unroll
                for (int e = 0; e < E; ++e) *xinv_dst(a, m, t + T * e, kyl) = v[e];
            } else {
                cd* out = pick(a, m);
#pragma unroll
                for (int e = 0; e < E; ++e) out[pidx(t + T * e, ky, a.ld_i)] = v[e];
            }
        }
    }
    if (NM == 2 && a.p2p) __threadfence_system();  // peer stores visible before the barrier
}

// y pass on a row pair (xa, xa+1).  Four inverse FFTs k = 0..3 over
// (row, field pair) = (xa, q0), (xa, q1), (xa+1, q0), (xa+1, q1), where
// q0 = (X[psi], X[kx w]) -> ux + i dx w and q1 = (X[kx psi], X[w]) -> uy + i dy w;
// the input rows of FFT k+1 stream into a shared-memory stage (cp.async)
// while FFT k runs.  Shared memory per group: split exchange (N doubles),
// the finished row-a product (N doubles), stage (2 ld_i complex).
template <int NY, int EM, bool CFL>
__global__ void __launch_bounds__(BFFT<NY, true, EM>::T >= 256 ? BFFT<NY, true, EM>::T : 256,
                                  EM == 8 ? 65536 / 64 / (BFFT<NY, true, EM>::T >= 256 ? BFFT<NY, true, EM>::T : 256) : 2)
    k3_phys(Ns2dArgs a) {
    using F = BFFT<NY, true, EM>;
    constexpr int T = F::T, E = F::E;
    constexpr int G = T >= 256 ? 1 : 256 / T;
    extern __shared__ cd smem[];
    const int ld = a.ld_i;
    const int slot = F::SMEM + NY / 2 + 2 * ld;
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const int bar = G > 1 ? g + 1 : 0;  // the groups' own barriers (line_sync)
    const int xa = 2 * (blockIdx.x * G + g);
    const bool active = xa < a.nx;
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    cd* sm = smem + g * slot;
    double* prow = reinterpret_cast<double*>(sm + F::SMEM);
    cd* st = sm + F::SMEM + NY / 2;
    const typename F::Bases wb = F::bases(t, a.twy);

    auto issue = [&](int k) {
        if (!active) return;
        const int x = xa + (k >> 1), q = k & 1;
        const cd* P = pick(a, q ? 1 : 0);
        const cd* Q = pick(a, q ? 3 : 2);
        for (int i = t; i < a.ky_in; i += T) {
            cp_async16(&st[i], P + pidx(x, i, ld));
            cp_async16(&st[ld + i], Q + pidx(x, i, ld));
        }
    };
    issue(0);
    cp_async_commit();
    constexpr bool cfl = CFL;  // max |u_d| of the step's initial state (adaptive dt)
    double mx = 0.0, my = 0.0;
    double acc[E];
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
        const int q = k & 1;
        cp_async_wait_all();
        line_sync<T>(bar);
        cd v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int idx = t + T * e;
            const bool mirror = idx > NY / 2;
            const int ki = mirror ? NY - idx : idx;
            cd ah = zero(), bh = zero();
            if (active && ki < a.ky_in) {
                const double kyv = a.ky_scale * (double)ki;
                const cd p = st[ki];
                const cd qq = st[ld + ki];
                if (q == 0) {
                    ah = mk(-kyv * p.y, kyv * p.x);   // ux: i ky X[psi]
                    bh = muli(qq);                    // dx w: i X[kx w]
                } else {
                    ah = mulmi(p);                    // uy: -i X[kx psi]
                    bh = mk(-kyv * qq.y, kyv * qq.x); // dy w: i ky X[w]
                }
                if (ki == 0 || 2 * ki == NY) {  // c2r ignores these imaginary parts
                    ah.y = 0.0;
                    bh.y = 0.0;
                }
            }
            // packed spectrum of (a + i b) over the full ky range
            v[e] = mirror ? mk(ah.x + bh.y, bh.x - ah.y) : mk(ah.x - bh.y, ah.y + bh.x);
        }
        line_sync<T>(bar);  // stage consumed
        if (k < 3) issue(k + 1);
        cp_async_commit();
        F::template run<+1>(v, sm, t, wb, 0, bar);
        if constexpr (cfl) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (q == 0) mx = fmax(mx, fabs(v[e].x));
                else my = fmax(my, fabs(v[e].x));
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double p = v[e].x * v[e].y;  // ux dx w | uy dy w
            if (q == 0) {
                acc[e] = p;
            } else {
                const double fin = -(acc[e] + p);  // solvers.cpp:162-163
                if (k == 1) prow[t + T * e] = fin;
                else acc[e] = fin;
            }
        }
    }
    if constexpr (cfl) umax_accumulate(a.dyn, 2, mx, my, 0.0);
    // forward r2c of both rows packed: z = prod_a + i prod_b
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = mk(prow[t + T * e], acc[e]);
    F::template run<-1>(v, sm, t, wb, 0, bar);
    // exchange + prow form one contiguous N-complex buffer now
    using FF = BFFT<NY, false, EM>;
#pragma unroll
    for (int e = 0; e < E; ++e) sm[FF::pad(t + T * e)] = v[e];
    line_sync<T>(bar);
    if (active) {
        const double h = 0.5 * a.inv_n;
        cd* rp = a.nl + (size_t)(xa >> 1) * a.ld_o * 2;  // row pair block
        for (int k = t; k < a.ld_o; k += T) {
            cd zk = sm[FF::pad(k)];
            cd zm = sm[FF::pad((NY - k) & (NY - 1))];
            rp[2 * k] = mk((zk.x + zm.x) * h, (zk.y - zm.y) * h);
            rp[2 * k + 1] = mk((zk.y + zm.y) * h, (zm.x - zk.x) * h);
        }
    }
}

template <int NX>
__global__ void __launch_bounds__(BFFT<NX>::T > 256 ? BFFT<NX>::T : 256, BFFT<NX>::T > 256 ? 1 : 2)
    k4_xfwd(Ns2dArgs a, int stage) {
    using F = BFFT<NX>;
    constexpr int T = F::T, E = F::E;
    constexpr int LPC = T >= 256 ? 1 : 256 / T;
    extern __shared__ cd smem[];
    const int l = threadIdx.x / T, t = threadIdx.x % T;
    const int ky = blockIdx.x * LPC + l;
    const bool active = ky < a.ld_o;
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    cd* sm = smem + l * F::SMEM;
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e)
        v[e] = active ? a.nl[pidx(t + T * e, ky, a.ld_o)] : zero();
    F::template run<-1>(v, sm, t, a.twx);
    if (!active) return;
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    cd* kout = stage == 1 ? a.k1 : stage == 2 ? a.k2 : a.k3;
    bool bad = false;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = t + T * e;
        const int si = signed_index(i, NX);
        bool keep = abs(si) <= a.kcx;
        if (i == 0 && ky == 0) keep = false;  // mean mode of the tendency is 0
        if (!keep && a.pruned) continue;
        const size_t idx = (size_t)ky * NX + i;
        cd kv = keep ? v[e] : zero();
        if (a.force && keep) kv = add(kv, a.force[idx]);  // forcing addend (simulation.cpp:544-547)
        if (!final) {
            kout[idx] = kv;
        } else {
            cd u = a.u[idx];
            cd un;
            if (a.has_sigma) {
                const double e1 = a.e1x[i] * a.e1y[ky];
                const double e2 = a.e2x[i] * a.e2y[ky];
                if (a.rk2) {
                    un = add(scale(u, e2), scale(kv, dt_of(a) * e1));
                } else {
                    cd k1 = a.k1[idx], k2 = a.k2[idx], k3 = a.k3[idx];
                    cd sum = add(add(scale(k1, e2), scale(add(k2, k3), 2.0 * e1)), kv);
                    un = add(scale(u, e2), scale(sum, sdt_of(a)));
                }
            } else {
                cd delta;
                if (a.rk2) {
                    delta = scale(kv, dt_of(a));
                } else {
                    cd k1 = a.k1[idx], k2 = a.k2[idx], k3 = a.k3[idx];
                    delta = scale(add(add(k1, scale(add(k2, k3), 2.0)), kv), sdt_of(a));
                }
                un = (delta.x != 0.0 || delta.y != 0.0) ? add(u, delta) : u;
            }
            a.u[idx] = un;
            bad |= !finite2(un);
        }
    }
    if (bad) {
        atomicMin(&a.flags->div_var, 0);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
}

// Unpruned final update of the ky columns above the cut: tendency is zero
// there, so u <- E2 u (time_stepping.cpp:186-192 with k = 0).
__global__ void k4_decay(Ns2dArgs a) {
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    const size_t cols = (size_t)(a.nh - (a.kcy + 1));
    const size_t total = cols * a.nx;
    bool bad = false;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int ky = a.kcy + 1 + (int)(q / a.nx);
        const int i = (int)(q % a.nx);
        const size_t idx = (size_t)ky * a.nx + i;
        cd u = a.u[idx];
        if (a.has_sigma) {
            const double e2 = a.e2x[i] * a.e2y[ky];
            u = scale(u, e2);
            a.u[idx] = u;
        }
        bad |= !finite2(u);
    }
    if (bad) {
        atomicMin(&a.flags->div_var, 0);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
}

// =====================================================================
// Fast path for dealiased states (Basdevant form, 4 real transforms).
// For fields band-limited by the 2/3 rule (3 kc < n on both axes) the grid
// products below are alias-free on every kept mode, so
//   -FT[u . grad w] = kx ky FT(v^2 - u^2) + (kx^2 - ky^2) FT(u v)
// equals the reference's -FT[ux dx w + uy dy w] (solvers.cpp:133-174) up to
// rounding, with u = i ky psi, v = -i kx psi.  Per RK stage: x-inverse of
// psi and kx psi (2 FFTs/column), one c2r + one r2c per row (2 FFTs/row),
// x-forward of the two product spectra (2 FFTs/column): 20% fewer FFTs and
// intermediate bytes than the 4-inverse + 1-forward form, which stays in use
// for states that are not dealiased.

// y pass, one row per group iteration, persistent over rows; the next row's
// two input lines stream into shared memory (cp.async) during the FFTs.
// Resident CTAs per SM of the fast y pass (256-thread CTAs): 2 with
// 16-element rows (128 registers); SKG_Y8_MINB with 8-element rows -- 3 or 4
// (85 / 64 registers, one wave of rows at 1024^2) spill and measured slower
// (1024^2: 0.147 / 0.140 vs 0.117 ms/step), so 2.
template <int NY, int EM>
constexpr int y_minb() {
    return BFFT<NY, false, EM>::T > 256 ? 1 : EM == 16 ? 2 : EM == 4 ? 256 / SKG_EM4_REGS : SKG_Y8_MINB;
}

template <int NY, bool CFL, int EM = 16>
__global__ void __launch_bounds__(BFFT<NY, false, EM>::T > 256 ? BFFT<NY, false, EM>::T : 256,
                                  y_minb<NY, EM>())
    k3b_phys(Ns2dArgs a) {
    using F = BFFT<NY, false, EM>;
    constexpr int T = F::T, E = F::E;
    constexpr int G = T >= 256 ? 1 : 256 / T;
    // per-thread zero band: row elements e in [6, 10) (E = 16; [3, 5) for
    // E = 8), |ky| in [3N/8, N/2], are masked on input and not needed on
    // output (fast_ok: ky_in, ld_o <= 3N/8)
    constexpr int ZLO = E == 16 ? 6 : E == 8 ? 3 : E / 2, ZHI = E == 16 ? 10 : E == 8 ? 5 : E / 2;
    extern __shared__ cd smem[];
    const int ld = a.ld_i;
    const int slot = F::SMEM + 2 * ld;
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const int bar = G > 1 ? g + 1 : 0;  // the groups' own barriers (line_sync)
    const typename F::Bases wb = F::bases(t, a.twy);  // constant table: before the wait
    pdl_wait();
    const int dflag = *reinterpret_cast<const volatile int*>(&a.flags->diverged);
    cd* sm = smem + g * slot;
    cd* st = sm + F::SMEM;
    const int stride = gridDim.x * G;
    const cd* P = a.rI[0];  // X[psi]
    const cd* Q = a.rI[1];  // X[kx psi]
    // outputs (ypass_dst): FT_y(v^2 - u^2) / N and FT_y(u v) / N
    // x runs over this partition's local rows; input column ky comes from
    // the receive block of its owner r' (layout of r')
    auto issue = [&](int x) {
        if (x >= a.nrl) return;
        // ky_in <= ZLO T (fast_ok): a fixed trip count, unrolled, so the
        // copies of one row are issued back to back
#pragma unroll
        for (int j = 0; j < ZLO; ++j) {
            const int i = t + T * j;
            if (i >= a.ky_in) break;
            size_t q;
            if (a.G == 1) {
                q = ((size_t)(x / RG) * a.ky_in + i) * RG + (x % RG);
            } else {
                // owner of column i under cstart[q] = 2 floor(q PP / G), PP kept
                // column pairs (skgpu.cu create_impl), computed instead of loaded
                const int PP = (a.ky_in + 1) >> 1;
                const int ro = (((i >> 1) + 1) * a.G - 1) / PP;
                const int cs = 2 * (ro * PP / a.G);
                const int nc = (ro == a.G - 1 ? a.ky_in : 2 * ((ro + 1) * PP / a.G)) - cs;
                q = (size_t)a.nrl * cs + ((size_t)(x / RG) * nc + (i - cs)) * RG + (x % RG);
            }
            cp_async16(&st[i], P + q);
            cp_async16(&st[ld + i], Q + q);
        }
    };
    int x = blockIdx.x * G + g;
    issue(x);
    cp_async_commit();
    // divergence flag, one value per CTA (cta_diverged), checked with the
    // first row's loads in flight
    if (__syncthreads_or(dflag) != 0) {
        cp_async_wait_all();
        return;
    }
    if (a.ystage == 1 && blockIdx.x == 0 && threadIdx.x == 0 && a.lead) atomicAdd(&a.flags->steps, 1);
    const double h = 0.5 * a.inv_n;
    constexpr bool cfl = CFL;  // max |u_d| of the step's initial state (adaptive dt)
    double mx = 0.0, my = 0.0;
    // every group runs the same number of iterations (barriers inside)
    const int iters = (a.nrl + stride - 1) / stride;
#pragma unroll 1
    for (int it = 0; it < iters; ++it, x += stride) {
        const bool active = x < a.nrl;
        cp_async_wait_all();
        line_sync<T>(bar);
        cd v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= ZLO && e < ZHI) {  // |ky| >= 6T > kcy: zero (fast_ok)
                v[e] = zero();
                continue;
            }
            const int idx = t + T * e;
            const bool mirror = idx > NY / 2;
            const int ki = mirror ? NY - idx : idx;
            cd ah = zero(), bh = zero();
            if (active && ki < a.ky_in) {
                const double kyv = a.ky_scale * (double)ki;
                const cd p = st[ki];
                const cd q = st[ld + ki];
                ah = mk(-kyv * p.y, kyv * p.x);  // u: i ky X[psi]
                bh = mulmi(q);                   // v: -i X[kx psi]
                if (ki == 0 || 2 * ki == NY) {
                    ah.y = 0.0;
                    bh.y = 0.0;
                }
            }
            v[e] = mirror ? mk(ah.x + bh.y, bh.x - ah.y) : mk(ah.x - bh.y, ah.y + bh.x);
        }
        line_sync<T>(bar);  // stage consumed
        issue(x + stride);
        cp_async_commit();
        F::template run<+1>(v, sm, t, wb, 0, bar);  // u + i v on the row
        if constexpr (cfl) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                mx = fmax(mx, fabs(v[e].x));
                my = fmax(my, fabs(v[e].y));
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double u = v[e].x, w = v[e].y;
            v[e] = mk(w * w - u * u, u * w);  // (v^2 - u^2) + i (u v)
        }
        F::template run<-1>(v, sm, t, wb, 0, bar);
        // Hermitian split of the packed spectrum Z = FT(a + i b): output
        // k = t + T e (e < ZLO) pairs with NY - k = (T - t) + T (E - 1 - e),
        // element E - 1 - e of thread T - t (thread 0: its own element E - e),
        // so each thread publishes its elements [ZHI, E) and reads its
        // partner's -- one shared-memory round trip of E - ZHI values.
        static_assert(ZLO + ZHI == E, "zero band symmetric about N/2");
#pragma unroll
        for (int e = ZHI; e < E; ++e) sm[(e - ZHI) * T + t] = v[e];
        line_sync<T>(bar);
        if (active) {
            const int tp = t == 0 ? 0 : T - t;
#pragma unroll
            for (int e = 0; e < ZLO; ++e) {
                const int k = t + T * e;
                if (k >= a.ld_o) break;
                const cd zk = v[e];
                const cd zm = t == 0 ? (e == 0 ? v[0] : v[E - e]) : sm[(E - 1 - e - ZHI) * T + tp];
                *ypass_dst(a, 0, x, k) = mk((zk.x + zm.x) * h, (zk.y - zm.y) * h);
                *ypass_dst(a, 1, x, k) = mk((zk.y + zm.y) * h, (zm.x - zk.x) * h);
            }
        }
    }
    if constexpr (cfl) umax_accumulate(a.dyn, 2, mx, my, 0.0);
    if (a.p2p) __threadfence_system();
}

// Operands of one kept mode of the x-forward epilogue, loaded for a chunk
// of modes before any of them is computed (the k_j / u stores of a mode
// would otherwise keep the compiler from hoisting the next mode's loads).
struct XfOps {
    cd u, k1, k2, k3;
    double e1, e2;  // integrating factors of the mode (has_sigma)
};

__device__ __forceinline__ XfOps xf_load(const Ns2dArgs& a, bool final, bool fuse, int stage, double e1y,
                                         double e2y, int i, size_t idx) {
    XfOps o;
    o.u = (final || fuse) ? a.u[idx] : zero();
    if (final && !a.rk2) {
        o.k1 = a.k1[idx];
        o.k2 = a.k2[idx];
        o.k3 = a.k3[idx];
    }
    o.e1 = o.e2 = 1.0;
    if (a.has_sigma && (final || fuse)) {
        o.e1 = a.e1x[i] * e1y;
        if (final || stage + 1 == 4) o.e2 = a.e2x[i] * e2y;
    }
    return o;
}

// One kept mode (kx index i, local column kyl) of the x-forward epilogue:
// tendency kv (+ forcing) -> k_j, or the final RK update of u with the
// non-finite flag and the per-step diagnostics; returns the next stage state
// (fused kernels: stage_combine, or the new u = stage 1 of the next step).
__device__ __forceinline__ cd xf_point(const Ns2dArgs& a, int stage, bool final, bool fuse, double kyv,
                                       double kxv, double pw, size_t idx, cd kv, const XfOps& o,
                                       bool& bad, double& sE, double& sZ, double& sD) {
    if (a.force) kv = add(kv, a.force[idx]);  // forcing addend (simulation.cpp:544-547)
    if (!final) {
        cd* kout = stage == 1 ? a.k1 : stage == 2 ? a.k2 : a.k3;
        kout[idx] = kv;
        if (!fuse) return zero();
        // stage_combine of stage + 1 (time_stepping.cpp:128-170)
        const int ns = stage + 1;
        if (a.has_sigma) {
            if (ns == 2) return scale(add(o.u, scale(kv, hdt_of(a))), o.e1);
            if (ns == 3) return add(scale(o.u, o.e1), scale(kv, hdt_of(a)));
            return add(scale(o.u, o.e2), scale(kv, dt_of(a) * o.e1));
        }
        return add(o.u, scale(kv, ns == 4 ? dt_of(a) : hdt_of(a)));
    }
    const cd u = o.u;
    cd un;
    if (a.has_sigma) {
        if (a.rk2) {
            un = add(scale(u, o.e2), scale(kv, dt_of(a) * o.e1));
        } else {
            const cd sum = add(add(scale(o.k1, o.e2), scale(add(o.k2, o.k3), 2.0 * o.e1)), kv);
            un = add(scale(u, o.e2), scale(sum, sdt_of(a)));
        }
    } else {
        cd delta;
        if (a.rk2) {
            delta = scale(kv, dt_of(a));
        } else {
            delta = scale(add(add(o.k1, scale(add(o.k2, o.k3), 2.0)), kv), sdt_of(a));
        }
        un = (delta.x != 0.0 || delta.y != 0.0) ? add(u, delta) : u;
    }
    a.u[idx] = un;
    bad |= !finite2(un);
    if (a.diag) {
        const double ksq = kxv * kxv + kyv * kyv;
        const double n2 = un.x * un.x + un.y * un.y;
        sZ += 0.5 * pw * n2;
        if (ksq > 0.0) {
            const double en = 0.5 * pw * n2 * __drcp_rn(ksq);
            sE += en;
            if (a.has_sigma) sD += 2.0 * a.nu * ksq * en;
        }
    }
    return un;  // stage 1 of the next step
}

// x-forward of the two product spectra per kept ky column, combination
// kx ky A + (kx^2 - ky^2) B, dealias + mean 0 + RK epilogue (as k4_xfwd).
// FUSE (next != 0): the same CTA then runs the NEXT stage's x-inverse of its
// column (k1_xinv's body): the next stage state is formed in registers from
// the tendency just computed (stage_combine, or the new u after the final
// update = stage 1 of the next step), so k_j is not re-read, u is read once,
// and one launch per stage disappears.
template <int NX, int EM = 16, int CTW = 256, bool FUSE = false>
__global__ void __launch_bounds__(XCfg<NX, EM, CTW>::CT, XCfg<NX, EM, CTW>::MINB)
    k4b_xfwd(Ns2dArgs a, int stage, int next) {
    using F = BFFT<NX, false, EM>;
    constexpr int T = F::T, E = F::E;
    constexpr int LPC = XCfg<NX, EM, CTW>::LPC;
    constexpr int ZLO = XCfg<NX, EM>::ZLO, ZHI = XCfg<NX, EM>::ZHI;
    extern __shared__ cd smem[];
    const int l = threadIdx.x / T, t = threadIdx.x % T;
    const int kyl = blockIdx.x * LPC + l;  // local column
    const int ky = a.c0 + kyl;
    const bool active = kyl < a.ncols;
    const typename F::Bases wb = F::bases(t, a.twx);  // constant table: before the wait
    cd* sm = smem + l * xf_slot<NX, EM, CTW>();
    cd* sv = sm + F::SMEM;
    const double kyv = a.ky_scale * (double)ky;
    const size_t blk = (size_t)2 * ((a.ncols + 1) >> 1) * a.nrl;  // receive block per source
    auto ridx = [&](int x) {
        const int ro = x >> a.lg_nrl, xl = x & (a.nrl - 1);
        return ro * blk + ((size_t)(kyl >> 1) * a.nrl + xl) * 2 + (kyl & 1);
    };
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    const bool fuse = FUSE && next;
    pdl_wait();
    const int dflag = *reinterpret_cast<const volatile int*>(&a.flags->diverged);
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e)
        v[e] = active ? a.rA[0][ridx(t + T * e)] : zero();
    // divergence flag, one value per CTA (cta_diverged), checked after the
    // input loads are in flight
    if (__syncthreads_or(dflag) != 0) return;
    F::template run<-1>(v, sm, t, wb);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZLO && e < ZHI) continue;
        const int slot = e < ZLO ? e : e - (ZHI - ZLO);
        const double kxv = a.kx_scale * (double)signed_index(t + T * e, NX);
        sv[slot * T + t] = scale(v[e], kxv * kyv);
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
        v[e] = active ? a.rA[1][ridx(t + T * e)] : zero();
    F::template run<-1>(v, sm, t, wb);
    bool bad = false;
    // per-step E, Z, eps of the new state (Simulation::energy / enstrophy /
    // dissipation_rate, simulation.cpp:592-615; ns2d mode_energy solvers.cpp:211-218)
    double sE = 0.0, sZ = 0.0, sD = 0.0;
    const double pw = (ky == 0 || ky == a.nh - 1) ? 1.0 : 2.0;
    if (final && a.diag && active && ky == 0 && t == 0) {
        const cd u0 = a.u[(size_t)kyl * NX];  // mean mode: untouched, enstrophy only
        sZ += 0.5 * pw * (u0.x * u0.x + u0.y * u0.y);
    }
    const double e1y = a.has_sigma ? a.e1y[ky] : 1.0, e2y = a.has_sigma ? a.e2y[ky] : 1.0;
    // chunks of CH kept modes: the chunk's operand loads, then its arithmetic
    // (CH = 2 spills at 4096 and measured 262 vs 212 us)
    constexpr int CH = 1;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += CH) {
        if (!active) break;
        XfOps ops[CH];
        bool kp[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            const int e = e0 + j, i = t + T * e;
            kp[j] = !(e >= ZLO && e < ZHI) && abs(signed_index(i, NX)) <= a.kcx && !(i == 0 && ky == 0);
            if (kp[j]) ops[j] = xf_load(a, final, fuse, stage, e1y, e2y, i, (size_t)kyl * NX + i);
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            const int e = e0 + j;
            if (e >= ZLO && e < ZHI) continue;  // |kx| > kcx there
            const int slot = e < ZLO ? e : e - (ZHI - ZLO);
            const int i = t + T * e;
            if (!kp[j]) {
                if (fuse) sv[slot * T + t] = zero();  // psi of the next stage: 0 here
                continue;
            }
            const double kxv = a.kx_scale * (double)signed_index(i, NX);
            const size_t idx = (size_t)kyl * NX + i;
            const cd kv = add(sv[slot * T + t], scale(v[e], kxv * kxv - kyv * kyv));
            const cd wn = xf_point(a, stage, final, fuse, kyv, kxv, pw, idx, kv, ops[j], bad, sE, sZ, sD);
            if (fuse) {  // psi = w / |k|^2 of the next stage (k1_xinv prologue)
                const double ksq = kxv * kxv + kyv * kyv;
                const double r = __drcp_rn(ksq);  // ksq > 0: the mean mode was skipped
                sv[slot * T + t] = mk(wn.x * r, wn.y * r);
            }
        }
    }
    if (final && a.diag) diag_accumulate(a.diag + 3 * (a.flags->steps - 1), sE, sZ, sD);
    if (bad) {
        atomicMin(&a.flags->div_var, 0);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
    if constexpr (FUSE) {
        if (!next) return;
        // next stage's x-inverse of this column: X[psi], X[kx psi] (k1_xinv, NM = 2)
#pragma unroll 1
        for (int m = 0; m < 2; ++m) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (e >= ZLO && e < ZHI) {
                    v[e] = zero();
                    continue;
                }
                const int slot = e < ZLO ? e : e - (ZHI - ZLO);
                const cd psi = sv[slot * T + t];
                v[e] = m == 0 ? psi : scale(psi, a.kx_scale * (double)signed_index(t + T * e, NX));
            }
            F::template run<+1>(v, sm, t, wb);
            if (active) {
#pragma unroll
                for (int e = 0; e < E; ++e) *xinv_dst(a, m, t + T * e, kyl) = v[e];
            }
        }
        if (a.p2p) __threadfence_system();
    }
}

// Paired x-forward for grids with few kept columns (one wave of columns):
// one column per CTA and two line groups of T threads, group 0 on the
// product spectrum A, group 1 on B, so the column's two forward FFTs run
// side by side, and then (FUSE) the next stage's two x-inverse FFTs (psi and
// kx psi) too: the column's critical path holds 2 FFTs instead of 4.  The
// RK epilogue is split between the groups (kept slots [0, NS/2) in group 0,
// the rest in group 1).  Same arithmetic per mode as k4b_xfwd (xf_point).
template <int NX, int EM>
struct XPCfg {
    using C = XCfg<NX, EM, 1>;
    using F = typename C::F;
    static constexpr int T = F::T, CT = 2 * T;
    static constexpr int NS = F::E - (C::ZHI - C::ZLO);  // kept slots per thread
    static constexpr int MINB = 65536 / (CT * SKG_PAIRED_REGS) > 16 ? 16 : 65536 / (CT * SKG_PAIRED_REGS);
    static constexpr size_t SMEM = sizeof(cd) * (2 * F::SMEM + 2 * NS * T);
};

template <int NX, int EM, bool FUSE>
__global__ void __launch_bounds__(XPCfg<NX, EM>::CT, XPCfg<NX, EM>::MINB)
    k4p_xfwd(Ns2dArgs a, int stage, int next) {
    using P = XPCfg<NX, EM>;
    using F = typename P::F;
    constexpr int T = F::T, E = F::E, NS = P::NS;
    constexpr int ZLO = P::C::ZLO, ZHI = P::C::ZHI;
    extern __shared__ cd smem[];
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const int kyl = blockIdx.x;  // local column (grid = ncols)
    const int ky = a.c0 + kyl;
    const typename F::Bases wb = F::bases(t, a.twx);  // constant table: before the wait
    cd* ex = smem + g * F::SMEM;  // the group's exchange buffer
    cd* sa = smem + 2 * F::SMEM;  // kx ky A^, then psi of the next stage
    cd* sb = sa + NS * T;         // (kx^2 - ky^2) B^
    const int bar = g + 1;
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    const bool fuse = FUSE && next;
    const size_t col = (size_t)kyl * NX;
    const double kyv = a.ky_scale * (double)ky;
    const size_t blk = (size_t)2 * ((a.ncols + 1) >> 1) * a.nrl;  // receive block per source
    pdl_wait();
    const int dflag = *reinterpret_cast<const volatile int*>(&a.flags->diverged);
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int x = t + T * e;
        const int ro = x >> a.lg_nrl, xl = x & (a.nrl - 1);
        v[e] = a.rA[g][ro * blk + ((size_t)(kyl >> 1) * a.nrl + xl) * 2 + (kyl & 1)];
    }
    if (__syncthreads_or(dflag) != 0) return;
    F::template run<-1>(v, ex, t, wb, 0, bar);
    cd* own = g == 0 ? sa : sb;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZLO && e < ZHI) continue;
        const int slot = e < ZLO ? e : e - (ZHI - ZLO);
        const double kxv = a.kx_scale * (double)signed_index(t + T * e, NX);
        own[slot * T + t] = scale(v[e], g == 0 ? kxv * kyv : kxv * kxv - kyv * kyv);
    }
    __syncthreads();
    bool bad = false;
    double sE = 0.0, sZ = 0.0, sD = 0.0;
    const double pw = (ky == 0 || ky == a.nh - 1) ? 1.0 : 2.0;
    if (final && a.diag && ky == 0 && g == 0 && t == 0) {
        const cd u0 = a.u[col];  // mean mode: untouched, enstrophy only
        sZ += 0.5 * pw * (u0.x * u0.x + u0.y * u0.y);
    }
    const double e1y = a.has_sigma ? a.e1y[ky] : 1.0, e2y = a.has_sigma ? a.e2y[ky] : 1.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZLO && e < ZHI) continue;
        const int slot = e < ZLO ? e : e - (ZHI - ZLO);
        if ((slot < NS / 2) != (g == 0)) continue;
        const int i = t + T * e;
        if (abs(signed_index(i, NX)) > a.kcx || (i == 0 && ky == 0)) {
            if (fuse) sa[slot * T + t] = zero();  // psi of the next stage: 0 here
            continue;
        }
        const double kxv = a.kx_scale * (double)signed_index(i, NX);
        const XfOps o = xf_load(a, final, fuse, stage, e1y, e2y, i, col + i);
        const cd kv = add(sa[slot * T + t], sb[slot * T + t]);
        const cd wn = xf_point(a, stage, final, fuse, kyv, kxv, pw, col + i, kv, o, bad, sE, sZ, sD);
        if (fuse) {  // psi = w / |k|^2 of the next stage (k1_xinv prologue)
            const double ksq = kxv * kxv + kyv * kyv;
            const double r = __drcp_rn(ksq);
            sa[slot * T + t] = mk(wn.x * r, wn.y * r);
        }
    }
    if (final && a.diag) diag_accumulate(a.diag + 3 * (a.flags->steps - 1), sE, sZ, sD);
    if (bad) {
        atomicMin(&a.flags->div_var, 0);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
    if constexpr (FUSE) {
        if (!next) return;
        __syncthreads();  // psi complete
        // next stage's x-inverse: group 0 X[psi], group 1 X[kx psi]
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= ZLO && e < ZHI) {
                v[e] = zero();
                continue;
            }
            const int slot = e < ZLO ? e : e - (ZHI - ZLO);
            const cd psi = sa[slot * T + t];
            v[e] = g == 0 ? psi : scale(psi, a.kx_scale * (double)signed_index(t + T * e, NX));
        }
        F::template run<+1>(v, ex, t, wb, 0, bar);
#pragma unroll
        for (int e = 0; e < E; ++e) *xinv_dst(a, g, t + T * e, kyl) = v[e];
        if (a.p2p) __threadfence_system();
    }
}

template <int NX, bool PZ, int NM, int EM = 16, int CTW = 256>
cudaError_t launch_k1(const Ns2dArgs& a, int stage, cudaStream_t s) {
    using C = XCfg<NX, EM, CTW>;
    using F = typename C::F;
    constexpr int T = F::T, E = F::E;
    constexpr int LPC = C::LPC;
    constexpr int NS = PZ ? E - (C::ZHI - C::ZLO) : E;
    const size_t smem = sizeof(cd) * (F::SMEM + NS * T) * LPC;
    const int grid = ((NM == 2 ? a.ncols : a.ky_in) + LPC - 1) / LPC;
    if (grid == 0) return cudaSuccess;
    SKG_TRY(launch_pdl(k1_xinv<NX, PZ, NM, EM, CTW>, grid, T * LPC, smem, s, a, stage));
    return cudaGetLastError();
}

template <int NX>
cudaError_t launch_x(const Ns2dArgs& a, int stage, bool inverse, cudaStream_t s) {
    using F = BFFT<NX>;
    constexpr int T = F::T;
    constexpr int LPC = T >= 256 ? 1 : 256 / T;
    if (inverse) {
        if constexpr (NX >= 64) {
            if (a.pruned && a.kcx <= 6 * T - 1) return launch_k1<NX, true, 4>(a, stage, s);
        }
        return launch_k1<NX, false, 4>(a, stage, s);
    }
    const size_t smem = sizeof(cd) * F::SMEM * LPC;
    const int grid = (a.ld_o + LPC - 1) / LPC;
    if (grid == 0) return cudaSuccess;
    SKG_TRY(launch_pdl(k4_xfwd<NX>, grid, T * LPC, smem, s, a, stage));
    return cudaGetLastError();
}

template <int NY, bool CFL>
cudaError_t launch_y_v(const Ns2dArgs& a, cudaStream_t s) {
    constexpr int EM = 16;
    using F = BFFT<NY, true, EM>;
    constexpr int T = F::T;
    constexpr int G = T >= 256 ? 1 : 256 / T;
    const size_t smem = sizeof(cd) * (F::SMEM + NY / 2 + 2 * a.ld_i) * G;
    const int pairs = a.nx / 2;
    const int grid = (pairs + G - 1) / G;
    SKG_TRY(launch_pdl(k3_phys<NY, EM, CFL>, grid, T * G, smem, s, a));
    return cudaGetLastError();
}

template <int NY>
cudaError_t launch_y(const Ns2dArgs& a, cudaStream_t s) {
    return (a.dyn && a.ystage == 1) ? launch_y_v<NY, true>(a, s) : launch_y_v<NY, false>(a, s);
}

template <int NY, bool CFL>
cudaError_t launch_fast_y_v(const Ns2dArgs& a, cudaStream_t s) {
    constexpr int EM = NY >= 4096 ? SKG_FAST_Y_EM : NY <= SKG_Y_EM4_MAX ? 4 : SKG_FAST_Y_EM_SMALL;
    using F = BFFT<NY, false, EM>;
    constexpr int G = F::T >= 256 ? 1 : 256 / F::T;
    const size_t smem = sizeof(cd) * (F::SMEM + 2 * a.ld_i) * G;
    const int groups = (a.nrl + G - 1) / G;
    const int wave = a.wave / 2 * y_minb<NY, EM>();  // a.wave = 2 CTAs per SM
    const int grid = groups < wave ? groups : wave;
    SKG_TRY(launch_pdl(k3b_phys<NY, CFL, EM>, grid, F::T * G, smem, s, a));
    return cudaGetLastError();
}

template <int NY>
cudaError_t launch_fast_y(const Ns2dArgs& a, cudaStream_t s) {
    return (a.dyn && a.ystage == 1) ? launch_fast_y_v<NY, true>(a, s) : launch_fast_y_v<NY, false>(a, s);
}

// elements per thread of the fast path's x passes
template <int NX>
constexpr int fast_em() { return NX >= 4096 ? SKG_FAST_X_EM : NX <= SKG_X_EM4_MAX ? 4 : SKG_FAST_X_EM_SMALL; }

// mode 0: x-inverse (k1_xinv); 1: x-forward + RK; 2: x-forward + RK fused
// with the next stage's x-inverse.
template <int NX, int CTW, bool FUSE>
cudaError_t launch_k4b(const Ns2dArgs& a, int stage, cudaStream_t s) {
    constexpr int EM = fast_em<NX>();
    using C = XCfg<NX, EM, CTW>;
    using F = typename C::F;
    constexpr int T = F::T;
    constexpr int LPC = C::LPC;
    const size_t smem = sizeof(cd) * xf_slot<NX, EM, CTW>() * LPC;
    const int grid = (a.ncols + LPC - 1) / LPC;
    if (grid == 0) return cudaSuccess;
    SKG_TRY(launch_pdl(k4b_xfwd<NX, EM, CTW, FUSE>, grid, T * LPC, smem, s,
                          a, stage, FUSE ? 1 : 0));
    return cudaGetLastError();
}

template <int NX, bool FUSE>
cudaError_t launch_k4p(const Ns2dArgs& a, int stage, cudaStream_t s) {
    constexpr int EM = fast_em<NX>();
    using P = XPCfg<NX, EM>;
    if (a.ncols == 0) return cudaSuccess;
    SKG_TRY(launch_pdl(k4p_xfwd<NX, EM, FUSE>, a.ncols, P::CT, P::SMEM, s, a, stage, FUSE ? 1 : 0));
    return cudaGetLastError();
}

template <int NX, int CTW>
cudaError_t launch_fast_x_w(const Ns2dArgs& a, int stage, int mode, cudaStream_t s) {
    constexpr int EM = fast_em<NX>();
    if (mode == 0) return launch_k1<NX, true, 2, EM, CTW>(a, stage, s);
    if constexpr (NX >= SKG_PAIRED_X_MIN && NX <= SKG_PAIRED_X_MAX) {
        return mode == 2 ? launch_k4p<NX, true>(a, stage, s) : launch_k4p<NX, false>(a, stage, s);
    }

    if (mode == 2) return launch_k4b<NX, CTW, true>(a, stage, s);
    return launch_k4b<NX, CTW, false>(a, stage, s);
}

// Narrow CTAs (one column each) when 256-thread CTAs would leave SMs idle.
template <int NX>
cudaError_t launch_fast_x(const Ns2dArgs& a, int stage, int mode, cudaStream_t s) {
    constexpr int EM = fast_em<NX>();
    constexpr int LPC = XCfg<NX, EM>::LPC;
    if constexpr (LPC > 1) {
        if ((a.ncols + LPC - 1) / LPC < a.wave) return launch_fast_x_w<NX, 1>(a, stage, mode, s);
    }
    return launch_fast_x_w<NX, 256>(a, stage, mode, s);
}

#define SKG_POW2_CASES(X) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#define SKG_FAST_CASES(X) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)

cudaError_t dispatch_x(const Ns2dArgs& a, int stage, bool inverse, cudaStream_t s) {
    switch (a.nx) {
#define CASE(N) \
    case N: return launch_x<N>(a, stage, inverse, s);
        SKG_POW2_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t dispatch_y(const Ns2dArgs& a, cudaStream_t s) {
    switch (a.ny) {
#define CASE(N) \
    case N: return launch_y<N>(a, s);
        SKG_POW2_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t dispatch_fast_x(const Ns2dArgs& a, int stage, int mode, cudaStream_t s) {
    switch (a.nx) {
#define CASE(N) \
    case N: return launch_fast_x<N>(a, stage, mode, s);
        SKG_FAST_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t dispatch_fast_y(const Ns2dArgs& a, cudaStream_t s) {
    switch (a.ny) {
#define CASE(N) \
    case N: return launch_fast_y<N>(a, s);
        SKG_FAST_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

// Basdevant form applies when the state is dealiased, the 2/3 rule makes
// the products alias-free on the kept modes (3 kc < n on both axes) and the
// kept kx leave the per-thread zero band e in [6, 10) of the x FFT empty.
bool fast_ok(const Ns2dArgs& a) {
    if (!a.pruned || a.nx < 64 || a.ny < 64) return false;
    if (3 * a.kcx >= a.nx || 3 * a.kcy >= a.ny) return false;
    const int T = a.nx / 16;
    return a.kcx <= 6 * T - 1 && a.ky_in <= 6 * (a.ny / 16) && a.ld_o <= 6 * (a.ny / 16);
}

}  // namespace

// The general (non-dealiased) passes hold a whole line plus its stage in
// shared memory: 4096 is the largest extent that fits 227 KB for every
// state, so larger grids run the generic step (generic.cu) instead.
bool ns2d_supported(int nx, int ny) {
    auto ok = [](int n) { return n >= 4 && n <= 4096 && (n & (n - 1)) == 0; };
    return ok(nx) && ok(ny);
}

bool ns2d_fast_ok(const Ns2dArgs& a) { return fast_ok(a); }

cudaError_t ns2d_fast_pass(const Ns2dArgs& a, int pass, int stage, cudaStream_t s, long* launches,
                           const LaunchHook& hook, int next) {
    cudaError_t err;
    const double B = sizeof(cd);
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    const double kept = (2.0 * a.kcx + 1.0) * a.ncols;  // modes of this partition
    const double Kc = a.kcy + 1.0;
    if (pass == 0) {
        hook.begin(0);
        err = dispatch_fast_x(a, stage, 0, s);
        hook.end(0, B * (kept * (stage == 1 ? 1.0 : 2.0) + 2.0 * a.nx * a.ncols));
    } else if (pass == 1) {
        hook.begin(1);
        Ns2dArgs b = a;
        b.ystage = stage;
        err = dispatch_fast_y(b, s);
        hook.end(1, B * (4.0 * a.nrl * Kc));
    } else if (pass == 2 || !next) {
        hook.begin(2);
        err = dispatch_fast_x(a, stage, 1, s);
        hook.end(2, B * (2.0 * a.nx * a.ncols + (final ? (a.rk2 ? 3.0 : 5.0) : 1.0) * kept));
    } else {  // pass 3: x-forward + RK fused with the next stage's x-inverse
        hook.begin(2);
        err = dispatch_fast_x(a, stage, 2, s);
        hook.end(2, B * (4.0 * a.nx * a.ncols + (final ? (a.rk2 ? 3.0 : 5.0) : 2.0) * kept));
    }
    ++*launches;
    return err;
}

cudaError_t ns2d_launch_stage(const Ns2dArgs& a, int stage, cudaStream_t s, long* launches,
                              const LaunchHook& hook) {
    cudaError_t err;
    const double B = sizeof(cd);
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    const double kx_kept = a.pruned ? 2.0 * a.kcx + 1.0 : (double)a.nx;
    const double s_in = kx_kept * a.ky_in;          // modes K1 reads per field
    const double s_out = kx_kept * a.ld_o;          // modes K4 touches per field
    const double inter = (double)a.nx * a.ky_in;    // one intermediate field
    const double rows = (double)a.nx * a.ld_o;      // tendency rows
    if (fast_ok(a)) {
        for (int pass = 0; pass < 3; ++pass)
            if ((err = ns2d_fast_pass(a, pass, stage, s, launches, hook)) != cudaSuccess) return err;
        return cudaSuccess;
    }
    hook.begin(0);
    if ((err = dispatch_x(a, stage, true, s)) != cudaSuccess) return err;
    hook.end(0, B * (s_in * (stage == 1 ? 1.0 : 2.0) + 4.0 * inter));
    hook.begin(1);
    Ns2dArgs b = a;
    b.ystage = stage;
    if ((err = dispatch_y(b, s)) != cudaSuccess) return err;
    hook.end(1, B * (4.0 * inter + rows));
    hook.begin(2);
    if ((err = dispatch_x(a, stage, false, s)) != cudaSuccess) return err;
    hook.end(2, B * (rows + (final ? (a.rk2 ? 3.0 : 5.0) * s_out : s_out)));
    *launches += 3;
    if (final && !a.pruned && a.nh > a.kcy + 1) {
        hook.begin(3);
        SKG_TRY(launch_pdl(k4_decay, 296, 256, 0, s, a));
        hook.end(3, B * 2.0 * a.nx * (a.nh - a.kcy - 1));
        *launches += 1;
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace skg
