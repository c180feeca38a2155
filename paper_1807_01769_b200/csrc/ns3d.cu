// ns3d.cu -- fused RK stage of the 3D rotational-form solver on sm_100a.
//
// Ns3dSolver::tendency (reference proj/src/solvers.cpp:299-339):
//   w = curl v (grid.cpp:182-207); u, w <- 6 c2r; c = u x w (solvers.cpp:321-325);
//   3 r2c; Leray projection (grid.cpp:227-249); dealias; mean 0.
// One RK stage = five kernels, each one 1D FFT pass with the pointwise work
// fused into its prologue / epilogue (SURVEY.md 8(a), ns3d mapping):
//   k1_3d  x-inverse per (ky, kz) line: RK stage state (time_stepping.cpp:
//          128-170) of vx, vy, vz -> X[vx], X[vy], X[vz], X[kx vy], X[kx vz]
//   k2_3d  y-inverse per (x, kz) line: the three velocities and the three
//          vorticity components (ky, kz factors applied here)
//   k3_3d  z pass per pair of (x, y) rows: 6 c2r (3 packed complex FFTs),
//          u x w, 3 r2c (2 packed FFTs per row pair + 1 shared), *1/N
//   k2f_3d y-forward per (x, kz) line, kept ky only
//   k4_3d  x-forward per (ky, kz) line, projection, dealias, mean 0, RK
//          update and the check_finite guard (simulation.cpp:557-563)
// Strided-axis kernels map consecutive lanes to consecutive kz lines (the
// contiguous axis), so every global access is a run of >= 128 bytes; lines
// sharing a warp get distinct shared-memory banks through the FFT salt.
// "pruned" (dealiased state): only kept (ky, kz) lines / kept modes are
// touched; otherwise every mode is processed with identical results.
#include "skg_internal.h"

namespace skg {

namespace {

__device__ __forceinline__ bool finite2(cd v) { return isfinite(v.x) && isfinite(v.y); }

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Inter-pass intermediates are written once and read once by the next
// kernel, gigabytes later: SKG3_STCS = 1 stores them with the streaming
// (evict-first) policy so they do not displace the L2-resident reuse sets
// (scratch slots, secondary fields, twiddle tables).  A/B macro.
#ifndef SKG3_STCS
#define SKG3_STCS 0
#endif
__device__ __forceinline__ void st_stream(cd* p, cd v) {
#if SKG3_STCS
    __stcs(p, v);
#else
    *p = v;
#endif
}

// RK stage state from loaded u and previous k (time_stepping.cpp:128-170).
__device__ __forceinline__ cd stage_combine3(const Ns3dArgs& a, int stage, int i, int ky, int kz,
                                             cd u, cd k) {
    if (stage <= 1) return u;
    if (a.has_sigma) {
        const double e1 = a.e1x[i] * a.e1y[ky] * a.e1z[kz];
        if (stage == 2) return scale(add(u, scale(k, hdt_of(a))), e1);
        if (stage == 3) return add(scale(u, e1), scale(k, hdt_of(a)));
        const double e2 = a.e2x[i] * a.e2y[ky] * a.e2z[kz];
        return add(scale(u, e2), scale(k, dt_of(a) * e1));
    }
    return add(u, scale(k, stage == 4 ? dt_of(a) : hdt_of(a)));
}

// ky of the kyi-th processed line of the x passes.
__device__ __forceinline__ int ky_of(const Ns3dArgs& a, int kyi) {
    if (!a.pruned) return kyi;
    return kyi <= a.kcy ? kyi : a.ny - (2 * a.kcy + 1) + kyi;
}

// state index of mode (kx, line ys of the state layout, kz)
__device__ __forceinline__ size_t sidx(const Ns3dArgs& a, int kx, int ys, int kz) {
    return ((size_t)kx * a.ystate + ys) * a.sz + kz;
}

// Owner rank, first line and line count of compact kept line kyi under the
// partition kstart[q] = q K / G (K = 2 kcy + 1 kept lines; skgpu.cu
// create_impl), computed instead of loaded: q = ((kyi + 1) G - 1) / K.
__device__ __forceinline__ void line_owner(const Ns3dArgs& a, int kyi, int& q, int& ks, int& nk) {
    const int K = 2 * a.kcy + 1;
    q = ((kyi + 1) * a.G - 1) / K;
    ks = q * K / a.G;
    nk = (q + 1) * K / a.G - ks;
}

// Per-CTA table (shared memory) of the offset of line j (fixed x row) in the
// x-pass buffer read by k2 / written by k2f, for kz stride kzs; -1 where the
// line is masked.  Full layout: (x ny + j) kzs; slab layout: the owner's
// block [xl][kyl][kz] (line_owner), computed once per CTA instead of per
// element and field.
template <int NY>
__device__ __forceinline__ void line_offsets(const Ns3dArgs& a, int x, int kzs, int* off);

// compact kept index of a kept ky (0..kcy, then ny-kcy..ny-1)
__device__ __forceinline__ int ky_compact(const Ns3dArgs& a, int ky) {
    return ky <= a.kcy ? ky : ky - (a.ny - (2 * a.kcy + 1));
}

// x-inverse and y-forward: one component / field per CTA (blockIdx.y; a
// launch covers components [comp0, comp0 + ncomp), normally all three; the
// NCCL slab path launches them one at a time so the all-to-all of one
// overlaps the next one's pass) instead of three in sequence -- shorter dependent chains per CTA (ms/step:
// 64^3 0.201 -> 0.184, 128^3 0.601 -> 0.588, 512^3 31.10 -> 30.94,
// 256^3 3.889 -> 3.914).

// z pass, dealiased states: the Hermitian split of the forward output from
// registers (z_store_pair) instead of a shared-memory round trip of all
// elements.  Measured (ms/step) with the zero band on, register-fetch z
// pass: 512^3 32.55 vs 32.09 without it, 256^3 3.88 vs 3.95, 128^3 0.644 vs
// 0.632 -- off; the zero band alone: 512^3 32.70 -> 32.09, 256^3 4.06 -> 3.95.
// With the staged, shared-memory-bound 512^3 z pass it pays (below: on
// there, SKG3_Z_HERM forces it everywhere).
#ifndef SKG3_Z_HERM
#define SKG3_Z_HERM 0
#endif

// z pass inputs staged in shared memory by bulk (TMA 1D) copies on an
// mbarrier, one packed pair ahead, so the loads of the next pair land while
// the current FFT runs (the register-fetch variant waits on them: long
// scoreboard was the z pass's top stall); the second inverse FFT's output
// (wy + i wz) stays in registers instead of two shared-memory rows.
// Measured (ms/step, B200): 512^3 31.52 -> 30.74 with 3 row-pair groups per
// CTA (168 registers, no spills; two CTAs per SM) and the second inverse
// output in shared memory, 30.50 with 2 groups (3 CTAs per SM), 30.38 with
// one group per CTA (64 threads, 6 CTAs per SM: independent scheduling);
// 256^3 3.82 -> 3.79 with 8 groups and that output in registers; 128^3
// slower (0.574 -> 0.617) -- so 256 and 512 (1024: SKG3_ZSTAGE1024).
#ifndef SKG3_ZSTAGE
#define SKG3_ZSTAGE 1
#endif

#ifndef SKG3_ZG512
#define SKG3_ZG512 1
#endif
#ifndef SKG3_ZSTAGE1024
#define SKG3_ZSTAGE1024 0
#endif
template <int NZ>
constexpr bool zstage() { return SKG3_ZSTAGE && (NZ == 256 || NZ == 512 || (NZ == 1024 && SKG3_ZSTAGE1024)); }
// 512^3, staged: the second inverse output in registers (168 of them) and
// the Hermitian split from registers -- the pass is shared-memory bound, and
// these remove ~55 KB of its ~510 KB of shared traffic per row pair:
// 30.38 -> 29.50 ms/step (either alone: 30.45 / 29.91); at 256^3 the split
// from registers is slower (3.78 -> 3.89).
template <int NZ>
constexpr bool zreg() { return NZ == 256 || NZ == 512; }
template <int NZ>
constexpr bool zherm() { return NZ == 512 && zstage<NZ>(); }

// Elements per thread of the strided (x, y) passes: 8 for N <= SKG3_EM8_MAX
// (twice the threads per line; the small grids have too few lines to fill
// the GPU with 16-element lines), else 16.  Measured (ms/step): 64^3
// 0.341 -> 0.222, 128^3 0.634 -> 0.630, 256^3 4.19 -> 4.06, 512^3 32.8 -> 36.4
// (so 16 from 512 on).
// z pass at NZ = 128: 14 row-pair groups per CTA (224 threads) instead of
// 16: two CTAs per SM then hold 148 * 28 = 4144 groups, and the 8192 row
// pairs of 128^3 take 1.98 waves instead of 1.73 (a 73%-full second wave).
// 128^3: 0.584 -> 0.568 ms/step (10 groups: 0.604, 8: 0.597).
#ifndef SKG3_ZG128
#define SKG3_ZG128 14
#endif
#ifndef SKG3_EM8_MAX
#define SKG3_EM8_MAX 256
#endif
template <int N>
constexpr int em3() { return N <= SKG3_EM8_MAX && N >= 16 ? 8 : 16; }
template <int N>
using BF3 = BFFT<N, false, em3<N>()>;

// Lines per CTA for the strided passes: lanes walk the contiguous kz axis.
template <int N, int CT = 256>
struct Strided {
    using F = BF3<N>;
    static constexpr int T = F::T;
    static constexpr int C = T >= CT ? 1 : CT / T;
    static constexpr int MINB = T * C >= 512 ? 1 : 512 / (T * C);  // keeps <= 128 registers
};

// ------------------------------------------------------------------ x-inverse
// Each velocity component's stage state is computed once (u and k_{j-1}
// streamed into shared memory with cp.async) and kept in thread-private
// slots for its one or two FFTs.  PZ: dealiased state with kcx < 6T, so the
// per-thread elements e in [6, 10) are zero and need no slot.
template <int NX, bool PZ, int CB = 256>
__global__ void __launch_bounds__(CB, Strided<NX, CB>::MINB) k1_3d(Ns3dArgs a, int stage) {
    using F = BF3<NX>;
    constexpr int T = F::T, E = F::E, C = Strided<NX, CB>::C;
    // zero band e in [3E/8, 5E/8): kx in [3N/8, 5N/8)
    constexpr int ZLO = PZ ? 3 * E / 8 : E, ZHI = PZ ? 5 * E / 8 : E;
    constexpr int CT = T * C;  // threads per CTA
    extern __shared__ cd smem[];
    const int l = threadIdx.x % C, t = threadIdx.x / C;
    const int nkzb = (a.kz_in + C - 1) / C;
    const int kyi = a.kys + blockIdx.x / nkzb;
    const int kz = (blockIdx.x % nkzb) * C + l;
    const bool active = kz < a.kz_in;
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    if (stage == 1 && blockIdx.x == 0 && blockIdx.y == 0 && a.comp0 == 0 && threadIdx.x == 0 && a.lead)
        atomicAdd(&a.flags->steps, 1);
    const int ky = ky_of(a, kyi);
    const int ys = a.slab ? kyi - a.kys : ky;
    cd* sm = smem + l * F::SMEM;
    cd* slots = smem + C * F::SMEM;  // slots[slot * CT + tid]
    cd* kst = smem;                  // k staging in the idle exchange buffers
    const int salt = l & 7;
    const typename F::Bases wb = F::bases(t, a.twx);
    const cd* kprev = stage == 2 ? a.k1 : stage == 3 ? a.k2 : a.k3;
    // one velocity component per CTA
    const int c0 = a.comp0 + blockIdx.y, c1 = c0 + 1;
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
        const size_t ubase = sidx(a, t, ys, kz) + c * a.vstride, ustr = (size_t)T * a.ystate * a.sz;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= ZLO && e < ZHI) continue;
            const int slot = e < ZLO ? e : e - (ZHI - ZLO);
            const int i = t + T * e;
            const bool keep = active && (!a.pruned || abs(signed_index(i, NX)) <= a.kcx);
            if (keep) {
                const size_t idx = ubase + e * ustr;  // sidx(a, i, ys, kz) + c * a.vstride
                cp_async16(&slots[slot * CT + threadIdx.x], a.u + idx);
                if (stage > 1) cp_async16(&kst[slot * CT + threadIdx.x], kprev + idx);
            }
        }
        cp_async_commit();
        cp_async_wait_all();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= ZLO && e < ZHI) continue;
            const int slot = e < ZLO ? e : e - (ZHI - ZLO);
            const int i = t + T * e;
            const bool keep = active && (!a.pruned || abs(signed_index(i, NX)) <= a.kcx);
            cd s = zero();
            if (keep)
                s = stage_combine3(a, stage, i, ky, kz, slots[slot * CT + threadIdx.x],
                                   stage > 1 ? kst[slot * CT + threadIdx.x] : zero());
            slots[slot * CT + threadIdx.x] = s;
        }
        __syncthreads();  // k staging lived in the exchange buffers
#pragma unroll 1
        for (int q = 0; q < (c == 0 ? 1 : 2); ++q) {
            const int m = q == 0 ? c : c + 2;  // X[v_c] or X[kx v_c]
            cd v[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (e >= ZLO && e < ZHI) {
                    v[e] = zero();
                    continue;
                }
                const int slot = e < ZLO ? e : e - (ZHI - ZLO);
                const cd sv = slots[slot * CT + threadIdx.x];
                v[e] = q == 0 ? sv : scale(sv, a.kx_scale * (double)signed_index(t + T * e, NX));
            }
            F::template run<+1>(v, sm, t, wb, salt);
            if (active) {
                if (!a.p2p) {
                    cd* out = a.A + m * a.fstride + ((size_t)t * a.ystate + ys) * a.kz_in + kz;
                    const size_t ost = (size_t)T * a.ystate * a.kz_in;
#pragma unroll
                    for (int e = 0; e < E; ++e) st_stream(out + e * ost, v[e]);
                } else {  // straight into the row owner's receive block (layout [xl][kyl][kz])
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int x = t + T * e, q = x / a.nrl, xl = x - q * a.nrl;
                        a.peer_rA[q][m * a.rfs + (size_t)a.nrl * a.kys * a.kz_in +
                                     ((size_t)xl * a.nkyl + ys) * a.kz_in + kz] = v[e];
                    }
                }
            }
        }
    }
    if (a.p2p) __threadfence_system();  // peer stores visible before the barrier
}

// p2p y-forward destinations of line j for local row x: the owner q's receive
// block from this rank, r nrl nk_q kz + (x nk_q + kyi - ks_q) kz (exchange3's
// layout), and the owner in own[j]
template <int NY>
__device__ __forceinline__ void line_offsets_p2p(const Ns3dArgs& a, int x, int kzs, int* off, int* own) {
    for (int j = threadIdx.x; j < NY; j += blockDim.x) {
        const int sj = signed_index(j, NY);
        int o = -1, qq = 0;
        if (abs(sj) <= a.kcy) {
            const int kyi = ky_compact(a, j);
            int q, ks, nk;
            line_owner(a, kyi, q, ks, nk);
            o = a.r * a.nrl * nk * kzs + (x * nk + (kyi - ks)) * kzs;
            qq = q;
        }
        off[j] = o;
        own[j] = qq;
    }
    __syncthreads();
}

template <int NY>
__device__ __forceinline__ void line_offsets(const Ns3dArgs& a, int x, int kzs, int* off) {
    for (int j = threadIdx.x; j < NY; j += blockDim.x) {
        const int sj = signed_index(j, NY);
        int o = -1;
        if (!a.pruned || abs(sj) <= a.kcy) {
            if (!a.slab) {
                o = (x * a.ny + j) * kzs;
            } else {
                const int kyi = ky_compact(a, j);
                int q, ks, nk;
                line_owner(a, kyi, q, ks, nk);
                o = a.nrl * ks * kzs + (x * nk + (kyi - ks)) * kzs;
            }
        }
        off[j] = o;
    }
    __syncthreads();
}

// ------------------------------------------------------------------ y-inverse
template <int NY, int CT = 256>
__global__ void __launch_bounds__(CT, Strided<NY, CT>::MINB) k2_3d(Ns3dArgs a) {
    using F = BF3<NY>;
    constexpr int T = F::T, E = F::E, C = Strided<NY, CT>::C;
    extern __shared__ cd smem[];
    const int l = threadIdx.x % C, t = threadIdx.x / C;
    const int nkzb = (a.kz_in + C - 1) / C;
    const int x = blockIdx.x / nkzb;
    const int kz = (blockIdx.x % nkzb) * C + l;
    const bool active = kz < a.kz_in;
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    cd* sm = smem + l * F::SMEM;
    const int salt = l & 7;
    const typename F::Bases wb = F::bases(t, a.twy);
    const double kzv = a.kz_scale * (double)(a.kz0 + kz);
    const cd* Ab = a.slab ? a.rA : a.A;
    const size_t afs = a.slab ? a.rfs : a.fstride;
    const cd* A0 = Ab;
    const cd* A1 = Ab + afs;
    const cd* A2 = Ab + 2 * afs;
    const cd* A3 = Ab + 3 * afs;
    const cd* A4 = Ab + 4 * afs;
    int* loff = reinterpret_cast<int*>(smem + C * F::SMEM);
    line_offsets<NY>(a, x, a.kz_in, loff);
#pragma unroll 1
    for (int m = 0; m < 6; ++m) {
        cd v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = t + T * e;
            const int sj = signed_index(j, NY);
            const int lo = loff[j];
            cd r = zero();
            if (active && lo >= 0) {
                const size_t q = (size_t)lo + kz;
                const double kyv = a.ky_scale * (double)sj;
                switch (m) {
                    case 0: r = A0[q]; break;  // vx
                    case 1: r = A1[q]; break;  // vy
                    case 2: r = A2[q]; break;  // vz
                    case 3: {                  // wx = i (ky vz - kz vy)
                        const cd p2 = A2[q], p1 = A1[q];
                        r = muli(sub(scale(p2, kyv), scale(p1, kzv)));
                    } break;
                    case 4: {                  // wy = i (kz vx - kx vz)
                        const cd p0 = A0[q], p4 = A4[q];
                        r = muli(sub(scale(p0, kzv), p4));
                    } break;
                    default: {                 // wz = i (kx vy - ky vx)
                        const cd p3 = A3[q], p0 = A0[q];
                        r = muli(sub(p3, scale(p0, kyv)));
                    } break;
                }
            }
            v[e] = r;
        }
        F::template run<+1>(v, sm, t, wb, salt);
        if (active) {
            cd* out = a.B + m * a.fstride;
#pragma unroll
            for (int e = 0; e < E; ++e)
                out[((size_t)x * a.ny + (t + T * e)) * a.kz_in + kz] = v[e];
        }
    }
}

// Staged variant (dealiased states): the kept lines of the next output's
// primary field stream into shared memory (cp.async, compact kept-line
// index) while the current FFT runs; the secondary field of the three
// vorticity outputs is read directly (recently read by this CTA: L2).
// Output m: primary / secondary = A0 / -, A1 / -, A2 / -, A2 / A1, A4 / A0,
// A3 / A0 (processed as two halves, see the order below).
// ZB: kcy < 3 NY / 8, so the inputs e in [3E/8, 5E/8) are masked (zero)
// One tile of the staged y-inverse: x row and kz block from bx, outputs
// i0..i1 of the processing order below (all six, or one self-contained half).
template <int NY, int CT, bool ZB>
__device__ __forceinline__ void y_inv_tile(const Ns3dArgs& a, cd* smem, int bx, int i0, int i1) {
    using F = BF3<NY>;
    constexpr int T = F::T, E = F::E, C = Strided<NY, CT>::C;
    constexpr int ZLO = ZB ? 3 * E / 8 : E, ZHI = ZB ? 5 * E / 8 : E;
    const int l = threadIdx.x % C, t = threadIdx.x / C;
    const int nkzb = (a.kz_in + C - 1) / C;
    const int x = bx / nkzb;
    const int kz0 = (bx % nkzb) * C;
    const int kz = kz0 + l;
    const bool active = kz < a.kz_in;
    const int K = 2 * a.kcy + 1;  // kept lines
    cd* sm = smem + l * F::SMEM;
    cd* stg = smem + C * F::SMEM;                       // [kyi][l]
    int* loff = reinterpret_cast<int*>(stg + (size_t)K * C);
    const int salt = l & 7;
    const typename F::Bases wb = F::bases(t, a.twy);
    const double kzv = a.kz_scale * (double)(a.kz0 + kz);
    const cd* Ab = a.slab ? a.rA : a.A;
    const size_t afs = a.slab ? a.rfs : a.fstride;
    line_offsets<NY>(a, x, a.kz_in, loff);
    const int nl = a.kz_in - kz0 < C ? a.kz_in - kz0 : C;  // active lanes
    auto issue = [&](int f) {
        const cd* src = Ab + (size_t)f * afs + kz0;
        for (int i = threadIdx.x; i < K * C; i += blockDim.x) {
            const int kyi = i / C, ll = i % C;
            if (ll >= nl) continue;
            const int j = kyi <= a.kcy ? kyi : kyi + (NY - K);
            cp_async16(&stg[i], src + loff[j] + ll);
        }
        cp_async_commit();
    };
    // Processing order 0, 5, 4, 1, 3, 2: each secondary field (A0 for
    // outputs 5 and 4, A1 for 3) was this CTA's previous primary (still in
    // L2), and outputs 3 and 2 share the primary A2, staged once.  With
    // gridDim.y == 2 the two halves {0, 5, 4} and {1, 3, 2} (each closed
    // under its secondary) run in separate CTAs.
    auto order = [](int i) { return i == 0 ? 0 : i == 1 ? 5 : i == 2 ? 4 : i == 3 ? 1 : i == 4 ? 3 : 2; };
    auto primary = [](int m) { return m == 3 ? 2 : m == 4 ? 4 : m == 5 ? 3 : m; };
    issue(primary(order(i0)));
#pragma unroll 1
    for (int i = i0; i < i1; ++i) {
        const int m = order(i);
        cp_async_wait_all();
        __syncthreads();
        const cd* sec = Ab + (size_t)(m == 3 ? 1 : 0) * afs;
        cd v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= ZLO && e < ZHI) {
                v[e] = zero();
                continue;
            }
            const int j = t + T * e;
            const int sj = signed_index(j, NY);
            cd r = zero();
            if (active && abs(sj) <= a.kcy) {
                const int kyi = sj >= 0 ? sj : sj + K;
                const cd p = stg[kyi * C + l];
                const double kyv = a.ky_scale * (double)sj;
                if (m < 3) {
                    r = p;
                } else {
                    const cd q = sec[(size_t)loff[j] + kz];
                    if (m == 3) r = muli(sub(scale(p, kyv), scale(q, kzv)));  // wx = i (ky vz - kz vy)
                    else if (m == 4) r = muli(sub(scale(q, kzv), p));         // wy = i (kz vx - kx vz)
                    else r = muli(sub(p, scale(q, kyv)));                     // wz = i (kx vy - ky vx)
                }
            }
            v[e] = r;
        }
        if (i + 1 < i1 && primary(order(i + 1)) != primary(m)) {
            __syncthreads();  // stage consumed
            issue(primary(order(i + 1)));
        }
        F::template run<+1>(v, sm, t, wb, salt);
        if (active) {
            if (a.zfused) {  // pencil: straight into the row owner's z-pass input
                const size_t base = m * a.fsz + (size_t)x * a.nyl * a.kzf + a.kz0 + kz;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int y = t + T * e;
                    a.peer_Z[y >> a.lg_nyl][base + (size_t)(y & (a.nyl - 1)) * a.kzf] = v[e];
                }
            } else {
                cd* out = a.B + m * a.fstride + ((size_t)x * a.ny + t) * a.kz_in + kz;
                const unsigned ost = (unsigned)T * (unsigned)a.kz_in;
#pragma unroll
                for (int e = 0; e < E; ++e) st_stream(out + e * ost, v[e]);
            }
        }
    }
    if (a.zfused && a.p2p) __threadfence_system();  // peer stores visible before the barrier
    __syncthreads();  // smem (stage, line offsets) free for the next tile
}

template <int NY, int CT = 256, bool ZB = false>
__global__ void __launch_bounds__(CT, Strided<NY, CT>::MINB) k2s_3d(Ns3dArgs a) {
    extern __shared__ cd smem[];
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    // with gridDim.y == 2 the two output halves in separate CTAs
    const int i0 = gridDim.y == 2 ? 3 * blockIdx.y : 0, i1 = gridDim.y == 2 ? i0 + 3 : 6;
    y_inv_tile<NY, CT, ZB>(a, smem, blockIdx.x, i0, i1);
}

// ------------------------------------------------------------------ z pass
// Per group: one row pair (r, r+1) of (x, y) rows along z.
// 8 elements per thread (twice the warps per byte of shared memory).
// Elements per thread of the z lines: 8, except at 1024, where 16 saves an
// exchange of the shared-memory-bound pass (1024 = 16 * 16 * 4: three passes
// instead of 8 * 8 * 8 * 2's four) at 64 threads per line.  Measured at
// 1024^3 (ms per z-pass launch / ms per step, B200): 8 elements, 2 groups of
// 128 threads per CTA 28.1 / 318.2; 16 elements with 2 groups per CTA (two
// CTAs per SM) 22.9 / 297.4, 4 groups (one CTA) 23.7 / 301.0, ONE group per
// 64-thread CTA (three CTAs per SM) 22.3 / 295.0, staged inputs (bulk copies,
// SKG3_ZSTAGE1024) 25.1 / 306.0.  At 128^3 16 elements are slower (8 threads
// per line: 0.572 -> 0.632 ms/step with 16 groups per CTA, 0.722 with 28).
#ifndef SKG3_ZE128
#define SKG3_ZE128 8
#endif
#ifndef SKG3_ZE1024
#define SKG3_ZE1024 16
#endif
#ifndef SKG3_ZG1024
#define SKG3_ZG1024 1
#endif
template <int NZ>
constexpr int ze3() { return NZ == 128 ? SKG3_ZE128 : NZ == 1024 ? SKG3_ZE1024 : 8; }

template <int NZ>
struct Z3 {
    using F = BFFT<NZ, false, ze3<NZ>()>;
    static constexpr int T = F::T;
    static constexpr int G = NZ == 128                          ? SKG3_ZG128
                             : (NZ == 512 && zstage<NZ>())      ? SKG3_ZG512
                             : (NZ == 1024 && zstage<NZ>())     ? 1
                             : (NZ == 1024 && SKG3_ZG1024 != 0) ? SKG3_ZG1024
                             : T >= 256                         ? 1
                                                                : 256 / T;
    static constexpr bool STG = zstage<NZ>(), REG = zreg<NZ>();
    // resident CTAs: 2, or 6 groups per SM at 512 (168 registers)
    static constexpr int MINB = (NZ == 512 && STG)                             ? 6 / G
                                : (NZ == 1024 && STG)                          ? 3
                                : (NZ == 1024 && ze3<NZ>() == 16 && G * T >= 256) ? 1
                                                                               : 2;
    // exchange + 5 rows of doubles (cd units); staged: 3 rows when the
    // second inverse output stays in registers, + the bulk-copy stage of
    // one packed pair
    static constexpr int KZS = NZ / 2 + 1;
    static constexpr int SLOT = STG ? F::SMEM + (REG ? 3 : 5) * NZ / 2 + 2 * KZS : F::SMEM + 5 * NZ / 2;
    // + one mbarrier per group (staged variant)
    static constexpr size_t BYTES = sizeof(cd) * SLOT * G + (STG ? 16 * ((G + 1) / 2) : 0);
};

// ZB: kz_in, kz_o <= 3 NZ / 8 (dealiased states), so the row elements
// e in [3E/8, 5E/8) of every thread (|kz| in [3NZ/8, NZ/2]) are zero on input
// and not needed on output.
template <int NZ, bool ZB>
struct ZBand {
    static constexpr int E = Z3<NZ>::F::E;
    static constexpr int LO = ZB ? 3 * E / 8 : E, HI = ZB ? 5 * E / 8 : E;
};

// Raw inputs of one packed c2r (fields P, Q of a row; kept kz only).
template <int NZ, bool ZB>
__device__ __forceinline__ void fetch_pair(const Ns3dArgs& a, const cd* P, const cd* Q, size_t row,
                                           bool active, int t, cd* p, cd* q) {
    using F = typename Z3<NZ>::F;
    constexpr int T = F::T, E = F::E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZBand<NZ, ZB>::LO && e < ZBand<NZ, ZB>::HI) {
            p[e] = q[e] = zero();
            continue;
        }
        const int idx = t + T * e;
        const int ki = idx > NZ / 2 ? NZ - idx : idx;
        p[e] = zero();
        q[e] = zero();
        if (active && ki < a.kz_in) {
            p[e] = P[row + ki];
            q[e] = Q[row + ki];
        }
    }
}

// Hermitian-extended P + i Q (two c2r as one complex FFT).
template <int NZ, bool ZB>
__device__ __forceinline__ void pack_pair(int t, const cd* p, const cd* q, cd* v) {
    using F = typename Z3<NZ>::F;
    constexpr int T = F::T, E = F::E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e >= ZBand<NZ, ZB>::LO && e < ZBand<NZ, ZB>::HI) {
            v[e] = zero();
            continue;
        }
        const int idx = t + T * e;
        const bool mirror = idx > NZ / 2;
        const int ki = mirror ? NZ - idx : idx;
        cd pp = p[e], qq = q[e];
        if (ki == 0 || 2 * ki == NZ) {  // c2r ignores these imaginary parts
            pp.y = 0.0;
            qq.y = 0.0;
        }
        v[e] = mirror ? mk(pp.x + qq.y, qq.x - pp.y) : mk(pp.x - qq.y, pp.y + qq.x);
    }
}

// Separate the forward FFT Z = FT(a + i b) of two real rows into their
// half spectra, x 1/N (h = 1/(2N)), kept kz < kz_o only.  ZB: output
// k = t + T e (e < LO) pairs with NZ - k = (T - t) + T (E - 1 - e), element
// E - 1 - e of thread T - t (thread 0: its own element E - e), so each thread
// publishes its elements [HI, E) and reads its partner's.  Leaves sm free
// (ends with a barrier).
template <int NZ, bool ZB>
__device__ __forceinline__ void z_store_pair(const Ns3dArgs& a, const cd* v, cd* sm, int t, int bar,
                                             bool active, cd* o0, cd* o1, double h) {
    using F = typename Z3<NZ>::F;
    constexpr int T = F::T, E = F::E, LO = ZBand<NZ, ZB>::LO, HI = ZBand<NZ, ZB>::HI;
    if constexpr (ZB && (SKG3_Z_HERM || zherm<NZ>())) {
        static_assert(LO + HI == E, "zero band symmetric about N/2");
#pragma unroll
        for (int e = HI; e < E; ++e) sm[(e - HI) * T + t] = v[e];
        line_sync<T>(bar);
        if (active) {
            const int tp = t == 0 ? 0 : T - t;
#pragma unroll
            for (int e = 0; e < LO; ++e) {
                const int k = t + T * e;
                if (k >= a.kz_o) break;
                const cd zk = v[e];
                const cd zm = t == 0 ? (e == 0 ? v[0] : v[E - e]) : sm[(E - 1 - e - HI) * T + tp];
                st_stream(o0 + k, mk((zk.x + zm.x) * h, (zk.y - zm.y) * h));
                st_stream(o1 + k, mk((zk.y + zm.y) * h, (zm.x - zk.x) * h));
            }
        }
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) sm[F::pad(t + T * e)] = v[e];
        line_sync<T>(bar);
        if (active) {
            for (int k = t; k < a.kz_o; k += T) {
                const cd zk = sm[F::pad(k)];
                const cd zm = sm[F::pad((NZ - k) & (NZ - 1))];
                st_stream(o0 + k, mk((zk.x + zm.x) * h, (zk.y - zm.y) * h));
                st_stream(o1 + k, mk((zk.y + zm.y) * h, (zm.x - zk.x) * h));
            }
        }
    }
    line_sync<T>(bar);
}

// CFL: also reduce max |u_d| (adaptive dt, stage 1 only; a separate
// instantiation so the common path carries no extra registers).
// One tile of the z pass (G row pairs from bx).
template <int NZ, bool CFL, bool ZB>
__device__ __forceinline__ void z_tile(const Ns3dArgs& a, cd* smem, long long bx) {
    using F = typename Z3<NZ>::F;
    constexpr int T = F::T, E = F::E, G = Z3<NZ>::G;
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const long long r0 = 2ll * (bx * G + g);
    const bool active = r0 < (long long)a.nrl * a.ny;
    cd* sm = smem + g * Z3<NZ>::SLOT;
    const int bar = G > 1 ? g + 1 : 0;  // the groups' own barriers (line_sync)
    double* st = reinterpret_cast<double*>(sm + F::SMEM);  // w, wx, wy, wz, cz_a rows
    const typename F::Bases wb = F::bases(t, a.twz);
    const cd* B = a.B;
    const size_t fs = a.fstride;
    const double h = 0.5 * a.inv_n;
    // input field pairs of the three packed inverse FFTs of a row
    const cd* FP[3] = {B + 2 * fs, B + 4 * fs, B + 0 * fs};
    const cd* FQ[3] = {B + 3 * fs, B + 5 * fs, B + 1 * fs};
    if (active) {  // the row pair of all six fields into L2 up front
        const size_t bytes = sizeof(cd) * 2 * a.kz_in;
        for (int f = 0; f < 6; ++f)
            l2_prefetch(B + f * fs + (size_t)r0 * a.kz_in, bytes, t, T);
    }
    constexpr bool cfl = CFL;  // max |u_d| of the step's initial state
    double mx = 0.0, my = 0.0, mz = 0.0;
    cd p[E], q[E];
#pragma unroll 1
    for (int rr = 0; rr < 2; ++rr) {
        const size_t row = (size_t)(r0 + rr) * a.kz_in;
        cd v[E];
        // w + i wx
        fetch_pair<NZ, ZB>(a, FP[0], FQ[0], row, active, t, p, q);
        pack_pair<NZ, ZB>(t, p, q, v);
        F::template run<+1>(v, sm, t, wb, 0, bar);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            st[0 * NZ + t + T * e] = v[e].x;
            st[1 * NZ + t + T * e] = v[e].y;
        }
        // wy + i wz
        fetch_pair<NZ, ZB>(a, FP[1], FQ[1], row, active, t, p, q);
        pack_pair<NZ, ZB>(t, p, q, v);
        F::template run<+1>(v, sm, t, wb, 0, bar);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            st[2 * NZ + t + T * e] = v[e].x;
            st[3 * NZ + t + T * e] = v[e].y;
        }
        // u + i v, then the cross product (solvers.cpp:321-325)
        fetch_pair<NZ, ZB>(a, FP[2], FQ[2], row, active, t, p, q);
        pack_pair<NZ, ZB>(t, p, q, v);
        F::template run<+1>(v, sm, t, wb, 0, bar);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int y = t + T * e;
            const double ux = v[e].x, uy = v[e].y;
            const double uz = st[0 * NZ + y], ox = st[1 * NZ + y];
            if constexpr (cfl) {
                mx = fmax(mx, fabs(ux));
                my = fmax(my, fabs(uy));
                mz = fmax(mz, fabs(uz));
            }
            const double oy = st[2 * NZ + y], oz = st[3 * NZ + y];
            const double cx = uy * oz - uz * oy;
            const double cy = uz * ox - ux * oz;
            const double cz = ux * oy - uy * ox;
            v[e] = mk(cx, cy);
            st[(rr == 0 ? 4 : 0) * NZ + y] = cz;  // row b reuses the dead w row
        }
        F::template run<-1>(v, sm, t, wb, 0, bar);
        cd* o0 = a.A + (size_t)(r0 + rr) * a.kz_o;
        z_store_pair<NZ, ZB>(a, v, sm, t, bar, active, o0, o0 + fs, h);
    }
    if constexpr (cfl) umax_accumulate(a.dyn, 3, mx, my, mz);
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = mk(st[4 * NZ + t + T * e], st[0 * NZ + t + T * e]);
    F::template run<-1>(v, sm, t, wb, 0, bar);
    cd* oa = a.A + 2 * fs + (size_t)r0 * a.kz_o;
    z_store_pair<NZ, ZB>(a, v, sm, t, bar, active, oa, oa + a.kz_o, h);
}

// Staged z tile: same arithmetic as z_tile, inputs through shared memory.
template <int NZ, bool CFL, bool ZB>
__device__ __forceinline__ void z_tile_s(const Ns3dArgs& a, cd* smem, long long bx) {
    using Z = Z3<NZ>;
    using F = typename Z::F;
    constexpr int T = F::T, E = F::E, G = Z::G, KZS = Z::KZS;
    constexpr int LO = ZBand<NZ, ZB>::LO, HI = ZBand<NZ, ZB>::HI;
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const long long r0 = 2ll * (bx * G + g);
    const bool active = r0 < (long long)a.nrl * a.ny;
    cd* sm = smem + g * Z::SLOT;
    const int bar = G > 1 ? g + 1 : 0;
    double* st = reinterpret_cast<double*>(sm + F::SMEM);  // rows: w, wx, cz_a (cz_b reuses w)
    cd* stg = sm + F::SMEM + (Z::REG ? 3 : 5) * NZ / 2;  // P row, Q row of the next pair
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(smem + G * Z::SLOT) + g;
    const typename F::Bases wb = F::bases(t, a.twz);
    const cd* B = a.B;
    const size_t fs = a.fstride;
    const double h = 0.5 * a.inv_n;
    const cd* FP[3] = {B + 2 * fs, B + 4 * fs, B + 0 * fs};
    const cd* FQ[3] = {B + 3 * fs, B + 5 * fs, B + 1 * fs};
    const unsigned bytes = 16u * (unsigned)a.kz_in;
    auto issue = [&](int k) {  // packed pair k = 3 rr + pr (one thread)
        const size_t row = (size_t)(r0 + k / 3) * a.kz_in;
        mbar_expect_tx(mb, 2 * bytes);
        bulk_g2s(stg, FP[k % 3] + row, bytes, mb);
        bulk_g2s(stg + KZS, FQ[k % 3] + row, bytes, mb);
    };
    // divergence flag (cta_diverged): loaded here, checked once the first
    // bulk copy is in flight, so its round trip overlaps the copy's (the
    // wait for the first pair was 55% of the z pass's long-scoreboard
    // samples, profiles/r27)
    const int dflag = *reinterpret_cast<const volatile int*>(&a.flags->diverged);
    if (t == 0) mbar_init(mb, 1);
    line_sync<T>(bar);
    if (active && t == 0) {
        issue(0);
        const size_t rb = sizeof(cd) * 2 * a.kz_in;  // the rest of the row pair into L2
        for (int f = 0; f < 6; ++f)
            if (f != 2 && f != 3) l2_prefetch(B + f * fs + (size_t)r0 * a.kz_in, rb, 0, 1);
    }
    if (__syncthreads_or(dflag) != 0) {  // frozen state: let the copy land, then leave
        if (active) mbar_wait(mb, 0);
        return;
    }
    unsigned phase = 0;
    // packed spectrum of pair k from the stage; then the stage is released
    // and pair k + 1 requested
    auto fetch = [&](int k, cd* v) {
        if (active) mbar_wait(mb, phase);
        phase ^= 1u;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e >= LO && e < HI) {
                v[e] = zero();
                continue;
            }
            const int idx = t + T * e;
            const bool mirror = idx > NZ / 2;
            const int ki = mirror ? NZ - idx : idx;
            cd pp = zero(), qq = zero();
            if (active && ki < a.kz_in) {
                pp = stg[ki];
                qq = stg[KZS + ki];
                if (ki == 0 || 2 * ki == NZ) {  // c2r ignores these imaginary parts
                    pp.y = 0.0;
                    qq.y = 0.0;
                }
            }
            v[e] = mirror ? mk(pp.x + qq.y, qq.x - pp.y) : mk(pp.x - qq.y, pp.y + qq.x);
        }
        line_sync<T>(bar);
        if (active && t == 0 && k < 5) issue(k + 1);
    };
    constexpr bool cfl = CFL;
    double mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll 1
    for (int rr = 0; rr < 2; ++rr) {
        cd v[E];
        fetch(3 * rr, v);  // w + i wx
        F::template run<+1>(v, sm, t, wb, 0, bar);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            st[0 * NZ + t + T * e] = v[e].x;
            st[1 * NZ + t + T * e] = v[e].y;
        }
        cd w2[Z::REG ? E : 1];
        if constexpr (Z::REG) {
            fetch(3 * rr + 1, w2);  // wy + i wz, kept in registers
            F::template run<+1>(w2, sm, t, wb, 0, bar);
        } else {
            fetch(3 * rr + 1, v);  // wy + i wz
            F::template run<+1>(v, sm, t, wb, 0, bar);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                st[3 * NZ + t + T * e] = v[e].x;
                st[4 * NZ + t + T * e] = v[e].y;
            }
        }
        fetch(3 * rr + 2, v);  // u + i v, then the cross product (solvers.cpp:321-325)
        F::template run<+1>(v, sm, t, wb, 0, bar);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int y = t + T * e;
            const double ux = v[e].x, uy = v[e].y;
            const double uz = st[0 * NZ + y], ox = st[1 * NZ + y];
            if constexpr (cfl) {
                mx = fmax(mx, fabs(ux));
                my = fmax(my, fabs(uy));
                mz = fmax(mz, fabs(uz));
            }
            const double oy = Z::REG ? w2[Z::REG ? e : 0].x : st[3 * NZ + y];
            const double oz = Z::REG ? w2[Z::REG ? e : 0].y : st[4 * NZ + y];
            const double cx = uy * oz - uz * oy;
            const double cy = uz * ox - ux * oz;
            const double cz = ux * oy - uy * ox;
            v[e] = mk(cx, cy);
            st[(rr == 0 ? 2 : 0) * NZ + y] = cz;  // row b reuses the dead w row
        }
        F::template run<-1>(v, sm, t, wb, 0, bar);
        cd* o0 = a.A + (size_t)(r0 + rr) * a.kz_o;
        z_store_pair<NZ, ZB>(a, v, sm, t, bar, active, o0, o0 + fs, h);
    }
    if constexpr (cfl) umax_accumulate(a.dyn, 3, mx, my, mz);
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = mk(st[2 * NZ + t + T * e], st[0 * NZ + t + T * e]);
    F::template run<-1>(v, sm, t, wb, 0, bar);
    cd* oa = a.A + 2 * fs + (size_t)r0 * a.kz_o;
    z_store_pair<NZ, ZB>(a, v, sm, t, bar, active, oa, oa + a.kz_o, h);
}

template <int NZ, bool CFL, bool ZB>
__global__ void __launch_bounds__(Z3<NZ>::T * Z3<NZ>::G, Z3<NZ>::MINB) k3_3d(Ns3dArgs a) {
    extern __shared__ cd smem[];
    pdl_wait();
    if constexpr (Z3<NZ>::STG) {
        z_tile_s<NZ, CFL, ZB>(a, smem, blockIdx.x);  // checks the divergence flag itself
    } else {
        if (cta_diverged(a.flags)) return;
        z_tile<NZ, CFL, ZB>(a, smem, blockIdx.x);
    }
}

// ------------------------------------------------------------------ y-forward
// A/B switches (round 2).  SKG3_YF_LD = 1: one base pointer + element stride
// per thread, so the 16 input loads issue back to back instead of ~45 integer
// instructions apart (per-element 64-bit index arithmetic behind a branch).
// Measured SLOWER for this pass, the one closest to the HBM roof: 512^3
// y-forward 857 vs 790 us per launch (two runs each) -- the spread-out issue
// stays.  The same hoisting pays in the x-inverse loads/stores (1225 -> 1212),
// the y-inverse stores (2066 -> 2050) and the x-forward loads (with fewer
// spills: 1220 -> 1041).  SKG3_X4_SBASE = 1 (state index as base + e * stride in
// the x-forward epilogue): 1064 vs 1048 us (more spills), off.
#ifndef SKG3_YF_LD
#define SKG3_YF_LD 0
#endif
#ifndef SKG3_X4_SBASE
#define SKG3_X4_SBASE 0
#endif
// ZB: kcy < 3 NY / 8, so the outputs e in [3E/8, 5E/8) are masked (not stored)
// One tile of the y-forward: x row and kz block from bx, fields m0..m1.
template <int NY, int CT, bool ZB>
__device__ __forceinline__ void yf_tile(const Ns3dArgs& a, cd* smem, int bx, int m0, int m1) {
    using F = BF3<NY>;
    constexpr int T = F::T, E = F::E, C = Strided<NY, CT>::C;
    constexpr int ZLO = ZB ? 3 * E / 8 : E, ZHI = ZB ? 5 * E / 8 : E;
    const int l = threadIdx.x % C, t = threadIdx.x / C;
    const int nkzb = (a.kz_o + C - 1) / C;
    const int x = bx / nkzb;
    const int kz = (bx % nkzb) * C + l;
    const bool active = kz < a.kz_o;
    cd* sm = smem + l * F::SMEM;
    const int salt = l & 7;
    const typename F::Bases wb = F::bases(t, a.twy);
    int* loff = reinterpret_cast<int*>(smem + C * F::SMEM);
    int* lown = loff + NY;
    if (a.p2p) line_offsets_p2p<NY>(a, x, a.kz_o, loff, lown);
    else line_offsets<NY>(a, x, a.kz_o, loff);
#pragma unroll 1
    for (int m = m0; m < m1; ++m) {
        // C fields live in A's memory
        cd v[E];
#if SKG3_YF_LD
        const cd* in = a.A + m * a.fstride + ((size_t)x * a.ny + t) * a.kz_o + (active ? kz : a.kz_o - 1);
        const unsigned ist = (unsigned)T * (unsigned)a.kz_o;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = in[e * ist];
#else
        const cd* in = a.A + m * a.fstride;
#pragma unroll
        for (int e = 0; e < E; ++e)
            v[e] = active ? in[((size_t)x * a.ny + (t + T * e)) * a.kz_o + kz] : zero();
#endif
        F::template run<-1>(v, sm, t, wb, salt);
        if (active) {
            cd* out = a.slab ? a.sD + m * a.rfs
                             : a.B + m * a.fstride;  // D fields live in B's memory
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (e >= ZLO && e < ZHI) continue;
                const int lo = loff[t + T * e];
                if (lo >= 0 && abs(signed_index(t + T * e, NY)) <= a.kcy) {  // masked: never read
                    if (a.p2p) a.peer_D[lown[t + T * e]][m * a.dfs + (size_t)lo + kz] = v[e];
                    else st_stream(out + (size_t)lo + kz, v[e]);
                }
            }
        }
    }
    if (a.p2p) __threadfence_system();
}

template <int NY, int CT = 256, bool ZB = false>
__global__ void __launch_bounds__(CT, Strided<NY, CT>::MINB) k2f_3d(Ns3dArgs a) {
    extern __shared__ cd smem[];
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    // one field per CTA
    const int m0 = a.comp0 + blockIdx.y;
    yf_tile<NY, CT, ZB>(a, smem, blockIdx.x, m0, m0 + 1);
}

// ------------------------------------------------------------------ x-forward + RK
// SKG3_XSCR_HINT = 1: scratch-slot stores and loads carry an L2 evict_last
// policy (512^3 x-forward 1048 -> 1015 us per launch, step 28.58 -> 28.42 ms;
// 256^3 3.700 -> 3.695)
#ifndef SKG3_XSCR_HINT
#define SKG3_XSCR_HINT 1
#endif
__device__ __forceinline__ unsigned long long l2_keep_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_keep(cd* p, cd v, unsigned long long pol) {
#if SKG3_XSCR_HINT
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
#else
    (void)pol;
    *p = v;
#endif
}
__device__ __forceinline__ cd ld_keep(const cd* p, unsigned long long pol) {
#if SKG3_XSCR_HINT
    cd v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol) : "memory");
    return v;
#else
    (void)pol;
    return *p;
#endif
}
// The transformed components 0 and 1 wait for the projection (which needs all
// three at a mode) outside the register file: in a per-SM scratch slot of
// global memory (xscr: [component][element][thread], written and re-read by
// the same thread, fully coalesced).  A CTA claims one of its SM's slots
// through a bit mask (one atomicOr by thread 0, released at the end), so the
// ~30 MB of slots of all resident CTAs are rewritten by every wave and stay
// in L2: the raw lines never reach HBM.  The earlier in-place write-back into
// the D lines (kept as the fallback when no slot is free or SKG_NO_XSCR is
// set) wrote 2 x 0.44 F per launch to DRAM on top of the algorithmic bytes
// (512^3, ncu r08: 1.93 GB written for 0.96 GB of k_j).
// FIN: final-stage instantiation (RK update, diagnostics); the other stages
// run a leaner one that only stores k_j.
template <int NX, int CT = 256, bool FIN = false>
__global__ void __launch_bounds__(CT, Strided<NX, CT>::MINB) k4_3d(Ns3dArgs a, int stage) {
    using F = BF3<NX>;
    constexpr int T = F::T, E = F::E, C = Strided<NX, CT>::C;
    extern __shared__ cd smem[];
    const int l = threadIdx.x % C, t = threadIdx.x / C;
    const int nkzb = (a.kz_o + C - 1) / C;
    const int kyi = a.kys + blockIdx.x / nkzb;
    const int kz = (blockIdx.x % nkzb) * C + l;
    const bool active = kz < a.kz_o;
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    const int ky = ky_of(a, kyi);
    const int ys = a.slab ? kyi - a.kys : ky;
    const int sky = signed_index(ky, a.ny);
    const bool keep_y = abs(sky) <= a.kcy;
    cd* sm = smem + l * F::SMEM;
    const int salt = l & 7;
    const typename F::Bases wb = F::bases(t, a.twx);
    const bool io = active && keep_y;
    const size_t lbase = (size_t)ys * a.kz_o + kz;     // + x * ystate * kz_o
    const size_t xstr = (size_t)a.ystate * a.kz_o;
    // scratch slot of this CTA: claimed by thread 0, published after the
    // first FFT
    constexpr int CTT = T * C, PER_CTA = 2 * E * CTT;
    constexpr int NSLOT = SKG_XSCR_SM / PER_CTA < 32 ? SKG_XSCR_SM / PER_CTA : 32;
    __shared__ int s_slot;
    unsigned smid = 0;
    if (threadIdx.x == 0) {
        int slot = -1;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (a.xscr && (int)smid < a.xscr_nsm) {
            for (int k = 0; k < NSLOT && slot < 0; ++k)
                if (!(atomicOr(a.xscr_mask + smid, 1u << k) & (1u << k))) slot = k;
        }
        s_slot = slot;
    }
    // element e of this thread: D line element (t + T e) at Dm + lt + e * ls;
    // components 0 and 1 wait at P0 / P1 + e * ps (scratch slot, or in place)
    const size_t lt = lbase + (size_t)t * xstr, ls = (size_t)T * xstr;
    cd* const D = a.p2p ? a.rD : a.B;
    const size_t dstr = a.p2p ? a.dfs : a.fstride;
    cd* P0 = D + lt;
    size_t ps = ls, p1 = dstr;  // P1 = P0 + p1
    const unsigned long long pol = SKG3_XSCR_HINT ? l2_keep_policy() : 0ull;
    cd v[E];
#pragma unroll 1
    for (int m = 0; m < 3; ++m) {
        const cd* line = D + m * dstr + lt;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = io ? line[e * ls] : zero();
        F::template run<-1>(v, sm, t, wb, salt);
        if (m == 0) {
            __syncthreads();
            if (s_slot >= 0) {
                unsigned id;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
                P0 = a.xscr + (size_t)id * SKG_XSCR_SM + (size_t)s_slot * PER_CTA + threadIdx.x;
                ps = CTT;
                p1 = (size_t)E * CTT;
            }
        }
        if (m < 2 && io) {
            cd* w = m == 0 ? P0 : P0 + p1;
#pragma unroll
            for (int e = 0; e < E; ++e)  // only the kept kx are read back
                if (!a.pruned || abs(signed_index(t + T * e, NX)) <= a.kcx) st_keep(w + e * ps, v[e], pol);
        }
    }
    constexpr bool final = FIN;
    cd* kout = stage == 1 ? a.k1 : stage == 2 ? a.k2 : a.k3;
    const double kyv = a.ky_scale * (double)sky;
    const double kzv = a.kz_scale * (double)(a.kz0 + kz);
    const size_t sbase = sidx(a, t, ys, kz), sstr = (size_t)T * a.ystate * a.sz;
    int bad = 3;
    // per-step E and eps of the new state (Solver::mode_energy default,
    // simulation.cpp:163-170; dissipation_rate simulation.cpp:608-615)
    double sE = 0.0, sD = 0.0;
    const int kzg = a.kz0 + kz;  // global kz (pencil layout: kz is the local index)
    const double pw = (kzg == 0 || kzg == a.nh - 1) ? 1.0 : 2.0;
    if (final && a.diag && active && ky == 0 && kzg == 0 && t == 0) {
        for (int c = 0; c < 3; ++c) {  // mean flow: untouched, energy only
            const cd u0 = a.u[sidx(a, 0, ys, 0) + c * a.vstride];
            sE += 0.5 * pw * (u0.x * u0.x + u0.y * u0.y);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (!active) break;
        const int i = t + T * e;
        const int si = signed_index(i, NX);
        bool keep = keep_y && abs(si) <= a.kcx;
        if (i == 0 && ky == 0 && kzg == 0) keep = false;  // mean mode of the tendency is 0
        if (!keep && a.pruned) continue;
        cd c0 = zero(), c1 = zero(), c2 = zero();
        if (keep) {
            c0 = ld_keep(P0 + e * ps, pol);
            c1 = ld_keep(P0 + p1 + e * ps, pol);
            c2 = v[e];
            // Leray projection (grid.cpp:227-249)
            const double kxv = a.kx_scale * (double)si;
            const double ksq = kxv * kxv + kyv * kyv + kzv * kzv;
            if (ksq != 0.0) {
                const cd dot = add(add(scale(c0, kxv), scale(c1, kyv)), scale(c2, kzv));
                const double rk = __drcp_rn(ksq);
                const cd sp = mk(dot.x * rk, dot.y * rk);
                c0 = sub(c0, scale(sp, kxv));
                c1 = sub(c1, scale(sp, kyv));
                c2 = sub(c2, scale(sp, kzv));
            }
        }
        const cd kc[3] = {c0, c1, c2};
#if SKG3_X4_SBASE
        const size_t base = sbase + e * sstr;  // sidx(a, i, ys, kz)
#else
        const size_t base = sidx(a, i, ys, kz);
#endif
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const size_t idx = base + c * a.vstride;
            cd kv = kc[c];
            if (a.force && keep) kv = add(kv, a.force[idx]);  // forcing addend (simulation.cpp:544-547)
            if (!final) {
                st_stream(kout + idx, kv);
                continue;
            }
            const cd u = a.u[idx];
            cd un;
            if (a.has_sigma) {
                const double e1 = a.e1x[i] * a.e1y[ky] * a.e1z[kz];
                const double e2 = a.e2x[i] * a.e2y[ky] * a.e2z[kz];
                if (a.rk2) {
                    un = add(scale(u, e2), scale(kv, dt_of(a) * e1));
                } else {
                    const cd k1 = a.k1[idx], k2 = a.k2[idx], k3 = a.k3[idx];
                    const cd sum = add(add(scale(k1, e2), scale(add(k2, k3), 2.0 * e1)), kv);
                    un = add(scale(u, e2), scale(sum, sdt_of(a)));
                }
            } else {
                cd delta;
                if (a.rk2) {
                    delta = scale(kv, dt_of(a));
                } else {
                    const cd k1 = a.k1[idx], k2 = a.k2[idx], k3 = a.k3[idx];
                    delta = scale(add(add(k1, scale(add(k2, k3), 2.0)), kv), sdt_of(a));
                }
                un = (delta.x != 0.0 || delta.y != 0.0) ? add(u, delta) : u;
            }
            a.u[idx] = un;
            if (!finite2(un) && c < bad) bad = c;
            if (a.diag) {
                const double n2 = un.x * un.x + un.y * un.y;
                const double kxv = a.kx_scale * (double)si;
                const double ksq = kxv * kxv + kyv * kyv + kzv * kzv;
                sE += 0.5 * pw * n2;
                if (a.has_sigma) sD += 2.0 * a.nu * ksq * (0.5 * pw * n2);
            }
        }
    }
    if (final && a.diag) diag_accumulate(a.diag + 3 * (a.flags->steps - 1), sE, 0.0, sD);
    if (bad < 3) {
        atomicMin(&a.flags->div_var, bad);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
    __syncthreads();  // every thread has consumed its scratch values
    if (threadIdx.x == 0 && s_slot >= 0) atomicAnd(a.xscr_mask + smid, ~(1u << s_slot));
}

// Unpruned final update of the kz planes above the cut (tendency zero there).
__global__ void k4_3d_decay(Ns3dArgs a) {
    pdl_wait();
    if (cta_diverged(a.flags)) return;
    const int nk = a.nh - a.kz_o;
    const size_t total = (size_t)a.nx * a.ny * nk;
    int bad = 3;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int kz = a.kz_o + (int)(q % nk);
        const size_t r = q / nk;
        const int ky = (int)(r % a.ny);
        const int i = (int)(r / a.ny);
        const size_t base = sidx(a, i, ky, kz);
        for (int c = 0; c < 3; ++c) {
            const size_t idx = base + c * a.vstride;
            cd u = a.u[idx];
            if (a.has_sigma) {
                u = scale(u, a.e2x[i] * a.e2y[ky] * a.e2z[kz]);
                a.u[idx] = u;
            }
            if (!finite2(u) && c < bad) bad = c;
        }
    }
    if (bad < 3) {
        atomicMin(&a.flags->div_var, bad);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
}

// ------------------------------------------------------------------ launchers
template <int NX, int CT>
cudaError_t launch_x3_v(const Ns3dArgs& a, int stage, bool inverse, cudaStream_t s) {
    constexpr int C = Strided<NX, CT>::C;
    using F = BF3<NX>;
    if (inverse) {
        const dim3 grid(a.nkyl * ((a.kz_in + C - 1) / C), a.ncomp);
        const bool pz = NX >= 64 && a.pruned && a.kcx <= 3 * F::E / 8 * F::T - 1;
        if (pz) {
            if constexpr (NX >= 64) {
                const size_t smem = sizeof(cd) * (F::SMEM * C + (F::E - F::E / 4) * F::T * C);
                SKG_TRY(launch_pdl(k1_3d<NX, true, CT>, grid, F::T * C, smem, s, a, stage));
            }
        } else {
            if constexpr (CT == 256) {
                const size_t smem = sizeof(cd) * (F::SMEM * C + F::E * F::T * C);
                SKG_TRY(launch_pdl(k1_3d<NX, false>, grid, F::T * C, smem, s, a, stage));
            } else {
                return launch_x3_v<NX, 256>(a, stage, inverse, s);
            }
        }
    } else {
        const size_t smem = sizeof(cd) * F::SMEM * C;
        const int grid = a.nkyl * ((a.kz_o + C - 1) / C);
        if (a.rk2 ? stage == 2 : stage == 4) {
            SKG_TRY(launch_pdl(k4_3d<NX, CT, true>, grid, F::T * C, smem, s, a, stage));
        } else {
            SKG_TRY(launch_pdl(k4_3d<NX, CT, false>, grid, F::T * C, smem, s, a, stage));
        }
    }
    return cudaGetLastError();
}

// 128-thread CTAs (fewer kz lanes, finer kz blocks) when 256-thread CTAs
// would leave SMs idle (small grids)
// 1024-point strided passes with 512-thread CTAs (8 kz lanes: 128-byte runs
// instead of 64, one CTA per SM); bit 0 x-inverse, 1 x-forward, 2 y-inverse,
// 3 y-forward.  Measured at 1024^3 (ms per launch, 256- vs 512-thread CTAs):
// x-inverse 11.9 -> 10.9, x-forward + RK 13.0 -> 10.4, y-inverse 18.2 -> 17.7,
// y-forward 8.24 -> 8.63 (kept at 256); step 297.4 -> 282.1 ms.  (At 512^3
// the 256-thread CTAs already have 128-byte runs and 512 threads measured
// slower, DESIGN 6b.)
#ifndef SKG3_CT1024
#define SKG3_CT1024 7
#endif

template <int NX>
cudaError_t launch_x3(const Ns3dArgs& a, int stage, bool inverse, cudaStream_t s) {
    constexpr int C = Strided<NX, 256>::C;
    if constexpr (NX == 1024 && (SKG3_CT1024 & 3) != 0) {
        if (a.pruned && ((SKG3_CT1024 >> (inverse ? 0 : 1)) & 1)) return launch_x3_v<NX, 512>(a, stage, inverse, s);
    }
    if constexpr (C > 1) {
        const int kz = inverse ? a.kz_in : a.kz_o;
        if (a.nkyl * ((kz + C - 1) / C) < a.wave) return launch_x3_v<NX, 128>(a, stage, inverse, s);
    }
    return launch_x3_v<NX, 256>(a, stage, inverse, s);
}

template <int NY, int CT>
cudaError_t launch_y3_v(const Ns3dArgs& a, bool inverse, cudaStream_t s) {
    constexpr int C = Strided<NY, CT>::C;
    using F = BF3<NY>;
    const size_t smem = sizeof(cd) * F::SMEM * C + 2 * sizeof(int) * NY;  // + line offsets, owners
    const bool zb = NY >= 16 && 8 * a.kcy < 3 * NY;  // kept ky clear of the per-thread zero band
    if (inverse && a.pruned) {
        const size_t smem_s = sizeof(cd) * ((size_t)F::SMEM * C + (size_t)(2 * a.kcy + 1) * C) +
                              sizeof(int) * NY;
        // the two output halves in separate CTAs (ms/step: 64^3 0.218 -> 0.202,
        // 128^3 0.621 -> 0.600, 512^3 31.27 -> 31.20, 256^3 3.868 -> 3.888)
        const dim3 grid(a.nrl * ((a.kz_in + C - 1) / C), 2);
        if (zb) {
            SKG_TRY(launch_pdl(k2s_3d<NY, CT, true>, grid, F::T * C, smem_s, s, a));
        } else {
            SKG_TRY(launch_pdl(k2s_3d<NY, CT, false>, grid, F::T * C, smem_s, s, a));
        }
    } else if (inverse) {
        const int grid = a.nrl * ((a.kz_in + C - 1) / C);
        SKG_TRY(launch_pdl(k2_3d<NY, CT>, grid, F::T * C, smem, s, a));
    } else {
        const dim3 grid(a.nrl * ((a.kz_o + C - 1) / C), a.ncomp);
        if (zb) {
            SKG_TRY(launch_pdl(k2f_3d<NY, CT, true>, grid, F::T * C, smem, s, a));
        } else {
            SKG_TRY(launch_pdl(k2f_3d<NY, CT, false>, grid, F::T * C, smem, s, a));
        }
    }
    return cudaGetLastError();
}

template <int NY>
cudaError_t launch_y3(const Ns3dArgs& a, bool inverse, cudaStream_t s) {
    constexpr int C = Strided<NY, 256>::C;
    if constexpr (NY == 1024 && (SKG3_CT1024 & 12) != 0) {
        if (a.pruned && ((SKG3_CT1024 >> (inverse ? 2 : 3)) & 1)) return launch_y3_v<NY, 512>(a, inverse, s);
    }
    if constexpr (C > 1) {
        const int kz = inverse ? a.kz_in : a.kz_o;
        if (a.nrl * ((kz + C - 1) / C) < a.wave) return launch_y3_v<NY, 128>(a, inverse, s);
    }
    return launch_y3_v<NY, 256>(a, inverse, s);
}

template <int NZ>
cudaError_t launch_z3(const Ns3dArgs& a, cudaStream_t s) {
    using Z = Z3<NZ>;
    const size_t smem = Z::BYTES;
    const long long pairs = (long long)a.nrl * a.ny / 2;
    const int grid = (int)((pairs + Z::G - 1) / Z::G);
    // zero band (dealiased states): kept kz of both directions below 3 NZ / 8
    const bool zb = NZ >= 16 && 8 * a.kz_in <= 3 * NZ && 8 * a.kz_o <= 3 * NZ;
    if (zb) {
        if constexpr (NZ >= 16) {
            if (a.dyn && a.ystage == 1) {
                SKG_TRY(launch_pdl(k3_3d<NZ, true, true>, grid, Z::T * Z::G, smem, s, a));
            } else {
                SKG_TRY(launch_pdl(k3_3d<NZ, false, true>, grid, Z::T * Z::G, smem, s, a));
            }
        }
    } else if (a.dyn && a.ystage == 1) {
        SKG_TRY(launch_pdl(k3_3d<NZ, true, false>, grid, Z::T * Z::G, smem, s, a));
    } else {
        SKG_TRY(launch_pdl(k3_3d<NZ, false, false>, grid, Z::T * Z::G, smem, s, a));
    }
    return cudaGetLastError();
}


#define SKG3_CASES(X) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

cudaError_t dispatch_x3(const Ns3dArgs& a, int stage, bool inverse, cudaStream_t s) {
    switch (a.nx) {
#define CASE(N) \
    case N: return launch_x3<N>(a, stage, inverse, s);
        SKG3_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t dispatch_y3(const Ns3dArgs& a, bool inverse, cudaStream_t s) {
    switch (a.ny) {
#define CASE(N) \
    case N: return launch_y3<N>(a, inverse, s);
        SKG3_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t dispatch_z3(const Ns3dArgs& a, cudaStream_t s) {
    switch (a.nz) {
#define CASE(N) \
    case N: return launch_z3<N>(a, s);
        SKG3_CASES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

bool ns3d_supported(int nx, int ny, int nz) {
    auto ok = [](int n) { return n >= 8 && n <= 1024 && (n & (n - 1)) == 0; };
    return ok(nx) && ok(ny) && ok(nz);
}

cudaError_t ns3d_pass(const Ns3dArgs& a, int pass, int stage, cudaStream_t s, long* launches,
                      const LaunchHook& hook) {
    // Bytes models use this rank's share: nkyl kept lines (x passes) and
    // nrl x rows (y/z passes); G = 1 gives the whole grid.
    cudaError_t err;
    const double B = sizeof(cd);
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    const double kyk = a.pruned ? 2.0 * a.kcy + 1 : (double)a.ny;  // ky read by k2
    const double kxk = a.pruned ? 2.0 * a.kcx + 1 : (double)a.nx;
    const double lines_in = (double)a.nkyl * a.kz_in;
    const double lines_o = (double)a.nkyl * a.kz_o;
    const double plane_in = (double)a.nrl * a.ny * a.kz_in;
    const double plane_o = (double)a.nrl * a.ny * a.kz_o;
    if (pass == 0) {
        // component c reads v_c (and k_c) and writes X[v_c] (+ X[kx v_c] for c > 0)
        const double nin = a.ncomp, nout = a.ncomp == 3 ? 5.0 : (a.comp0 == 0 ? 1.0 : 2.0) * a.ncomp;
        hook.begin(0);
        if ((err = dispatch_x3(a, stage, true, s)) != cudaSuccess) return err;
        hook.end(0, B * (nin * kxk * lines_in * (stage == 1 ? 1.0 : 2.0) + nout * a.nx * lines_in));
        *launches += 1;
    } else if (pass == 1 || pass == 3 || pass == 4 || pass == 5 || pass == 6) {
        // 1: y-inverse, z, y-forward; 3: y-inverse, z; 4: y-forward; pencil
        // layout: 5: y-inverse only, 6: z pass only
        Ns3dArgs b = a;  // the z pass of stage 1 feeds the CFL max
        b.ystage = stage;
        if (pass != 4) {
            if (pass != 6) {
                hook.begin(3);
                if ((err = dispatch_y3(a, true, s)) != cudaSuccess) return err;
                hook.end(3, B * (5.0 * a.nrl * kyk * a.kz_in + 6.0 * plane_in));
                *launches += 1;
            }
            if (pass != 5) {
                hook.begin(1);
                if ((err = dispatch_z3(b, s)) != cudaSuccess) return err;
                hook.end(1, B * (6.0 * plane_in + 3.0 * plane_o));
                *launches += 1;
            }
        }
        if (pass == 1 || pass == 4) {
            const double nf = pass == 4 ? a.ncomp : 3.0;
            hook.begin(5);
            if ((err = dispatch_y3(a, false, s)) != cudaSuccess) return err;
            hook.end(5, B * nf * (plane_o + a.nrl * kyk * a.kz_o));
            *launches += 1;
        }
    } else {
        hook.begin(2);
        if ((err = dispatch_x3(a, stage, false, s)) != cudaSuccess) return err;
        hook.end(2, B * (3.0 * a.nx * lines_o +
                         3.0 * kxk * lines_o * (final ? (a.rk2 ? 3.0 : 5.0) : 1.0)));
        *launches += 1;
        if (final && !a.pruned && a.nh > a.kz_o) {
            hook.begin(3);
            SKG_TRY(launch_pdl(k4_3d_decay, 592, 256, 0, s, a));
            hook.end(3, B * 6.0 * a.nx * a.ny * (a.nh - a.kz_o));
            *launches += 1;
            if ((err = cudaGetLastError()) != cudaSuccess) return err;
        }
    }
    return cudaSuccess;
}

cudaError_t ns3d_launch_stage(const Ns3dArgs& a, int stage, cudaStream_t s, long* launches,
                              const LaunchHook& hook) {
    cudaError_t err;
    for (int pass = 0; pass < 3; ++pass)
        if ((err = ns3d_pass(a, pass, stage, s, launches, hook)) != cudaSuccess) return err;
    return cudaSuccess;
}

}  // namespace skg
