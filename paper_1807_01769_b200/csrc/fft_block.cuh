// fft_block.cuh -- register-resident FP64 Stockham FFT for one line per
// thread group, exchanging through shared memory between radix passes.
//
// Replaces the FFTW execution behind FftPlan (reference proj/src/fft.cpp:92-106)
// on the hot path.  Layout contract ("natural"): a line of N complex values is
// held by T = N/E threads, thread t owning elements t + T*e, e in [0, E).
// Every pass reads natural order from registers, and the last pass leaves the
// result in natural order in registers, so the caller loads inputs and stores
// outputs fully coalesced and fuses its prologue/epilogue arithmetic there.
//
// Pass p (radix R, Ns = product of earlier radices), butterfly j in [0, N/R):
//   u[r] = x[j + r N/R] * W_{Ns R}^{(j mod Ns) r}      (skip when Ns == 1)
//   u    = DFT_R(u)
//   y[(j / Ns) Ns R + (j mod Ns) + r Ns] = u[r]          (to smem, autosort)
// Radix 16 (4x4 in registers) until the remainder is < 16, then 2/4/8, so a
// 4096-point line costs 3 register passes and 2 shared-memory exchanges.
// Twiddles W_N^m come from a per-length table built on the host in extended
// precision (forward sign; the inverse uses the conjugate).
#pragma once
#include <cuda_runtime.h>

namespace skg {

typedef double2 cd;

__device__ __forceinline__ cd mk(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ cd add(cd a, cd b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cd sub(cd a, cd b) { return mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cd mul(cd a, cd b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ cd mulconj(cd a, cd b) {  // a * conj(b)
    return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ cd conj(cd a) { return mk(a.x, -a.y); }
__device__ __forceinline__ cd scale(cd a, double s) { return mk(a.x * s, a.y * s); }
__device__ __forceinline__ cd muli(cd a) { return mk(-a.y, a.x); }   // i * a
__device__ __forceinline__ cd mulmi(cd a) { return mk(a.y, -a.x); }  // -i * a
__device__ __forceinline__ cd zero() { return mk(0.0, 0.0); }

// S = -1 forward (e^{-i}), S = +1 inverse (e^{+i}).
template <int S>
__device__ __forceinline__ cd rot90(cd a) {  // a * W_4^1 = a * (S i)
    return S < 0 ? mulmi(a) : muli(a);
}

constexpr double kC8 = 0.70710678118654752440084436210484904;   // cos(pi/4)
constexpr double kC16 = 0.92387953251128675612818318939678829;  // cos(pi/8)
constexpr double kS16 = 0.38268343236508977172845837907404220;  // sin(pi/8)

// a * W_R^M with W_R = e^{S 2 pi i / R}; constant-folded special cases.
template <int S, int M, int R>
__device__ __forceinline__ cd twc(cd a) {
    constexpr int m = ((M % R) + R) % R;
    if constexpr (m == 0) return a;
    else if constexpr (4 * m == R) return rot90<S>(a);
    else if constexpr (2 * m == R) return mk(-a.x, -a.y);
    else if constexpr (4 * m == 3 * R) return rot90<-S>(a);
    else if constexpr (8 * m == R) {  // (1 + S i)/sqrt2
        return S < 0 ? mk((a.x + a.y) * kC8, (a.y - a.x) * kC8)
                     : mk((a.x - a.y) * kC8, (a.y + a.x) * kC8);
    } else if constexpr (8 * m == 3 * R) {  // (-1 + S i)/sqrt2
        return S < 0 ? mk((a.y - a.x) * kC8, -(a.x + a.y) * kC8)
                     : mk(-(a.x + a.y) * kC8, (a.x - a.y) * kC8);
    } else if constexpr (8 * m == 5 * R) {  // (-1 - S i)/sqrt2
        return S < 0 ? mk(-(a.x + a.y) * kC8, (a.x - a.y) * kC8)
                     : mk((a.y - a.x) * kC8, -(a.x + a.y) * kC8);
    } else if constexpr (8 * m == 7 * R) {  // (1 - S i)/sqrt2
        return S < 0 ? mk((a.x - a.y) * kC8, (a.y + a.x) * kC8)
                     : mk((a.x + a.y) * kC8, (a.y - a.x) * kC8);
    } else {
        static_assert(R == 16, "general twiddle only for radix 16");
        // m in {1,3,5,7,9,11,13,15}: cos/sin of 2 pi m / 16
        constexpr double c = (m == 1 || m == 15) ? kC16
                             : (m == 3 || m == 13) ? kS16
                             : (m == 5 || m == 11) ? -kS16
                                                   : -kC16;
        constexpr double s0 = (m == 1 || m == 7) ? kS16
                              : (m == 3 || m == 5) ? kC16
                              : (m == 9 || m == 15) ? -kS16
                                                    : -kC16;
        constexpr double s = S * s0;
        return mk(a.x * c - a.y * s, a.x * s + a.y * c);
    }
}

template <int S>
__device__ __forceinline__ void dft2(cd& a, cd& b) {
    cd t = a;
    a = add(t, b);
    b = sub(t, b);
}

template <int S>
__device__ __forceinline__ void dft4(cd& x0, cd& x1, cd& x2, cd& x3) {
    cd a = add(x0, x2), b = sub(x0, x2), c = add(x1, x3), d = rot90<S>(sub(x1, x3));
    x0 = add(a, c);
    x2 = sub(a, c);
    x1 = add(b, d);
    x3 = sub(b, d);
}

// Natural order in, natural order out.
template <int S>
__device__ __forceinline__ void dft8(cd* x) {
    // n = 2 n1 + n2 (n1 < 4, n2 < 2); k = k1 + 4 k2
    dft4<S>(x[0], x[2], x[4], x[6]);
    dft4<S>(x[1], x[3], x[5], x[7]);
    // y[n2][k1] at x[2 k1 + n2]; twiddle W_8^{n2 k1}
    x[3] = twc<S, 1, 8>(x[3]);
    x[5] = twc<S, 2, 8>(x[5]);
    x[7] = twc<S, 3, 8>(x[7]);
    cd o[8];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        cd a = x[2 * k1], b = x[2 * k1 + 1];
        o[k1] = add(a, b);
        o[k1 + 4] = sub(a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = o[i];
}

template <int S>
__device__ __forceinline__ void dft16(cd* x) {
    // n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<S>(x[n2], x[4 + n2], x[8 + n2], x[12 + n2]);
    // y[n2][k1] stored at x[4 k1 + n2]; twiddle W_16^{n2 k1}
    x[5] = twc<S, 1, 16>(x[5]);
    x[6] = twc<S, 2, 16>(x[6]);
    x[7] = twc<S, 3, 16>(x[7]);
    x[9] = twc<S, 2, 16>(x[9]);
    x[10] = twc<S, 4, 16>(x[10]);
    x[11] = twc<S, 6, 16>(x[11]);
    x[13] = twc<S, 3, 16>(x[13]);
    x[14] = twc<S, 6, 16>(x[14]);
    x[15] = twc<S, 9, 16>(x[15]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<S>(x[4 * k1], x[4 * k1 + 1], x[4 * k1 + 2], x[4 * k1 + 3]);
    // X[k1 + 4 k2] now at x[4 k1 + k2]
    cd o[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) o[k1 + 4 * k2] = x[4 * k1 + k2];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = o[i];
}

template <int R, int S>
__device__ __forceinline__ void dft(cd* x) {
    if constexpr (R == 1) {
    } else if constexpr (R == 2) dft2<S>(x[0], x[1]);
    else if constexpr (R == 4) dft4<S>(x[0], x[1], x[2], x[3]);
    else if constexpr (R == 8) dft8<S>(x);
    else if constexpr (R == 16) dft16<S>(x);
    else static_assert(R == 16, "unsupported radix");
}

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }

// u[r] *= w^r, r = 1..R-1, where w = W_N^m (forward sign) from the table and
// the direction S conjugates it.  Powers are generated in registers so a pass
// issues one table load per butterfly instead of R-1.  Radix 16 uses the
// 4x4 split w^(4 n1 + n2) = (w^4)^n1 w^n2 to keep few powers live.
template <int S, int R>
__device__ __forceinline__ void apply_twiddles(cd* u, cd w) {
    if constexpr (S > 0) w = conj(w);
    if constexpr (R == 2) {
        u[1] = mul(u[1], w);
    } else if constexpr (R == 4) {
        const cd w2 = mul(w, w);
        u[1] = mul(u[1], w);
        u[2] = mul(u[2], w2);
        u[3] = mul(u[3], mul(w2, w));
    } else if constexpr (R == 8) {
        const cd w2 = mul(w, w);
        const cd w3 = mul(w2, w);
        const cd w4 = mul(w2, w2);
        u[1] = mul(u[1], w);
        u[2] = mul(u[2], w2);
        u[3] = mul(u[3], w3);
        u[4] = mul(u[4], w4);
        u[5] = mul(u[5], mul(w4, w));
        u[6] = mul(u[6], mul(w4, w2));
        u[7] = mul(u[7], mul(w4, w3));
    } else {
        static_assert(R == 16, "radix");
        const cd w2 = mul(w, w);
        const cd w3 = mul(w2, w);
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) {
            u[4 * n1 + 1] = mul(u[4 * n1 + 1], w);
            u[4 * n1 + 2] = mul(u[4 * n1 + 2], w2);
            u[4 * n1 + 3] = mul(u[4 * n1 + 3], w3);
        }
        const cd w4 = mul(w2, w2);
        const cd w8 = mul(w4, w4);
        const cd w12 = mul(w8, w4);
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
            u[4 + n2] = mul(u[4 + n2], w4);
            u[8 + n2] = mul(u[8 + n2], w8);
            u[12 + n2] = mul(u[12 + n2], w12);
        }
    }
}

// Barrier of the threads that share one exchange buffer: the whole CTA
// (bar == 0); otherwise only this line's T threads -- a named barrier
// (bar = 1..15, T a multiple of 32) or the T-lane slice of one warp (T < 32)
// -- so independent lines of one CTA do not wait for each other.
template <int T>
__device__ __forceinline__ void line_sync(int bar) {
#if defined(__CUDA_ARCH__)
    if (bar == 0) {
        __syncthreads();
    } else if constexpr (T == 32) {
        __syncwarp();
    } else if constexpr (T > 32) {
        asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(T) : "memory");
    } else {
        const unsigned lane = threadIdx.x & 31u;
        __syncwarp(((1u << T) - 1u) << (lane & ~(unsigned)(T - 1)));
    }
#else
    (void)bar;  // host emulation (tests/host_emu): one barrier domain
    __syncthreads();
#endif
}

// Block FFT of a power-of-two length N in natural layout.  SPLIT exchanges
// the real and imaginary parts in two rounds through an N-double buffer
// (half the shared memory, twice the barriers).
template <int N, bool SPLIT = false, int EMAX = 16>
struct BFFT {
    static_assert((N & (N - 1)) == 0 && N >= 2, "power-of-two length");
    static_assert(EMAX == 4 || EMAX == 8 || EMAX == 16, "4, 8 or 16 elements per thread");
    static constexpr int E = N < EMAX ? N : EMAX;  // elements per thread
    static constexpr int T = N / E;            // threads per line
    static constexpr int SH = ilog2c(E);
    // Exchange buffer: N slots, XOR-swizzled on the 16-byte slot within each
    // 128-byte line so the stride-E writes of the first pass and the
    // unit-stride reads are both conflict-free (no padding).
    static constexpr int SMEM = SPLIT ? (N + 1) / 2 : N;  // in cd (16-byte) units
    __device__ __forceinline__ static int pad(int i) {
        if constexpr (E >= 4) return i ^ ((i >> SH) & 7);
        else return i;
    }
    // 8-byte slots: XOR the slot within each 128-byte line.
    __device__ __forceinline__ static int pad8(int i) {
        if constexpr (E >= 16) return i ^ ((i >> 4) & 15);
        else if constexpr (E == 8) return i ^ ((i >> 4) & 7);
        else return i;
    }

    static constexpr int npasses() {
        int p = 0;
        for (int ns = 1; ns < N; ns *= (N / ns >= E ? E : N / ns)) ++p;
        return p;
    }
    static constexpr int NP = npasses();

    // Per-thread twiddle bases, one per pass after the first:
    // w[p] = W_N^{(t mod Ns_p) * N / (Ns_p R_p)}.  Loaded once per kernel so
    // no global load sits between a barrier and the butterflies.
    struct Bases {
        cd w[NP > 1 ? NP - 1 : 1];
    };
    __device__ __forceinline__ static Bases bases(int t, const cd* __restrict__ tw) {
        Bases b;
        int ns = 1;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int R = N / ns >= E ? E : N / ns;
            if (p > 0) b.w[p - 1] = __ldg(&tw[(t & (ns - 1)) * (N / (ns * R))]);
            ns *= R;
        }
        return b;
    }

    // w * W_E^q (forward sign), q a compile-time constant after unrolling.
    template <int Q>
    __device__ __forceinline__ static cd twq(cd w) {
        if constexpr (Q == 0) return w;
        else return twc<-1, Q, E>(w);
    }
    __device__ __forceinline__ static cd twc_e(cd w, int b) {
        cd r = w;
#define SKG_TWQ(Q) \
    if constexpr (Q < E) {  \
        if (b == Q) r = twq<Q>(w); \
    }
        SKG_TWQ(1) SKG_TWQ(2) SKG_TWQ(3) SKG_TWQ(4) SKG_TWQ(5) SKG_TWQ(6) SKG_TWQ(7)
        SKG_TWQ(8) SKG_TWQ(9) SKG_TWQ(10) SKG_TWQ(11) SKG_TWQ(12) SKG_TWQ(13) SKG_TWQ(14)
        SKG_TWQ(15)
#undef SKG_TWQ
        return r;
    }

    // One pass, then recurse.
    // salt (0..7) is XORed into the 16-byte slot index: lines interleaved
    // lane-by-lane in one warp (strided-axis kernels) then hit distinct banks.
    template <int S, int Ns, int P>
    __device__ __forceinline__ static void pass(cd* v, cd* sm, int t, const Bases& wb, int salt,
                                                int bar) {
        constexpr int rem = N / Ns;
        constexpr int R = rem >= E ? E : rem;
        constexpr int B = E / R;  // butterflies per thread in this pass (> 1 only in the last)
        constexpr bool last = (Ns * R == N);
        static_assert(E % R == 0, "radix must divide elements per thread");
        static_assert(B == 1 || last, "multi-butterfly passes only at the end");
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int j = t + T * b;
            cd u[R];
#pragma unroll
            for (int r = 0; r < R; ++r) u[r] = v[b + r * B];
            const int jm = j & (Ns - 1);
            if constexpr (Ns > 1) {
                // last pass: W_N^{t + T b} = W_N^t W_E^b (step 1, jm = j)
                const cd w = b > 0 ? twc_e(wb.w[P - 1], b) : wb.w[P - 1];
                apply_twiddles<S, R>(u, w);
            }
            dft<R, S>(u);
            if constexpr (last || SPLIT) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[b + r * B] = u[r];
            } else {
                const int base = (j / Ns) * Ns * R + jm;
#pragma unroll
                for (int r = 0; r < R; ++r) sm[pad(base + r * Ns) ^ salt] = u[r];
            }
        }
        if constexpr (!last) {
            if constexpr (SPLIT) {
                // B == 1 here: element r goes to base + r Ns
                double* sd = reinterpret_cast<double*>(sm);
                const int base = (t / Ns) * Ns * R + (t & (Ns - 1));
#pragma unroll
                for (int r = 0; r < R; ++r) sd[pad8(base + r * Ns)] = v[r].x;
                line_sync<T>(bar);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e].x = sd[pad8(t + T * e)];
                line_sync<T>(bar);
#pragma unroll
                for (int r = 0; r < R; ++r) sd[pad8(base + r * Ns)] = v[r].y;
                line_sync<T>(bar);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e].y = sd[pad8(t + T * e)];
                line_sync<T>(bar);
            } else {
                line_sync<T>(bar);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = sm[pad(t + T * e) ^ salt];
                line_sync<T>(bar);
            }
            pass<S, Ns * R, P + 1>(v, sm, t, wb, salt, bar);
        }
    }

    // bar: 0 = CTA-wide barriers; otherwise this line's own (line_sync)
    template <int S>
    __device__ __forceinline__ static void run(cd* v, cd* sm, int t, const Bases& wb, int salt = 0,
                                               int bar = 0) {
        pass<S, 1, 0>(v, sm, t, wb, salt, bar);
    }
    template <int S>
    __device__ __forceinline__ static void run(cd* v, cd* sm, int t, const cd* __restrict__ tw,
                                               int salt = 0, int bar = 0) {
        pass<S, 1, 0>(v, sm, t, bases(t, tw), salt, bar);
    }
};

}  // namespace skg
