// fft_ops.cu -- the transform operators FftPlan::forward / FftPlan::inverse
// (reference proj/src/fft.cpp:92-106) on the device, for any rank-1..3 shape
// with even extents (fft.cpp:34-44).
//
// forward: r2c along the last axis (two real rows packed into one complex
//          FFT), c2c along the leading axes, then *= 1/N (fft.cpp:96-97);
// inverse: c2c along the leading axes on a copy (the input stays intact,
//          fft.cpp:100-106), then c2r rows (two rows packed), dropping the
//          imaginary parts of the last-axis index-0 and Nyquist entries.
// Power-of-two extents use the register Stockham FFT of fft_block.cuh; other
// extents up to 4096 use Bluestein's chirp convolution on that FFT, larger
// ones a direct O(n^2) line DFT in shared memory (still on the GPU).
#include <cmath>
#include <complex>
#include <map>
#include <mutex>
#include <vector>

#include "skg_internal.h"

namespace skg {

namespace {

// -------------------------------------------------- power-of-two lines
// c2c along one axis of a [outer][N][inner] complex array, in place.
template <int N, int S>
__global__ void __launch_bounds__(BFFT<N>::T > 256 ? BFFT<N>::T : 256) c2c_axis_tw(cd* data, long long outer, long long inner,
                                                   const cd* __restrict__ tw) {
    using F = BFFT<N>;
    constexpr int T = F::T, E = F::E;
    constexpr int LPC = T >= 256 ? 1 : 256 / T;
    extern __shared__ cd smem[];
    const int l = threadIdx.x / T, t = threadIdx.x % T;
    const long long line = (long long)blockIdx.x * LPC + l;
    const bool active = line < outer * inner;
    const long long o = active ? line / inner : 0, i = active ? line % inner : 0;
    cd* base = data + o * N * inner + i;
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? base[(long long)(t + T * e) * inner] : zero();
    F::template run<S>(v, smem + l * F::SMEM, t, tw);
    if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) base[(long long)(t + T * e) * inner] = v[e];
    }
}

// r2c of real rows of length N, two rows per thread group; out rows N/2+1.
template <int N>
__global__ void __launch_bounds__(BFFT<N>::T > 256 ? BFFT<N>::T : 256) r2c_rows(const double* __restrict__ u, cd* __restrict__ out,
                                                long long rows, const cd* __restrict__ tw) {
    using F = BFFT<N>;
    constexpr int T = F::T, E = F::E;
    constexpr int G = T >= 256 ? 1 : 256 / T;
    constexpr int H = N / 2 + 1;
    extern __shared__ cd smem[];
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const long long ra = 2 * ((long long)blockIdx.x * G + g), rb = ra + 1;
    cd* sm = smem + g * F::SMEM;
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int idx = t + T * e;
        const double a = ra < rows ? u[ra * N + idx] : 0.0;
        const double b = rb < rows ? u[rb * N + idx] : 0.0;
        v[e] = mk(a, b);
    }
    F::template run<-1>(v, sm, t, tw);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) sm[F::pad(t + T * e)] = v[e];
    __syncthreads();
    for (int k = t; k < H; k += T) {
        cd zk = sm[F::pad(k)];
        cd zm = sm[F::pad((N - k) & (N - 1))];
        if (ra < rows) out[ra * H + k] = mk(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        if (rb < rows) out[rb * H + k] = mk(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    }
}

// c2r of half rows (N/2+1) into real rows of length N, two rows per group.
template <int N>
__global__ void __launch_bounds__(BFFT<N>::T > 256 ? BFFT<N>::T : 256) c2r_rows(const cd* __restrict__ in, double* __restrict__ u,
                                                long long rows, const cd* __restrict__ tw) {
    using F = BFFT<N>;
    constexpr int T = F::T, E = F::E;
    constexpr int G = T >= 256 ? 1 : 256 / T;
    constexpr int H = N / 2 + 1;
    extern __shared__ cd smem[];
    const int g = threadIdx.x / T, t = threadIdx.x % T;
    const long long ra = 2 * ((long long)blockIdx.x * G + g), rb = ra + 1;
    cd* sm = smem + g * F::SMEM;
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int idx = t + T * e;
        const bool mirror = idx > N / 2;
        const int ki = mirror ? N - idx : idx;
        cd ah = ra < rows ? in[ra * H + ki] : zero();
        cd bh = rb < rows ? in[rb * H + ki] : zero();
        if (ki == 0 || 2 * ki == N) {
            ah.y = 0.0;
            bh.y = 0.0;
        }
        v[e] = mirror ? mk(ah.x + bh.y, bh.x - ah.y) : mk(ah.x - bh.y, ah.y + bh.x);
    }
    F::template run<+1>(v, sm, t, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int idx = t + T * e;
        if (ra < rows) u[ra * N + idx] = v[e].x;
        if (rb < rows) u[rb * N + idx] = v[e].y;
    }
}

// -------------------------------------------------- generic (any even n)
// Direct DFT of one line per block: X[k] = sum_j x[j] W^{jk}, W from tw (len n).
__global__ void dft_axis_generic(cd* data, long long outer, int n, long long inner, int sign,
                                 const cd* __restrict__ tw) {
    extern __shared__ cd line[];
    const long long lid = blockIdx.x;
    const long long o = lid / inner, i = lid % inner;
    cd* base = data + o * n * inner + i;
    for (int j = threadIdx.x; j < n; j += blockDim.x) line[j] = base[(long long)j * inner];
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        cd acc = zero();
        for (int j = 0; j < n; ++j) {
            cd w = tw[(int)(((long long)j * k) % n)];
            if (sign > 0) w = conj(w);
            acc = add(acc, mul(line[j], w));
        }
        base[(long long)k * inner] = acc;
    }
}

__global__ void dft_r2c_generic(const double* u, cd* out, int n, const cd* __restrict__ tw) {
    extern __shared__ double rline[];
    const long long r = blockIdx.x;
    const int h = n / 2 + 1;
    for (int j = threadIdx.x; j < n; j += blockDim.x) rline[j] = u[r * n + j];
    __syncthreads();
    for (int k = threadIdx.x; k < h; k += blockDim.x) {
        cd acc = zero();
        for (int j = 0; j < n; ++j) {
            cd w = tw[(int)(((long long)j * k) % n)];
            acc = add(acc, scale(w, rline[j]));
        }
        out[r * h + k] = acc;
    }
}

__global__ void dft_c2r_generic(const cd* in, double* u, int n, const cd* __restrict__ tw) {
    extern __shared__ cd hline[];
    const long long r = blockIdx.x;
    const int h = n / 2 + 1;
    for (int k = threadIdx.x; k < h; k += blockDim.x) hline[k] = in[r * h + k];
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double acc = hline[0].x;
        acc += ((j & 1) ? -1.0 : 1.0) * hline[n / 2].x;
        double s = 0.0;
        for (int k = 1; k < n / 2; ++k) {
            cd w = conj(tw[(int)(((long long)j * k) % n)]);
            s += hline[k].x * w.x - hline[k].y * w.y;
        }
        u[r * n + j] = acc + 2.0 * s;
    }
}

// -------------------------------------------------- Bluestein (any n <= 4096)
// X_k = c_k sum_j (x_j c_j) conj(c_{k-j}),  c_j = exp(s i pi j^2 / n): the
// convolution runs as two power-of-two register FFTs of length M >= 2n - 1
// (one CTA per line), against the precomputed spectrum of the conj(c) chirp.
struct BlueTab {
    int M = 0;
    cd* chirp[2] = {nullptr, nullptr};  // [sign < 0, sign > 0], n entries
    cd* bhat[2] = {nullptr, nullptr};   // M entries
    cd* twm = nullptr;                  // W_M table for the register FFT
};

// mode 0: c2c along an axis of [outer][n][inner] (in place);
// 1: r2c of real rows (n) into half rows (n/2+1); 2: c2r of half rows.
template <int M, int S>
__global__ void __launch_bounds__(BFFT<M>::T) bluestein_line(cd* data, long long inner, int n, int mode,
                                                             const double* ureal, double* ureal_out,
                                                             const cd* __restrict__ chirp,
                                                             const cd* __restrict__ bhat,
                                                             const cd* __restrict__ twm) {
    using F = BFFT<M>;
    constexpr int T = F::T, E = F::E;
    extern __shared__ cd smem[];
    const int t = threadIdx.x;
    const long long line = blockIdx.x;
    const int h = n / 2 + 1;
    cd* base = nullptr;
    if (mode == 0) base = data + (line / inner) * n * inner + (line % inner);
    const typename F::Bases wb = F::bases(t, twm);
    cd v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int j = t + T * e;
        cd x = zero();
        if (j < n) {
            if (mode == 0) {
                x = base[(long long)j * inner];
            } else if (mode == 1) {
                x = mk(ureal[line * n + j], 0.0);
            } else {  // Hermitian extension; c2r ignores Im of the DC/Nyquist entries
                const int k = j <= n / 2 ? j : n - j;
                x = data[line * h + k];
                if (k == 0 || 2 * k == n) x.y = 0.0;
                if (j > n / 2) x = conj(x);
            }
            x = mul(x, chirp[j]);
        }
        v[e] = x;
    }
    F::template run<-1>(v, smem, t, wb);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = mul(v[e], bhat[t + T * e]);
    F::template run<+1>(v, smem, t, wb);
    const double im = 1.0 / (double)M;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int k = t + T * e;
        if (k >= n) continue;
        const cd X = scale(mul(v[e], chirp[k]), im);
        if (mode == 0) base[(long long)k * inner] = X;
        else if (mode == 1) { if (k < h) data[line * h + k] = X; }
        else ureal_out[line * n + k] = X.x;
    }
}

std::mutex g_blue_mu;
std::map<std::pair<int, int>, BlueTab> g_blue;

// Tables for length n on the current device (built once, before any graph
// capture: the first step of a batch runs eagerly).
const BlueTab* blue_tab(int n) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_blue_mu);
    auto key = std::make_pair(dev, n);
    auto it = g_blue.find(key);
    if (it != g_blue.end()) return &it->second;
    int M = 16;
    while (M < 2 * n - 1) M *= 2;
    if (M > 8192) return nullptr;
    const long double pi = 3.141592653589793238462643383279502884L;
    BlueTab tb;
    tb.M = M;
    std::vector<cd> wm(M);
    for (int m = 0; m < M; ++m) {
        const long double a = -2.0L * pi * (long double)m / (long double)M;
        wm[m] = make_double2((double)cosl(a), (double)sinl(a));
    }
    for (int si = 0; si < 2; ++si) {
        const long double sg = si == 0 ? -1.0L : 1.0L;
        std::vector<std::complex<long double>> c(n);
        for (int j = 0; j < n; ++j) {
            const long long j2 = ((long long)j * j) % (2LL * n);  // exact angle reduction
            const long double a = sg * pi * (long double)j2 / (long double)n;
            c[j] = std::complex<long double>(cosl(a), sinl(a));
        }
        // b_m = conj(c_|m|) wrapped onto [0, M); bhat = FFT_M(b), exact sums
        std::vector<cd> ch(n), bh(M);
        for (int j = 0; j < n; ++j) ch[j] = make_double2((double)c[j].real(), (double)c[j].imag());
        std::vector<std::complex<long double>> wml(M);
        for (int m = 0; m < M; ++m) {
            const long double a = -2.0L * pi * (long double)m / (long double)M;
            wml[m] = std::complex<long double>(cosl(a), sinl(a));
        }
        for (int q = 0; q < M; ++q) {
            std::complex<long double> acc = std::conj(c[0]);
            for (int m = 1; m < n; ++m) {
                const std::complex<long double> b = std::conj(c[m]);
                acc += b * (wml[(int)(((long long)q * m) % M)] + wml[(int)(((long long)q * (M - m)) % M)]);
            }
            bh[q] = make_double2((double)acc.real(), (double)acc.imag());
        }
        skg::dmalloc(&tb.chirp[si], sizeof(cd) * n);
        skg::dmalloc(&tb.bhat[si], sizeof(cd) * M);
        cudaMemcpy(tb.chirp[si], ch.data(), sizeof(cd) * n, cudaMemcpyHostToDevice);
        cudaMemcpy(tb.bhat[si], bh.data(), sizeof(cd) * M, cudaMemcpyHostToDevice);
    }
    skg::dmalloc(&tb.twm, sizeof(cd) * M);
    cudaMemcpy(tb.twm, wm.data(), sizeof(cd) * M, cudaMemcpyHostToDevice);
    return &(g_blue[key] = tb);
}

template <int M>
cudaError_t launch_blue_m(const BlueTab& tb, int si, cd* data, long long lines, long long inner, int n,
                          int mode, const double* ur, double* uo, cudaStream_t s) {
    using F = BFFT<M>;
    const size_t smem = sizeof(cd) * F::SMEM;
    SKG_TRY(si == 0 ? ensure_smem(reinterpret_cast<const void*>(bluestein_line<M, -1>), smem)
                    : ensure_smem(reinterpret_cast<const void*>(bluestein_line<M, 1>), smem));
    if (si == 0)
        bluestein_line<M, -1><<<(unsigned)lines, F::T, smem, s>>>(data, inner, n, mode, ur, uo,
                                                                  tb.chirp[0], tb.bhat[0], tb.twm);
    else
        bluestein_line<M, 1><<<(unsigned)lines, F::T, smem, s>>>(data, inner, n, mode, ur, uo,
                                                                 tb.chirp[1], tb.bhat[1], tb.twm);
    return cudaGetLastError();
}

// false when n needs M > 8192 (caller falls back to the direct DFT)
bool bluestein(int n, int sign, cd* data, long long lines, long long inner, int mode, const double* ur,
               double* uo, cudaStream_t s, cudaError_t* err) {
    const BlueTab* tb = blue_tab(n);
    if (!tb) return false;
    const int si = sign < 0 ? 0 : 1;
    switch (tb->M) {
#define BCASE(M) \
    case M: *err = launch_blue_m<M>(*tb, si, data, lines, inner, n, mode, ur, uo, s); return true;
        BCASE(16) BCASE(32) BCASE(64) BCASE(128) BCASE(256) BCASE(512) BCASE(1024) BCASE(2048)
        BCASE(4096) BCASE(8192)
#undef BCASE
        default: return false;
    }
}

__global__ void scale_kernel(cd* d, long long n, double s) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x)
        d[q] = scale(d[q], s);
}

template <int N, int S>
cudaError_t launch_c2c(cd* data, long long outer, long long inner, const cd* tw, cudaStream_t s) {
    using F = BFFT<N>;
    constexpr int LPC = F::T >= 256 ? 1 : 256 / F::T;
    const size_t smem = sizeof(cd) * F::SMEM * LPC;
    SKG_TRY(ensure_smem(reinterpret_cast<const void*>(c2c_axis_tw<N, S>), smem));
    const long long lines = outer * inner;
    c2c_axis_tw<N, S><<<(unsigned)((lines + LPC - 1) / LPC), F::T * LPC, smem, s>>>(data, outer, inner, tw);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_r2c(const double* u, cd* out, long long rows, const cd* tw, cudaStream_t s) {
    using F = BFFT<N>;
    constexpr int G = F::T >= 256 ? 1 : 256 / F::T;
    const size_t smem = sizeof(cd) * F::SMEM * G;
    SKG_TRY(ensure_smem(reinterpret_cast<const void*>(r2c_rows<N>), smem));
    const long long pairs = (rows + 1) / 2;
    r2c_rows<N><<<(unsigned)((pairs + G - 1) / G), F::T * G, smem, s>>>(u, out, rows, tw);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_c2r(const cd* in, double* u, long long rows, const cd* tw, cudaStream_t s) {
    using F = BFFT<N>;
    constexpr int G = F::T >= 256 ? 1 : 256 / F::T;
    const size_t smem = sizeof(cd) * F::SMEM * G;
    SKG_TRY(ensure_smem(reinterpret_cast<const void*>(c2r_rows<N>), smem));
    const long long pairs = (rows + 1) / 2;
    c2r_rows<N><<<(unsigned)((pairs + G - 1) / G), F::T * G, smem, s>>>(in, u, rows, tw);
    return cudaGetLastError();
}

#define SKG_POW2_CASES(X) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

cudaError_t c2c(cd* data, long long outer, int n, long long inner, int sign, const cd* tw,
                cudaStream_t s) {
    switch (n) {
#define CASE(N) \
    case N: return sign < 0 ? launch_c2c<N, -1>(data, outer, inner, tw, s) : launch_c2c<N, 1>(data, outer, inner, tw, s);
        SKG_POW2_CASES(CASE)
#undef CASE
        default: {
            const long long lines = outer * inner;
            cudaError_t e = cudaSuccess;
            if (bluestein(n, sign, data, lines, inner, 0, nullptr, nullptr, s, &e)) return e;
            SKG_TRY(ensure_smem(reinterpret_cast<const void*>(dft_axis_generic), sizeof(cd) * n));
            dft_axis_generic<<<(unsigned)lines, 128, sizeof(cd) * n, s>>>(data, outer, n, inner, sign, tw);
            return cudaGetLastError();
        }
    }
}

cudaError_t r2c(const double* u, cd* out, long long rows, int n, const cd* tw, cudaStream_t s) {
    switch (n) {
#define CASE(N) \
    case N: return launch_r2c<N>(u, out, rows, tw, s);
        SKG_POW2_CASES(CASE)
#undef CASE
        default: {
            cudaError_t e = cudaSuccess;
            if (bluestein(n, -1, out, rows, 1, 1, u, nullptr, s, &e)) return e;
            SKG_TRY(ensure_smem(reinterpret_cast<const void*>(dft_r2c_generic), sizeof(double) * n));
            dft_r2c_generic<<<(unsigned)rows, 128, sizeof(double) * n, s>>>(u, out, n, tw);
            return cudaGetLastError();
        }
    }
}

cudaError_t c2r(const cd* in, double* u, long long rows, int n, const cd* tw, cudaStream_t s) {
    switch (n) {
#define CASE(N) \
    case N: return launch_c2r<N>(in, u, rows, tw, s);
        SKG_POW2_CASES(CASE)
#undef CASE
        default: {
            cudaError_t e = cudaSuccess;
            if (bluestein(n, 1, const_cast<cd*>(in), rows, 1, 2, nullptr, u, s, &e)) return e;
            SKG_TRY(ensure_smem(reinterpret_cast<const void*>(dft_c2r_generic), sizeof(cd) * (n / 2 + 1)));
            dft_c2r_generic<<<(unsigned)rows, 128, sizeof(cd) * (n / 2 + 1), s>>>(in, u, n, tw);
            return cudaGetLastError();
        }
    }
}

}  // namespace

bool fft_pow2(int n) { return n >= 4 && n <= 8192 && (n & (n - 1)) == 0; }

cudaError_t fft_forward_dev(int rank, const int* n, const double* d_u, cd* d_uhat, cd*,
                            const cd* const* tw, cudaStream_t s, long* launches, bool normalize) {
    long long rows = 1, P = 1;
    for (int d = 0; d < rank - 1; ++d) rows *= n[d];
    for (int d = 0; d < rank; ++d) P *= n[d];
    const int nl = n[rank - 1];
    const int h = nl / 2 + 1;
    cudaError_t err = r2c(d_u, d_uhat, rows, nl, tw[rank - 1], s);
    ++*launches;
    if (err != cudaSuccess) return err;
    for (int a = rank - 2; a >= 0; --a) {
        long long outer = 1, inner = h;
        for (int d = 0; d < a; ++d) outer *= n[d];
        for (int d = a + 1; d < rank - 1; ++d) inner *= n[d];
        if ((err = c2c(d_uhat, outer, n[a], inner, -1, tw[a], s)) != cudaSuccess) return err;
        ++*launches;
    }
    if (!normalize) return cudaSuccess;  // FFTW convention (fftw_execute_dft_r2c)
    scale_kernel<<<592, 256, 0, s>>>(d_uhat, rows * h, 1.0 / (double)P);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t fft_inverse_dev(int rank, const int* n, const cd* d_uhat, double* d_u, cd* d_work,
                            const cd* const* tw, cudaStream_t s, long* launches) {
    long long rows = 1;
    for (int d = 0; d < rank - 1; ++d) rows *= n[d];
    const int nl = n[rank - 1];
    const int h = nl / 2 + 1;
    cudaError_t err = cudaMemcpyAsync(d_work, d_uhat, sizeof(cd) * rows * h, cudaMemcpyDeviceToDevice, s);
    if (err != cudaSuccess) return err;
    for (int a = 0; a <= rank - 2; ++a) {
        long long outer = 1, inner = h;
        for (int d = 0; d < a; ++d) outer *= n[d];
        for (int d = a + 1; d < rank - 1; ++d) inner *= n[d];
        if ((err = c2c(d_work, outer, n[a], inner, +1, tw[a], s)) != cudaSuccess) return err;
        ++*launches;
    }
    err = c2r(d_work, d_u, rows, nl, tw[rank - 1], s);
    ++*launches;
    return err;
}

}  // namespace skg
