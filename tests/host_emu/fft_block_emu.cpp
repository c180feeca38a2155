// Host emulation of paper_1807_01769_b200/csrc/fft_block.cuh (test-only).
// One FFT line, T std::threads, a std::barrier standing in for __syncthreads,
// so the exact device index/twiddle/exchange logic runs on the CPU.
// Usage: fft_block_emu <N> <sign> [mode]  mode bit0: split exchange, bit1: 8 per thread   reads N complex (re im) from stdin,
// writes the transform to stdout.
#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

struct double2 {
    double x, y;
};
inline double2 make_double2(double x, double y) { return {x, y}; }
#define __device__
#define __host__
#define __forceinline__ inline
#define __restrict__
static thread_local std::barrier<>* g_bar;
inline void __syncthreads() { g_bar->arrive_and_wait(); }
template <class T>
inline T __ldg(const T* p) { return *p; }
#include FFT_BLOCK_HEADER

using namespace skg;

template <int N, int S, bool SPLIT, int EM>
void run_line(std::vector<cd>& x) {
    using F = BFFT<N, SPLIT, EM>;
    std::vector<cd> tw(N);
    for (int m = 0; m < N; ++m) {
        long double a = 6.283185307179586476925286766559005768L * m / N;
        tw[m] = make_double2((double)cosl(a), (double)-sinl(a));
    }
    std::vector<cd> sm(F::SMEM);
    std::barrier<> bar(F::T);
    std::vector<std::thread> th;
    for (int t = 0; t < F::T; ++t)
        th.emplace_back([&, t] {
            g_bar = &bar;
            cd v[F::E];
            for (int e = 0; e < F::E; ++e) v[e] = x[t + F::T * e];
            F::template run<S>(v, sm.data(), t, tw.data());
            bar.arrive_and_wait();
            for (int e = 0; e < F::E; ++e) x[t + F::T * e] = v[e];
        });
    for (auto& h : th) h.join();
}

template <int N>
void go(int sign, int split) {
    std::vector<cd> x(N);
    for (auto& c : x)
        if (std::scanf("%lf %lf", &c.x, &c.y) != 2) std::exit(2);
    const bool sp = split & 1, e8 = split & 2;
    if (e8) {
        if (sp) sign < 0 ? run_line<N, -1, true, 8>(x) : run_line<N, 1, true, 8>(x);
        else sign < 0 ? run_line<N, -1, false, 8>(x) : run_line<N, 1, false, 8>(x);
    } else {
        if (sp) sign < 0 ? run_line<N, -1, true, 16>(x) : run_line<N, 1, true, 16>(x);
        else sign < 0 ? run_line<N, -1, false, 16>(x) : run_line<N, 1, false, 16>(x);
    }
    for (auto& c : x) std::printf("%.17g %.17g\n", c.x, c.y);
}

int main(int argc, char** argv) {
    int n = std::atoi(argv[1]), s = std::atoi(argv[2]), sp = argc > 3 ? std::atoi(argv[3]) : 0;
    switch (n) {
        case 4: go<4>(s, sp); break;
        case 8: go<8>(s, sp); break;
        case 16: go<16>(s, sp); break;
        case 32: go<32>(s, sp); break;
        case 64: go<64>(s, sp); break;
        case 128: go<128>(s, sp); break;
        case 256: go<256>(s, sp); break;
        case 512: go<512>(s, sp); break;
        case 1024: go<1024>(s, sp); break;
        case 2048: go<2048>(s, sp); break;
        case 4096: go<4096>(s, sp); break;
        default: return 3;
    }
    return 0;
}
