// integration/fftw_gpu.cpp -- a GPU-backed libfftw3 for the reference's
// UNMODIFIED transform layer.  FftPlan (proj/src/fft.cpp)
// calls exactly these 9 FFTW-3 symbols (fft.cpp:67-104); linking the
// reference against this file instead of libfftw3 runs every FftPlan::forward
// / inverse on the B200 through skg_dft_r2c / skg_dft_c2r (include/skgpu.h).
//
// Reference-side glue a maintainer would add (not part of the product path):
// plans only record the shape, execute copies the caller's host arrays to
// the device and back (the reference keeps its fields on the host).
#include <cstdio>
#include <cstdlib>

#include "skgpu.h"

extern "C" {

typedef double fftw_complex[2];

struct skg_fftw_plan {
    int rank;
    int n[3];
};
typedef skg_fftw_plan* fftw_plan;

static int g_device = 0;

int fftw_init_threads(void) {
    const char* d = std::getenv("SKG_FFTW_DEVICE");
    g_device = d ? std::atoi(d) : 0;
    return 1;
}

void fftw_plan_with_nthreads(int) {}

static fftw_plan make_plan(int rank, const int* n) {
    if (rank < 1 || rank > 3) return nullptr;  // FftPlan throws on a NULL plan (fft.cpp:83)
    auto* p = new skg_fftw_plan{rank, {1, 1, 1}};
    for (int d = 0; d < rank; ++d) p->n[d] = n[d];
    return p;
}

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double*, fftw_complex*, unsigned) {
    return make_plan(rank, n);  // the planning arrays are not retained (fft.cpp:75-82)
}

fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex*, double*, unsigned) {
    return make_plan(rank, n);
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
    if (skg_dft_r2c(p->rank, p->n, in, reinterpret_cast<double*>(out), g_device) != SKG_OK) {
        std::fprintf(stderr, "fftw_gpu: %s\n", skg_last_error());
        std::abort();
    }
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
    if (skg_dft_c2r(p->rank, p->n, reinterpret_cast<const double*>(in), out, g_device) != SKG_OK) {
        std::fprintf(stderr, "fftw_gpu: %s\n", skg_last_error());
        std::abort();
    }
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
