/*
 * oracle/fftw3.h -- FFTW-3 API subset used by the reference transform layer.
 *
 * TEST INFRASTRUCTURE ONLY (part of the CPU oracle).  FFTW3 itself is not in
 * this image and not under /root/reference; the reference links it through
 * `find_library(FFTW3_LIB NAMES fftw3 REQUIRED)` (proj/CMakeLists.txt:19-21,
 * unpinned).  This header declares exactly the symbols the reference calls
 * (proj/src/fft.cpp:3-106) so that proj/src/ sources compile unmodified against
 * oracle/fft_shim.c, a restatement of FFTW's published transform definitions
 * (unnormalised DFT, forward sign -1, r2c/c2r halved last axis).
 */
#ifndef SK_ORACLE_FFTW3_H
#define SK_ORACLE_FFTW3_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct sk_shim_plan* fftw_plan;

#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

int fftw_init_threads(void);
void fftw_plan_with_nthreads(int nthreads);

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out,
                            unsigned flags);
fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out,
                            unsigned flags);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
