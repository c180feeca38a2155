/*
 * oracle/fft_shim.c -- CPU FFT behind the FFTW-3 API subset of oracle/fftw3.h.
 *
 * TEST INFRASTRUCTURE ONLY.  This file lets the reference's own transform
 * layer (proj/src/fft.cpp:56-106) link without FFTW3, which is absent from
 * the image and not vendored under /root/reference (proj/CMakeLists.txt:19-21,
 * README.md:22 "FFTW3 (double precision)", version unpinned).  It restates the
 * published FFTW transform definitions the reference relies on:
 *   - r2c: X[k] = sum_j x[j] exp(-2 pi i j.k / n), last axis stored 0..n/2,
 *     unnormalised (the reference applies 1/N itself, fft.cpp:92-98);
 *   - c2r: x[j] = sum over the Hermitian extension of X exp(+2 pi i j.k / n),
 *     unnormalised; computed as c2c along the leading axes followed by a
 *     last-axis c2r that uses only the real part of the index-0 and Nyquist
 *     entries; the input may be clobbered (FFTW semantics, fft.cpp:100-106);
 *   - plans never retain the planning buffers (fft.cpp:75-82) and execute on
 *     arbitrary unaligned pointers.
 * Algorithm: recursive mixed-radix decimation-in-time (radix 4/2/3/5 kernels,
 * direct DFT for other factors), r2c/c2r via the half-length complex FFT,
 * OpenMP over independent lines when fftw_plan_with_nthreads(n > 1).
 * Pinned by tests/test_oracle.py against direct summation (the reference's
 * test_fft.cpp:18-50 oracle) and against numpy.fft.
 */
#include "fftw3.h"

#define _USE_MATH_DEFINES
#include <math.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdlib.h>
#include <string.h>

typedef struct {
    double re, im;
} cpx;

static inline cpx cmul(cpx a, cpx b) {
    cpx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}
static inline cpx cadd(cpx a, cpx b) {
    cpx r = {a.re + b.re, a.im + b.im};
    return r;
}
static inline cpx csub(cpx a, cpx b) {
    cpx r = {a.re - b.re, a.im - b.im};
    return r;
}

/* ------------------------------------------------------------ 1D c2c plan */

typedef struct {
    int n;
    int sign; /* -1 forward, +1 backward */
    int nfac;
    int fac[64];
    cpx* w; /* w[j] = exp(sign 2 pi i j / n), j in [0, n) */
} cplan;

static cpx unit_root(long j, long n, int sign) {
    /* Accurate exp(sign 2 pi i j/n): reduce to the first octant. */
    j %= n;
    if (j < 0) j += n;
    /* angle = 2 pi j / n; use symmetry around quarter turns */
    long q4 = 4 * j; /* multiples of n/4 */
    double c, s;
    long quad = q4 / n;
    long rem4 = q4 - quad * n; /* in [0, n) -> angle within quadrant = 2 pi rem4/(4n) */
    double a = (2.0 * M_PI) * (double)rem4 / (4.0 * (double)n);
    double ca = cos(a), sa = sin(a);
    switch (quad) {
        case 0: c = ca; s = sa; break;
        case 1: c = -sa; s = ca; break;
        case 2: c = -ca; s = -sa; break;
        default: c = sa; s = -ca; break;
    }
    cpx r = {c, sign * s};
    return r;
}

static void cplan_init(cplan* p, int n, int sign) {
    p->n = n;
    p->sign = sign;
    p->nfac = 0;
    int m = n;
    while (m % 4 == 0) { p->fac[p->nfac++] = 4; m /= 4; }
    while (m % 2 == 0) { p->fac[p->nfac++] = 2; m /= 2; }
    for (int f = 3; m > 1; f += 2) {
        while (m % f == 0) { p->fac[p->nfac++] = f; m /= f; }
        if (f * f > m && m > 1) { p->fac[p->nfac++] = m; m = 1; }
    }
    p->w = (cpx*)malloc(sizeof(cpx) * (size_t)(n > 0 ? n : 1));
    for (int j = 0; j < n; ++j) p->w[j] = unit_root(j, n, sign);
}

static void cplan_free(cplan* p) { free(p->w); p->w = NULL; }

/* out[0..n) = DFT_n(in[0], in[s], ...); factors fac[0..nf) multiply to n.
 * W is the top-level table of length N; sub-length n uses stride N/n. */
static void cfft_rec(const cpx* in, long s, cpx* out, int n, const int* fac, int nf,
                     const cpx* W, int N) {
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    int r = fac[0];
    int m = n / r;
    for (int q = 0; q < r; ++q) cfft_rec(in + q * s, s * r, out + q * m, m, fac + 1, nf - 1, W, N);
    long wstep = N / n; /* W_n^e = W[e * wstep] */
    if (r == 2) {
        for (int k = 0; k < m; ++k) {
            cpx t0 = out[k];
            cpx t1 = cmul(out[m + k], W[(long)k * wstep]);
            out[k] = cadd(t0, t1);
            out[k + m] = csub(t0, t1);
        }
    } else if (r == 4) {
        const double sg = (double)((W[N / 4].im > 0) ? 1 : -1); /* W_4 = sg*i */
        for (int k = 0; k < m; ++k) {
            cpx t0 = out[k];
            cpx t1 = cmul(out[m + k], W[((long)k * wstep) % N]);
            cpx t2 = cmul(out[2 * m + k], W[((long)2 * k * wstep) % N]);
            cpx t3 = cmul(out[3 * m + k], W[((long)3 * k * wstep) % N]);
            cpx a = cadd(t0, t2), b = csub(t0, t2), c = cadd(t1, t3), d = csub(t1, t3);
            cpx id = {-sg * d.im, sg * d.re}; /* (sg i) * d */
            out[k] = cadd(a, c);
            out[k + m] = cadd(b, id);
            out[k + 2 * m] = csub(a, c);
            out[k + 3 * m] = csub(b, id);
        }
    } else {
        cpx t[64];
        cpx* tt = r <= 64 ? t : (cpx*)malloc(sizeof(cpx) * (size_t)r);
        long rstep = N / r; /* W_r^e */
        for (int k = 0; k < m; ++k) {
            for (int q = 0; q < r; ++q) tt[q] = cmul(out[q * m + k], W[((long)q * k * wstep) % N]);
            for (int sidx = 0; sidx < r; ++sidx) {
                cpx acc = tt[0];
                for (int q = 1; q < r; ++q)
                    acc = cadd(acc, cmul(tt[q], W[(((long)q * sidx) % r) * rstep]));
                out[k + sidx * m] = acc;
            }
        }
        if (tt != t) free(tt);
    }
}

static void cplan_exec(const cplan* p, const cpx* in, long s, cpx* out) {
    cfft_rec(in, s, out, p->n, p->fac, p->nfac, p->w, p->n);
}

/* --------------------------------------------------------- real-axis plan */

typedef struct {
    int n;        /* real length (even) */
    cplan half;   /* length n/2 complex, sign as the direction */
    cpx* tw;      /* tw[k] = exp(sign 2 pi i k / n), k in [0, n/2] */
} rplan;

static void rplan_init(rplan* p, int n, int sign) {
    p->n = n;
    cplan_init(&p->half, n / 2, sign);
    p->tw = (cpx*)malloc(sizeof(cpx) * (size_t)(n / 2 + 1));
    for (int k = 0; k <= n / 2; ++k) p->tw[k] = unit_root(k, n, sign);
}

static void rplan_free(rplan* p) {
    cplan_free(&p->half);
    free(p->tw);
}

/* r2c: x real length n -> X[0..n/2]; scratch has 2*(n/2) cpx. */
static void r2c_1d(const rplan* p, const double* x, cpx* X, cpx* scratch) {
    int h = p->n / 2;
    cpx* z = scratch;
    cpx* Z = scratch + h;
    for (int j = 0; j < h; ++j) {
        z[j].re = x[2 * j];
        z[j].im = x[2 * j + 1];
    }
    cplan_exec(&p->half, z, 1, Z);
    for (int k = 0; k <= h; ++k) {
        cpx a = Z[k % h];
        cpx b = Z[(h - k) % h];
        cpx bc = {b.re, -b.im};
        cpx e = {0.5 * (a.re + bc.re), 0.5 * (a.im + bc.im)}; /* even part */
        cpx o = {0.5 * (a.re - bc.re), 0.5 * (a.im - bc.im)}; /* i * odd part */
        /* odd = -i * o */
        cpx od = {o.im, -o.re};
        X[k] = cadd(e, cmul(p->tw[k], od));
    }
}

/* c2r: X[0..n/2] -> x real length n (unnormalised); imag of X[0], X[n/2] ignored. */
static void c2r_1d(const rplan* p, const cpx* Xin, double* x, cpx* scratch) {
    int h = p->n / 2;
    cpx* Z = scratch;
    cpx* z = scratch + h;
    for (int k = 0; k < h; ++k) {
        cpx a = Xin[k];
        cpx b = Xin[h - k];
        if (k == 0) {
            a.im = 0.0;
            b.im = 0.0;
        }
        cpx bc = {b.re, -b.im};
        cpx E = cadd(a, bc);
        cpx O = cmul(csub(a, bc), p->tw[k]);
        cpx iO = {-O.im, O.re};
        Z[k] = cadd(E, iO);
    }
    cplan_exec(&p->half, Z, 1, z);
    for (int j = 0; j < h; ++j) {
        x[2 * j] = z[j].re;
        x[2 * j + 1] = z[j].im;
    }
}

/* ----------------------------------------------------------- nd plans */

struct sk_shim_plan {
    int r2c; /* 1 = r2c (forward), 0 = c2r (backward) */
    int rank;
    int n[3];
    int h;           /* n[rank-1]/2 + 1 */
    int nthreads;
    rplan last;
    cplan axis[2];   /* leading axes */
};

static int g_nthreads = 1;

int fftw_init_threads(void) { return 1; }

void fftw_plan_with_nthreads(int nthreads) { g_nthreads = nthreads < 1 ? 1 : nthreads; }

static fftw_plan make_plan(int rank, const int* n, int r2c) {
    if (rank < 1 || rank > 3) return NULL;
    for (int d = 0; d < rank; ++d)
        if (n[d] < 2 || (d == rank - 1 && n[d] % 2 != 0)) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    p->r2c = r2c;
    p->rank = rank;
    for (int d = 0; d < rank; ++d) p->n[d] = n[d];
    p->h = n[rank - 1] / 2 + 1;
    p->nthreads = g_nthreads;
    int sign = r2c ? -1 : 1;
    rplan_init(&p->last, n[rank - 1], sign);
    for (int d = 0; d < rank - 1; ++d) cplan_init(&p->axis[d], n[d], sign);
    return p;
}

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out,
                            unsigned flags) {
    (void)in;
    (void)out;
    (void)flags;
    return make_plan(rank, n, 1);
}

fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out,
                            unsigned flags) {
    (void)in;
    (void)out;
    (void)flags;
    return make_plan(rank, n, 0);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    rplan_free(&p->last);
    for (int d = 0; d < p->rank - 1; ++d) cplan_free(&p->axis[d]);
    free(p);
}

/* c2c along leading axis `a` of the complex array with shape
 * (n[0], .., n[rank-2], h), in place, lines batched through a gather buffer. */
#define SK_BATCH 8
static void c2c_axis(const fftw_plan p, cpx* data, int a) {
    long len = p->n[a];
    long inner = p->h;
    for (int d = a + 1; d < p->rank - 1; ++d) inner *= p->n[d];
    long outer = 1;
    for (int d = 0; d < a; ++d) outer *= p->n[d];
    long nbatch_in = (inner + SK_BATCH - 1) / SK_BATCH;
    long total = outer * nbatch_in;
    const cplan* cp = &p->axis[a];
#pragma omp parallel num_threads(p->nthreads)
    {
        cpx* buf = (cpx*)malloc(sizeof(cpx) * (size_t)(2 * len * SK_BATCH));
        cpx* res = buf + len * SK_BATCH;
#pragma omp for schedule(static)
        for (long t = 0; t < total; ++t) {
            long o = t / nbatch_in;
            long i0 = (t % nbatch_in) * SK_BATCH;
            int nb = (int)((inner - i0) < SK_BATCH ? (inner - i0) : SK_BATCH);
            cpx* base = data + o * len * inner + i0;
            for (long j = 0; j < len; ++j)
                for (int b = 0; b < nb; ++b) buf[b * len + j] = base[j * inner + b];
            for (int b = 0; b < nb; ++b) cplan_exec(cp, buf + b * len, 1, res + b * len);
            for (long j = 0; j < len; ++j)
                for (int b = 0; b < nb; ++b) base[j * inner + b] = res[b * len + j];
        }
        free(buf);
    }
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
    long rows = 1;
    for (int d = 0; d < p->rank - 1; ++d) rows *= p->n[d];
    long nl = p->n[p->rank - 1];
    cpx* X = (cpx*)out;
#pragma omp parallel num_threads(p->nthreads)
    {
        cpx* scratch = (cpx*)malloc(sizeof(cpx) * (size_t)(nl + 2));
#pragma omp for schedule(static)
        for (long r = 0; r < rows; ++r) r2c_1d(&p->last, in + r * nl, X + r * p->h, scratch);
        free(scratch);
    }
    for (int a = p->rank - 2; a >= 0; --a) c2c_axis(p, X, a);
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
    cpx* X = (cpx*)in; /* clobbered, as FFTW's multi-dimensional c2r may do */
    for (int a = 0; a <= p->rank - 2; ++a) c2c_axis(p, X, a);
    long rows = 1;
    for (int d = 0; d < p->rank - 1; ++d) rows *= p->n[d];
    long nl = p->n[p->rank - 1];
#pragma omp parallel num_threads(p->nthreads)
    {
        cpx* scratch = (cpx*)malloc(sizeof(cpx) * (size_t)(nl + 2));
#pragma omp for schedule(static)
        for (long r = 0; r < rows; ++r) c2r_1d(&p->last, X + r * p->h, out + r * nl, scratch);
        free(scratch);
    }
}
