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
 * Algorithm: power-of-two lengths run a batched Stockham autosort FFT
 * (radix 4, one radix-2 pass for odd log2 n) over SK_B lines at a time in
 * split re/im work buffers, the batch index innermost so every butterfly
 * loop is a unit-stride SIMD loop; other lengths use a recursive
 * mixed-radix decimation-in-time FFT (radix 4/2/3/5 kernels, direct DFT for
 * other factors).  r2c/c2r via the half-length complex FFT; OpenMP over
 * batches of independent lines when fftw_plan_with_nthreads(n > 1).
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


/* ------------------------------------------- batched power-of-two c2c (SoA) */

#define SK_B 8 /* lines per batch: the SIMD (innermost) dimension */

typedef struct {
    int n;      /* power of two, >= 1 */
    int sign;
    double* wr; /* W_n^j = exp(sign 2 pi i j / n), j in [0, n) */
    double* wi;
} p2plan;

static int is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

static void p2plan_init(p2plan* p, int n, int sign) {
    p->n = n;
    p->sign = sign;
    p->wr = (double*)malloc(sizeof(double) * (size_t)n);
    p->wi = (double*)malloc(sizeof(double) * (size_t)n);
    for (int j = 0; j < n; ++j) {
        cpx w = unit_root(j, n, sign);
        p->wr[j] = w.re;
        p->wi[j] = w.im;
    }
}

static void p2plan_free(p2plan* p) {
    free(p->wr);
    free(p->wi);
    p->wr = p->wi = NULL;
}

/* One Stockham pass of radix R in {2, 4}: for butterfly j in [0, n/R),
 * k = j mod Ns: u_r = x[j + r n/R] W_{Ns R}^{k r}; u = DFT_R(u);
 * y[(j / Ns) Ns R + k + r Ns] = u_r.  Element e of line b lives at e*SK_B + b. */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void p2_pass(const p2plan* p, int R, int Ns, const double* restrict xr, const double* restrict xi,
                    double* restrict yr, double* restrict yi) {
    const int n = p->n, q = n / R;
    const int tstep = n / (Ns * R); /* W_{Ns R}^m = W_n^{m tstep} */
    const double sg = (double)p->sign;
    for (int j = 0; j < q; ++j) {
        const int k = j & (Ns - 1);
        const int ob = (j - k) * R + k;
        if (R == 2) {
            const double w1r = p->wr[k * tstep], w1i = p->wi[k * tstep];
            const double* ar = xr + (size_t)j * SK_B;
            const double* ai = xi + (size_t)j * SK_B;
            const double* br = xr + (size_t)(j + q) * SK_B;
            const double* bi = xi + (size_t)(j + q) * SK_B;
            double* o0r = yr + (size_t)ob * SK_B;
            double* o0i = yi + (size_t)ob * SK_B;
            double* o1r = yr + (size_t)(ob + Ns) * SK_B;
            double* o1i = yi + (size_t)(ob + Ns) * SK_B;
#pragma omp simd
            for (int b = 0; b < SK_B; ++b) {
                const double tr = br[b] * w1r - bi[b] * w1i;
                const double ti = br[b] * w1i + bi[b] * w1r;
                o0r[b] = ar[b] + tr;
                o0i[b] = ai[b] + ti;
                o1r[b] = ar[b] - tr;
                o1i[b] = ai[b] - ti;
            }
        } else {
            const double w1r = p->wr[k * tstep], w1i = p->wi[k * tstep];
            const double w2r = p->wr[2 * k * tstep], w2i = p->wi[2 * k * tstep];
            const double w3r = p->wr[3 * k * tstep], w3i = p->wi[3 * k * tstep];
            const double* x0r = xr + (size_t)j * SK_B;
            const double* x0i = xi + (size_t)j * SK_B;
            const double* x1r = xr + (size_t)(j + q) * SK_B;
            const double* x1i = xi + (size_t)(j + q) * SK_B;
            const double* x2r = xr + (size_t)(j + 2 * q) * SK_B;
            const double* x2i = xi + (size_t)(j + 2 * q) * SK_B;
            const double* x3r = xr + (size_t)(j + 3 * q) * SK_B;
            const double* x3i = xi + (size_t)(j + 3 * q) * SK_B;
            double* y0r = yr + (size_t)ob * SK_B;
            double* y0i = yi + (size_t)ob * SK_B;
            double* y1r = yr + (size_t)(ob + Ns) * SK_B;
            double* y1i = yi + (size_t)(ob + Ns) * SK_B;
            double* y2r = yr + (size_t)(ob + 2 * Ns) * SK_B;
            double* y2i = yi + (size_t)(ob + 2 * Ns) * SK_B;
            double* y3r = yr + (size_t)(ob + 3 * Ns) * SK_B;
            double* y3i = yi + (size_t)(ob + 3 * Ns) * SK_B;
#pragma omp simd
            for (int b = 0; b < SK_B; ++b) {
                const double u0r = x0r[b], u0i = x0i[b];
                const double u1r = x1r[b] * w1r - x1i[b] * w1i, u1i = x1r[b] * w1i + x1i[b] * w1r;
                const double u2r = x2r[b] * w2r - x2i[b] * w2i, u2i = x2r[b] * w2i + x2i[b] * w2r;
                const double u3r = x3r[b] * w3r - x3i[b] * w3i, u3i = x3r[b] * w3i + x3i[b] * w3r;
                const double ar = u0r + u2r, ai = u0i + u2i, br = u0r - u2r, bi = u0i - u2i;
                const double cr = u1r + u3r, ci = u1i + u3i;
                /* d = (u1 - u3) * (sg i) */
                const double dr = -sg * (u1i - u3i), di = sg * (u1r - u3r);
                y0r[b] = ar + cr;
                y0i[b] = ai + ci;
                y2r[b] = ar - cr;
                y2i[b] = ai - ci;
                y1r[b] = br + dr;
                y1i[b] = bi + di;
                y3r[b] = br - dr;
                y3i[b] = bi - di;
            }
        }
    }
}

/* SK_B-line batched FFT of the lines in (ar, ai); the result is left in
 * (ar, ai) or (br, bi): returns 0 or 1 accordingly. */
static int p2_exec(const p2plan* p, double* ar, double* ai, double* br, double* bi) {
    double* xr = ar;
    double* xi = ai;
    double* yr = br;
    double* yi = bi;
    int where = 0;
    for (int Ns = 1; Ns < p->n;) {
        const int R = (p->n / Ns) >= 4 ? 4 : 2;
        p2_pass(p, R, Ns, xr, xi, yr, yi);
        double* t = xr; xr = yr; yr = t;
        t = xi; xi = yi; yi = t;
        where ^= 1;
        Ns *= R;
    }
    return where;
}

/* --------------------------------------------------------- real-axis plan */

typedef struct {
    int n;        /* real length (even) */
    int pow2;     /* n / 2 is a power of two: batched path */
    cplan half;   /* length n/2 complex, sign as the direction */
    p2plan hp;    /* the same, batched (pow2) */
    cpx* tw;      /* tw[k] = exp(sign 2 pi i k / n), k in [0, n/2] */
} rplan;

static void rplan_init(rplan* p, int n, int sign) {
    p->n = n;
    p->pow2 = is_pow2(n / 2);
    cplan_init(&p->half, n / 2, sign);
    if (p->pow2) p2plan_init(&p->hp, n / 2, sign);
    p->tw = (cpx*)malloc(sizeof(cpx) * (size_t)(n / 2 + 1));
    for (int k = 0; k <= n / 2; ++k) p->tw[k] = unit_root(k, n, sign);
}

static void rplan_free(rplan* p) {
    cplan_free(&p->half);
    if (p->pow2) p2plan_free(&p->hp);
    free(p->tw);
}

/* r2c of nb <= SK_B rows (row r at x + r nl) into X + r h, through the
 * half-length batched FFT; buf holds 4 (n/2) SK_B doubles. */
static void r2c_batch(const rplan* p, const double* x, cpx* X, int nb, double* buf) {
    const int h = p->n / 2, nl = p->n, hs = h + 1;
    double* zr = buf;
    double* zi = zr + (size_t)h * SK_B;
    double* Zr = zi + (size_t)h * SK_B;
    double* Zi = Zr + (size_t)h * SK_B;
    for (int b = 0; b < SK_B; ++b) {
        const double* row = x + (size_t)b * nl;
        for (int j = 0; j < h; ++j) {
            zr[(size_t)j * SK_B + b] = b < nb ? row[2 * j] : 0.0;
            zi[(size_t)j * SK_B + b] = b < nb ? row[2 * j + 1] : 0.0;
        }
    }
    const int w = p2_exec(&p->hp, zr, zi, Zr, Zi);
    const double* ZR = w ? Zr : zr;
    const double* ZI = w ? Zi : zi;
    for (int b = 0; b < nb; ++b) {
        cpx* out = X + (size_t)b * hs;
        for (int k = 0; k <= h; ++k) {
            const size_t ia = (size_t)(k % h) * SK_B + b, ib = (size_t)((h - k) % h) * SK_B + b;
            const double ar = ZR[ia], ai = ZI[ia], br = ZR[ib], bi = -ZI[ib];
            const double er = 0.5 * (ar + br), ei = 0.5 * (ai + bi);
            const double orr = 0.5 * (ar - br), oi = 0.5 * (ai - bi);
            const cpx od = {oi, -orr}; /* odd part = -i o */
            const cpx t = cmul(p->tw[k], od);
            out[k].re = er + t.re;
            out[k].im = ei + t.im;
        }
    }
}

/* c2r of nb <= SK_B rows X + r h -> x + r nl (unnormalised; imaginary parts
 * of the index-0 and Nyquist entries ignored). */
static void c2r_batch(const rplan* p, const cpx* X, double* x, int nb, double* buf) {
    const int h = p->n / 2, nl = p->n, hs = h + 1;
    double* Zr = buf;
    double* Zi = Zr + (size_t)h * SK_B;
    double* zr = Zi + (size_t)h * SK_B;
    double* zi = zr + (size_t)h * SK_B;
    for (int b = 0; b < SK_B; ++b) {
        const cpx* in = X + (size_t)b * hs;
        for (int k = 0; k < h; ++k) {
            double re = 0.0, im = 0.0;
            if (b < nb) {
                cpx a = in[k], c = in[h - k];
                if (k == 0) {
                    a.im = 0.0;
                    c.im = 0.0;
                }
                const cpx cc = {c.re, -c.im};
                const cpx E = cadd(a, cc);
                const cpx O = cmul(csub(a, cc), p->tw[k]);
                re = E.re - O.im;
                im = E.im + O.re;
            }
            Zr[(size_t)k * SK_B + b] = re;
            Zi[(size_t)k * SK_B + b] = im;
        }
    }
    const int w = p2_exec(&p->hp, Zr, Zi, zr, zi);
    const double* RR = w ? zr : Zr;
    const double* RI = w ? zi : Zi;
    for (int b = 0; b < nb; ++b) {
        double* row = x + (size_t)b * nl;
        for (int j = 0; j < h; ++j) {
            row[2 * j] = RR[(size_t)j * SK_B + b];
            row[2 * j + 1] = RI[(size_t)j * SK_B + b];
        }
    }
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
    p2plan paxis[2]; /* the same, batched (power-of-two lengths) */
    int axis_pow2[2];
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
    for (int d = 0; d < rank - 1; ++d) {
        cplan_init(&p->axis[d], n[d], sign);
        p->axis_pow2[d] = is_pow2(n[d]);
        if (p->axis_pow2[d]) p2plan_init(&p->paxis[d], n[d], sign);
    }
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
    for (int d = 0; d < p->rank - 1; ++d) {
        cplan_free(&p->axis[d]);
        if (p->axis_pow2[d]) p2plan_free(&p->paxis[d]);
    }
    free(p);
}

/* c2c along leading axis `a` of the complex array with shape
 * (n[0], .., n[rank-2], h), in place, lines batched through a gather buffer. */
#define SK_BATCH 8
static void c2c_axis_p2(const fftw_plan p, cpx* data, int a) {
    const long len = p->n[a];
    long inner = p->h;
    for (int d = a + 1; d < p->rank - 1; ++d) inner *= p->n[d];
    long outer = 1;
    for (int d = 0; d < a; ++d) outer *= p->n[d];
    const long nbatch_in = (inner + SK_B - 1) / SK_B;
    const long total = outer * nbatch_in;
    const p2plan* pp = &p->paxis[a];
#pragma omp parallel num_threads(p->nthreads)
    {
        double* buf = (double*)malloc(sizeof(double) * (size_t)(4 * len * SK_B));
        double* xr = buf;
        double* xi = xr + len * SK_B;
        double* yr = xi + len * SK_B;
        double* yi = yr + len * SK_B;
#pragma omp for schedule(static)
        for (long t = 0; t < total; ++t) {
            const long o = t / nbatch_in;
            const long i0 = (t % nbatch_in) * SK_B;
            const int nb = (int)((inner - i0) < SK_B ? (inner - i0) : SK_B);
            cpx* base = data + o * len * inner + i0;
            for (long j = 0; j < len; ++j) {
                const cpx* src = base + j * inner;
                for (int b = 0; b < SK_B; ++b) {
                    xr[j * SK_B + b] = b < nb ? src[b].re : 0.0;
                    xi[j * SK_B + b] = b < nb ? src[b].im : 0.0;
                }
            }
            const int w = p2_exec(pp, xr, xi, yr, yi);
            const double* RR = w ? yr : xr;
            const double* RI = w ? yi : xi;
            for (long j = 0; j < len; ++j) {
                cpx* dst = base + j * inner;
                for (int b = 0; b < nb; ++b) {
                    dst[b].re = RR[j * SK_B + b];
                    dst[b].im = RI[j * SK_B + b];
                }
            }
        }
        free(buf);
    }
}

static void c2c_axis(const fftw_plan p, cpx* data, int a) {
    if (p->axis_pow2[a]) {
        c2c_axis_p2(p, data, a);
        return;
    }
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
    if (p->last.pow2) {
        const long nbat = (rows + SK_B - 1) / SK_B;
#pragma omp parallel num_threads(p->nthreads)
        {
            double* buf = (double*)malloc(sizeof(double) * (size_t)(2 * nl * SK_B));
#pragma omp for schedule(static)
            for (long t = 0; t < nbat; ++t) {
                const long r0 = t * SK_B;
                const int nb = (int)(rows - r0 < SK_B ? rows - r0 : SK_B);
                r2c_batch(&p->last, in + r0 * nl, X + r0 * p->h, nb, buf);
            }
            free(buf);
        }
    } else {
#pragma omp parallel num_threads(p->nthreads)
        {
            cpx* scratch = (cpx*)malloc(sizeof(cpx) * (size_t)(nl + 2));
#pragma omp for schedule(static)
            for (long r = 0; r < rows; ++r) r2c_1d(&p->last, in + r * nl, X + r * p->h, scratch);
            free(scratch);
        }
    }
    for (int a = p->rank - 2; a >= 0; --a) c2c_axis(p, X, a);
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
    cpx* X = (cpx*)in; /* clobbered, as FFTW's multi-dimensional c2r may do */
    for (int a = 0; a <= p->rank - 2; ++a) c2c_axis(p, X, a);
    long rows = 1;
    for (int d = 0; d < p->rank - 1; ++d) rows *= p->n[d];
    long nl = p->n[p->rank - 1];
    if (p->last.pow2) {
        const long nbat = (rows + SK_B - 1) / SK_B;
#pragma omp parallel num_threads(p->nthreads)
        {
            double* buf = (double*)malloc(sizeof(double) * (size_t)(2 * nl * SK_B));
#pragma omp for schedule(static)
            for (long t = 0; t < nbat; ++t) {
                const long r0 = t * SK_B;
                const int nb = (int)(rows - r0 < SK_B ? rows - r0 : SK_B);
                c2r_batch(&p->last, X + r0 * p->h, out + r0 * nl, nb, buf);
            }
            free(buf);
        }
        return;
    }
#pragma omp parallel num_threads(p->nthreads)
    {
        cpx* scratch = (cpx*)malloc(sizeof(cpx) * (size_t)(nl + 2));
#pragma omp for schedule(static)
        for (long r = 0; r < rows; ++r) c2r_1d(&p->last, X + r * p->h, out + r * nl, scratch);
        free(scratch);
    }
}
