// forcing.cu -- the reference's random band forcing on the device
// (Simulation::refresh_forcing, proj/src/simulation.cpp:482-533;
// random_field, grid.cpp:276-306; prepare_forcing / injection_inner /
// addend_energy, solvers.cpp:242-272, 383-389, simulation.cpp:202-220).
//
// The white noise itself comes from the reference's generator on the host
// (std::mt19937_64 + std::normal_distribution, bit-identical with the same
// C++ library); everything after it runs here, on the reference layout:
//   band filter + unit magnitude -> prepare (dealias, mean 0; ns3d Leray
//   projection first) -> one reduction pass {<u,ub>, E(u), <u,f>, |f|^2}
//   -> coefficients (injection-rate split and the unit-energy fallback)
//   -> f = alpha f + beta ub, added to every RK stage's tendency.
// The addend energy after removing the component along ub is expanded
// algebraically: |f - c ub|^2 = |f|^2 - 2 c <ub,f> + c^2 |ub|^2 with the same
// metric, so one pass suffices.
#include "skg_internal.h"

namespace skg {

namespace {

constexpr int FB = 592, FT = 256;

struct FMode {
    double k[3], ksq, w;
    bool band, kept, mean;
};

__device__ __forceinline__ FMode fmode(const ForceGeo& g, long long q) {
    FMode m;
    int ix[3];
    long long r = q;
    for (int d = g.dims - 1; d >= 0; --d) {
        const int ext = d == g.dims - 1 ? g.nh : g.n[d];
        ix[d] = (int)(r % ext);
        r /= ext;
    }
    // k_sq in make_grid's order (grid.cpp:90-93: zero-padded leading axes)
    double ks[3] = {0.0, 0.0, 0.0};
    m.kept = true;
    for (int d = 0; d < g.dims; ++d) {
        const int si = d == g.dims - 1 ? ix[d] : signed_index(ix[d], g.n[d]);
        m.k[d] = g.ks[d] * (double)si;
        ks[3 - g.dims + d] = m.k[d];
        if (abs(si) > g.kc[d]) m.kept = false;
    }
    for (int d = g.dims; d < 3; ++d) m.k[d] = 0.0;
    m.ksq = ks[0] * ks[0] + ks[1] * ks[1] + ks[2] * ks[2];
    const double kc = (double)llround(sqrt(m.ksq) / g.delta_k) * g.delta_k;  // shell center
    m.band = !(kc < g.k_lo || kc > g.k_hi);
    const int il = ix[g.dims - 1];
    m.w = (il == 0 || il == g.nh - 1) ? 1.0 : 2.0;
    m.mean = q == 0;
    return m;
}

// random_field's band filter and unit magnitude (grid.cpp:293-302)
__global__ void f_band(ForceGeo g, cd* f) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.S;
         q += (long long)gridDim.x * blockDim.x) {
        const FMode m = fmode(g, q);
        for (int v = 0; v < g.nvars; ++v) {
            cd x = f[(size_t)v * g.S + q];
            if (!m.band) {
                x = zero();
            } else {
                const double mag = hypot(x.x, x.y);
                if (mag > 1e-300) x = mk(x.x / mag, x.y / mag);
            }
            f[(size_t)v * g.S + q] = x;
        }
    }
}

// prepare_forcing: ns2d dealias + mean 0 (solvers.cpp:269-272); ns3d Leray
// projection (grid.cpp:227-249), then dealias + mean 0 (solvers.cpp:383-389)
__global__ void f_prepare(ForceGeo g, cd* f, int zero_mean) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.S;
         q += (long long)gridDim.x * blockDim.x) {
        const FMode m = fmode(g, q);
        cd c[3];
        for (int v = 0; v < g.nvars; ++v) c[v] = f[(size_t)v * g.S + q];
        if (g.nvars == 3 && m.ksq != 0.0) {
            const cd dot = add(add(scale(c[0], m.k[0]), scale(c[1], m.k[1])), scale(c[2], m.k[2]));
            const cd sp = mk(dot.x / m.ksq, dot.y / m.ksq);
            for (int v = 0; v < 3; ++v) c[v] = sub(c[v], scale(sp, m.k[v]));
        }
        for (int v = 0; v < g.nvars; ++v)
            f[(size_t)v * g.S + q] = (!m.kept || (zero_mean && m.mean)) ? zero() : c[v];
    }
}

// {ibb = <u,ub>, eu = E(u), iuf = <u,f>, F = 2 addend(f)} with the solver's
// metrics: ns2d w Re(a conj b)/|k|^2 over |k| > 0 (solvers.cpp:242-262,
// 211-218), ns3d w Re(a conj b) over every mode (simulation.cpp:163-170, 202-220).
__global__ void f_reduce(ForceGeo g, const cd* u, const cd* f, double* out) {
    double ibb = 0.0, eu = 0.0, iuf = 0.0, ff = 0.0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.S;
         q += (long long)gridDim.x * blockDim.x) {
        const FMode m = fmode(g, q);
        double s = m.w;
        if (g.nvars == 1) {
            if (!(m.ksq > 0.0)) continue;
            s = m.w / m.ksq;
        }
        for (int v = 0; v < g.nvars; ++v) {
            const cd a = u[(size_t)v * g.S + q], b = f[(size_t)v * g.S + q];
            const double aa = a.x * a.x + a.y * a.y;
            if (m.band) ibb += s * aa;
            eu += 0.5 * s * aa;
            iuf += s * (a.x * b.x + a.y * b.y);
            ff += s * (b.x * b.x + b.y * b.y);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        ibb += __shfl_down_sync(0xffffffffu, ibb, o);
        eu += __shfl_down_sync(0xffffffffu, eu, o);
        iuf += __shfl_down_sync(0xffffffffu, iuf, o);
        ff += __shfl_down_sync(0xffffffffu, ff, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out + 0, ibb);
        atomicAdd(out + 1, eu);
        atomicAdd(out + 2, iuf);
        atomicAdd(out + 3, ff);
    }
}

// refresh_forcing's split (simulation.cpp:492-532): out[4] = alpha, out[5] =
// beta (f <- alpha f + beta ub), out[6] = last_injection, out[7] = fallback.
__global__ void f_coef(double rate, double* out) {
    const double ibb = out[0], eu = out[1], iuf = out[2], ff = out[3];
    double alpha, beta, inj, fb = 0.0;
    if (ibb <= 1e-6 * 2.0 * eu || eu <= 0.0) {
        const double ef = 0.5 * ff;
        if (ef <= 0.0) {
            alpha = 0.0;
            inj = 0.0;
        } else {
            alpha = 1.0 / sqrt(ef);
            inj = alpha * iuf;
        }
        beta = 0.0;
        fb = 1.0;
    } else {
        const double c = iuf / ibb;
        const double ef = 0.5 * (ff - 2.0 * c * iuf + c * c * ibb);
        const double unit = ef > 0.0 ? 1.0 / sqrt(ef) : 1.0;
        alpha = unit;
        beta = rate / ibb - unit * c;
        inj = rate;
    }
    out[4] = alpha;
    out[5] = beta;
    out[6] = inj;
    out[7] = fb;
}

__global__ void f_make(ForceGeo g, const cd* u, cd* f, const double* coef) {
    const double alpha = coef[4], beta = coef[5];
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.S;
         q += (long long)gridDim.x * blockDim.x) {
        const FMode m = fmode(g, q);
        for (int v = 0; v < g.nvars; ++v) {
            const size_t idx = (size_t)v * g.S + q;
            cd x = scale(f[idx], alpha);
            if (m.band) x = add(x, scale(u[idx], beta));
            f[idx] = x;
        }
    }
}

// Shell spectra of OutputManager::save_records_and_snapshot (output.cpp:231-257,
// bin_shells output.cpp:21-39): per-mode energy (solver metric), transfer
// w Re(conj(s) N) (ns2d / |k|^2, solvers.cpp:232-240; default simulation.cpp:176-185)
// and dissipation -2 nu |k|^2 e, binned by shell = round(|k| / delta_k).
__global__ void f_spectra(ForceGeo g, const cd* u, const cd* nl, double nu, int nsh, double* E,
                          double* Tr, double* D) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.S;
         q += (long long)gridDim.x * blockDim.x) {
        const FMode m = fmode(g, q);
        const long long sh = llround(sqrt(m.ksq) / g.delta_k);
        if (sh < 0 || sh >= nsh) continue;
        double s = m.w;
        if (g.nvars == 1) {
            if (!(m.ksq > 0.0)) continue;
            s = m.w / m.ksq;
        }
        double e = 0.0, t = 0.0;
        for (int v = 0; v < g.nvars; ++v) {
            const cd a = u[(size_t)v * g.S + q], b = nl[(size_t)v * g.S + q];
            e += 0.5 * s * (a.x * a.x + a.y * a.y);
            t += s * (a.x * b.x + a.y * b.y);
        }
        atomicAdd(E + sh, e);
        atomicAdd(Tr + sh, t);
        atomicAdd(D + sh, -2.0 * nu * m.ksq * e);
    }
}

}  // namespace

cudaError_t spectra_dev(const ForceGeo& g, const cd* u, const cd* nl, double nu, int nsh, double* out3,
                        cudaStream_t s, long* launches) {
    SKG_TRY(cudaMemsetAsync(out3, 0, sizeof(double) * 3 * nsh, s));
    f_spectra<<<FB, FT, 0, s>>>(g, u, nl, nu, nsh, out3, out3 + nsh, out3 + 2 * nsh);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t forcing_shape(const ForceGeo& g, cd* f, cudaStream_t s, long* launches) {
    f_band<<<FB, FT, 0, s>>>(g, f);
    f_prepare<<<FB, FT, 0, s>>>(g, f, 1);
    *launches += 2;
    return cudaGetLastError();
}

// Solver::sanitize_state: ns2d dealias + mean 0 (solvers.cpp:263-267); ns3d
// Leray projection + dealias (solvers.cpp:377-381), the mean kept.
cudaError_t sanitize_dev(const ForceGeo& g, cd* f, cudaStream_t s, long* launches) {
    f_prepare<<<FB, FT, 0, s>>>(g, f, g.nvars == 1 ? 1 : 0);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t forcing_finish(const ForceGeo& g, const cd* u, cd* f, double rate, double* red,
                           cudaStream_t s, long* launches) {
    SKG_TRY(cudaMemsetAsync(red, 0, 4 * sizeof(double), s));
    f_reduce<<<FB, FT, 0, s>>>(g, u, f, red);
    f_coef<<<1, 1, 0, s>>>(rate, red);
    f_make<<<FB, FT, 0, s>>>(g, u, f, red);
    *launches += 3;
    return cudaGetLastError();
}

}  // namespace skg
