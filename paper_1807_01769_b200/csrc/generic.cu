// generic.cu -- the RK step for extents the fused kernels do not cover
// (any even n >= 4 that is not a power of two in their range, e.g. 96, 384,
// 768): the reference's own operator sequence, one pass per operator, on the
// device.  State and every intermediate stay in the reference layout
// (row-major [n0][n1..][n_last/2+1]); the transforms are fft_ops.cu's
// FftPlan::forward/inverse (Stockham for powers of two, a line DFT otherwise).
//
//   Ns2dSolver::tendency (proj/src/solvers.cpp:133-174):
//     psi = w/|k|^2, ux = i ky psi, uy = -i kx psi (grid.cpp:251-274),
//     dx w, dy w (grid.cpp:124-143), 4 c2r, -(ux dx w + uy dy w), r2c,
//     dealias, mean 0
//   Ns3dSolver::tendency (solvers.cpp:299-339):
//     w = curl v (grid.cpp:182-207), 6 c2r, c = u x w, 3 r2c, Leray
//     projection (grid.cpp:227-249), dealias, mean 0
//   ExactLinStepper::step (time_stepping.cpp:72-194): stage states, RK4/RK2
//   combination, the no-linear-part branch, check_finite.
#include "skg_internal.h"

namespace skg {

namespace {

constexpr int GB = 592, GT = 256;  // grid-stride launch shape (4 x 148 SMs)

struct Mode {
    int i[3];
    double k[3];
    double ksq;
    bool kept;
};

__device__ __forceinline__ Mode mode_of(const GenArgs& a, long long q) {
    Mode m;
    long long r = q;
    for (int d = a.dims - 1; d >= 0; --d) {
        const int ext = d == a.dims - 1 ? a.nh : a.n[d];
        m.i[d] = (int)(r % ext);
        r /= ext;
    }
    m.ksq = 0.0;
    m.kept = true;
    for (int d = 0; d < a.dims; ++d) {
        const int si = d == a.dims - 1 ? m.i[d] : signed_index(m.i[d], a.n[d]);
        m.k[d] = a.ks[d] * (double)si;
        m.ksq += m.k[d] * m.k[d];
        if (abs(si) > a.kc[d]) m.kept = false;
    }
    for (int d = a.dims; d < 3; ++d) m.k[d] = 0.0;
    return m;
}

__device__ __forceinline__ double efac(const double* const* t, const GenArgs& a, const Mode& m) {
    double e = 1.0;
    for (int d = 0; d < a.dims; ++d) e *= t[d][m.i[d]];
    return e;
}

// RK stage state (time_stepping.cpp:128-170), every mode.
__global__ void g_stage(GenArgs a, int stage, cd* w) {
    pdl_wait();
    if (a.flags->diverged) return;
    const cd* kp = stage == 2 ? a.k1 : stage == 3 ? a.k2 : a.k3;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < a.S;
         q += (long long)gridDim.x * blockDim.x) {
        const Mode m = mode_of(a, q);
        const double e1 = a.has_sigma ? efac(a.e1, a, m) : 1.0;
        const double e2 = a.has_sigma ? efac(a.e2, a, m) : 1.0;
        for (int v = 0; v < a.nvars; ++v) {
            const size_t idx = (size_t)v * a.S + q;
            const cd u = a.u[idx];
            cd s = u;
            if (stage > 1) {
                const cd k = kp[idx];
                if (a.has_sigma) {
                    if (stage == 2) s = scale(add(u, scale(k, hdt_of(a))), e1);
                    else if (stage == 3) s = add(scale(u, e1), scale(k, hdt_of(a)));
                    else s = add(scale(u, e2), scale(k, dt_of(a) * e1));
                } else {
                    s = add(u, scale(k, stage == 4 ? dt_of(a) : hdt_of(a)));
                }
            }
            w[idx] = s;
        }
    }
}

// Spectral multipliers before the inverse transforms.
//  2D: out[0] = i ky psi, out[1] = -i kx psi, out[2] = i kx w, out[3] = i ky w
//  3D: out[0..2] = curl v
__global__ void g_pre(GenArgs a, const cd* w, cd* out) {
    pdl_wait();
    if (a.flags->diverged) return;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < a.S;
         q += (long long)gridDim.x * blockDim.x) {
        const Mode m = mode_of(a, q);
        if (a.dims == 2) {
            const cd ww = w[q];
            cd psi = zero();
            if (m.ksq != 0.0) psi = mk(ww.x / m.ksq, ww.y / m.ksq);
            out[q] = muli(scale(psi, m.k[1]));
            out[a.S + q] = mulmi(scale(psi, m.k[0]));
            out[2 * a.S + q] = muli(scale(ww, m.k[0]));
            out[3 * a.S + q] = muli(scale(ww, m.k[1]));
        } else {
            const cd vx = w[q], vy = w[a.S + q], vz = w[2 * a.S + q];
            out[q] = muli(sub(scale(vz, m.k[1]), scale(vy, m.k[2])));
            out[a.S + q] = muli(sub(scale(vx, m.k[2]), scale(vz, m.k[0])));
            out[2 * a.S + q] = muli(sub(scale(vy, m.k[0]), scale(vx, m.k[1])));
        }
    }
}

// Physical-space products (solvers.cpp:160-164 / 321-325), in place into
// p[0] (2D) or p[0..2] (3D); stage 1 of an adaptive step also reduces
// max |u_d| of the step's initial state.
//  2D: p = [ux, uy, dx w, dy w];  3D: p = [ux, uy, uz, wx, wy, wz]
__global__ void g_prod(GenArgs a, double* p, int cfl) {
    pdl_wait();
    if (a.flags->diverged) return;
    double mx = 0.0, my = 0.0, mz = 0.0;
    const long long P = a.P;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P;
         q += (long long)gridDim.x * blockDim.x) {
        if (a.dims == 2) {
            const double ux = p[q], uy = p[P + q];
            if (cfl) {
                mx = fmax(mx, fabs(ux));
                my = fmax(my, fabs(uy));
            }
            p[q] = -(ux * p[2 * P + q] + uy * p[3 * P + q]);
        } else {
            const double ux = p[q], uy = p[P + q], uz = p[2 * P + q];
            const double ox = p[3 * P + q], oy = p[4 * P + q], oz = p[5 * P + q];
            if (cfl) {
                mx = fmax(mx, fabs(ux));
                my = fmax(my, fabs(uy));
                mz = fmax(mz, fabs(uz));
            }
            p[q] = uy * oz - uz * oy;
            p[P + q] = uz * ox - ux * oz;
            p[2 * P + q] = ux * oy - uy * ox;
        }
    }
    if (cfl) umax_accumulate(a.dyn, a.dims, mx, my, mz);
}

// After the forward transforms (already x 1/N): projection (3D), dealias,
// mean 0 -> the tendency k; then either store k_j or, on the final stage,
// the RK update of u (time_stepping.cpp:171-193) with the non-finite flag.
// out == nullptr: tendency only, written into nl (skg_tendency).
__global__ void g_post(GenArgs a, cd* nl, int stage, cd* kout) {
    pdl_wait();
    if (a.flags->diverged) return;
    const bool final = a.rk2 ? stage == 2 : stage == 4;
    int bad = 3;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < a.S;
         q += (long long)gridDim.x * blockDim.x) {
        const Mode m = mode_of(a, q);
        const bool mean = m.ksq == 0.0 && m.i[0] == 0;
        cd c[3];
        for (int v = 0; v < a.nvars; ++v) c[v] = nl[(size_t)v * a.S + q];
        if (a.dims == 3 && m.ksq != 0.0) {
            const cd dot = add(add(scale(c[0], m.k[0]), scale(c[1], m.k[1])), scale(c[2], m.k[2]));
            const cd sp = mk(dot.x / m.ksq, dot.y / m.ksq);
            for (int v = 0; v < 3; ++v) c[v] = sub(c[v], scale(sp, m.k[v]));
        }
        for (int v = 0; v < a.nvars; ++v) {
            if (!m.kept || mean) c[v] = zero();
            if (a.force) c[v] = add(c[v], a.force[(size_t)v * a.S + q]);  // simulation.cpp:544-547
        }
        const double e1 = a.has_sigma ? efac(a.e1, a, m) : 1.0;
        const double e2 = a.has_sigma ? efac(a.e2, a, m) : 1.0;
        for (int v = 0; v < a.nvars; ++v) {
            const size_t idx = (size_t)v * a.S + q;
            const cd kv = c[v];
            if (!kout) {
                nl[idx] = kv;
            } else if (!final) {
                kout[idx] = kv;
            } else {
                const cd u = a.u[idx];
                cd un;
                if (a.has_sigma) {
                    if (a.rk2) {
                        un = add(scale(u, e2), scale(kv, dt_of(a) * e1));
                    } else {
                        const cd sum = add(add(scale(a.k1[idx], e2), scale(add(a.k2[idx], a.k3[idx]), 2.0 * e1)), kv);
                        un = add(scale(u, e2), scale(sum, sdt_of(a)));
                    }
                } else {
                    cd delta;
                    if (a.rk2) delta = scale(kv, dt_of(a));
                    else delta = scale(add(add(a.k1[idx], scale(add(a.k2[idx], a.k3[idx]), 2.0)), kv), sdt_of(a));
                    un = (delta.x != 0.0 || delta.y != 0.0) ? add(u, delta) : u;
                }
                a.u[idx] = un;
                if (!(isfinite(un.x) && isfinite(un.y)) && v < bad) bad = v;
            }
        }
    }
    if (bad < 3) {
        atomicMin(&a.flags->div_var, bad);
        atomicExch(&a.flags->div_step, a.flags->steps);
        atomicExch(&a.flags->diverged, 1);
    }
}

__global__ void g_count_step(DevFlags* flags) {
    pdl_wait();
    if (!flags->diverged) atomicAdd(&flags->steps, 1);
}

}  // namespace

cudaError_t generic_tendency(const GenArgs& a, const cd* w, int stage, cd* kout, GenScratch& g,
                             cudaStream_t s, long* launches) {
    const int dims = a.dims;
    const int nin = dims == 2 ? 4 : 6;
    // spectral inputs of the inverse transforms
    SKG_TRY(launch_pdl(g_pre, GB, GT, 0, s, a, w, g.spec));
    ++*launches;
    const cd* src[6];
    if (dims == 2) {
        for (int f = 0; f < 4; ++f) src[f] = g.spec + (size_t)f * a.S;
    } else {
        for (int f = 0; f < 3; ++f) src[f] = w + (size_t)f * a.S;
        for (int f = 0; f < 3; ++f) src[3 + f] = g.spec + (size_t)f * a.S;
    }
    for (int f = 0; f < nin; ++f)
        SKG_TRY(fft_inverse_dev(dims, a.n, src[f], g.phys + (size_t)f * a.P, g.work, g.tw, s, launches));
    SKG_TRY(launch_pdl(g_prod, GB, GT, 0, s, a, g.phys, (a.dyn && stage == 1) ? 1 : 0));
    ++*launches;
    for (int v = 0; v < a.nvars; ++v)
        SKG_TRY(fft_forward_dev(dims, a.n, g.phys + (size_t)v * a.P, g.nl + (size_t)v * a.S, g.work,
                                g.tw, s, launches));
    SKG_TRY(launch_pdl(g_post, GB, GT, 0, s, a, g.nl, stage, kout));
    ++*launches;
    return cudaSuccess;
}

cudaError_t generic_stage(const GenArgs& a, int stage, GenScratch& g, cudaStream_t s, long* launches) {
    if (stage == 1) {
        SKG_TRY(launch_pdl(g_count_step, 1, 1, 0, s, a.flags));
        ++*launches;
    }
    const cd* w = a.u;
    if (stage > 1) {
        SKG_TRY(launch_pdl(g_stage, GB, GT, 0, s, a, stage, g.w));
        ++*launches;
        w = g.w;
    }
    cd* kout = stage == 1 ? a.k1 : stage == 2 ? a.k2 : a.k3;
    if (a.rk2 ? stage == 2 : stage == 4) kout = a.k3;  // final: u updated in place; k unused
    return generic_tendency(a, w, stage, kout, g, s, launches);
}

}  // namespace skg
