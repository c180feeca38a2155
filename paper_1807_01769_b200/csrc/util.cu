// util.cu -- layout transposes, dealias-state check, device grid dump and
// diagnostic reductions.
#include <algorithm>
#include "skg_internal.h"

#include <cstdlib>
#include <map>
#include <vector>
#include <mutex>
#include <utility>

namespace skg {

namespace {

// DFMA throughput probe (skg_fp64_peak): 8 independent dependency chains per
// thread so the FP64 pipe, not latency, bounds the loop.
__global__ void __launch_bounds__(256) fp64_probe(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 123.456) out[0] = s;  // keeps the chains live
}


constexpr int TD = 32;

// out[c][r] = in[r][c] (complex), 32x32 tiles through shared memory.
__global__ void transpose_c(const cd* __restrict__ in, cd* __restrict__ out, int rows, int cols) {
    __shared__ cd tile[TD][TD + 1];
    const int c0 = blockIdx.x * TD, r0 = blockIdx.y * TD;
    for (int j = threadIdx.y; j < TD; j += blockDim.y) {
        const int r = r0 + j, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[j][threadIdx.x] = in[(size_t)r * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < TD; j += blockDim.y) {
        const int c = c0 + j, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[(size_t)c * rows + r] = tile[threadIdx.x][j];
    }
}

struct MaskGeo {
    int dims;
    int n[3];
    int nh;
    int kc[3];
};

// Multi-index (reference layout) of a flat spectral index.
__device__ __forceinline__ void unflatten(const MaskGeo& g, long long q, int* ix) {
    if (g.dims == 1) {
        ix[0] = (int)q;
    } else if (g.dims == 2) {
        ix[1] = (int)(q % g.nh);
        ix[0] = (int)(q / g.nh);
    } else {
        ix[2] = (int)(q % g.nh);
        long long r = q / g.nh;
        ix[1] = (int)(r % g.n[1]);
        ix[0] = (int)(r / g.n[1]);
    }
}

__device__ __forceinline__ bool kept(const MaskGeo& g, const int* ix) {
    for (int d = 0; d < g.dims; ++d) {
        const int si = d == g.dims - 1 ? ix[d] : signed_index(ix[d], g.n[d]);
        if (abs(si) > g.kc[d]) return false;
    }
    return true;
}

__global__ void count_masked(const cd* __restrict__ f, MaskGeo g, int nvars, long long S,
                             unsigned long long* count) {
    unsigned long long c = 0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < S;
         q += (long long)gridDim.x * blockDim.x) {
        int ix[3];
        unflatten(g, q, ix);
        if (kept(g, ix)) continue;
        for (int v = 0; v < nvars; ++v) {
            cd x = f[v * S + q];
            if (x.x != 0.0 || x.y != 0.0) ++c;
        }
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void grid_dump(MaskGeo g, int axis, double kscale, double* k, unsigned char* mask,
                          long long S) {
    const int ext = axis == g.dims - 1 ? g.nh : g.n[axis];
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < S;
         q += (long long)gridDim.x * blockDim.x) {
        if (q < ext) {
            const int si = axis == g.dims - 1 ? (int)q : signed_index((int)q, g.n[axis]);
            k[q] = kscale * (double)si;
        }
        if (mask) {
            int ix[3];
            unflatten(g, q, ix);
            mask[q] = kept(g, ix) ? 1 : 0;
        }
    }
}

struct EnGeo {
    MaskGeo m;
    double ks[3];
    int solver2d;  // 1: ns2d metric (solvers.cpp:211-218); 0: default (simulation.cpp:163-170)
    int cm;        // 1: ns2d CM layout [ky][kx]; 0: reference layout
    double nu;
};

// E and Z (Simulation::energy / enstrophy, simulation.cpp:592-615 with the
// ns2d mode_energy / mode_enstrophy of solvers.cpp:211-230 and the default
// Solver::mode_energy of simulation.cpp:163-170).
__global__ void energy_kernel(const cd* __restrict__ f, EnGeo g, int nvars, long long S,
                              double* out, const int* steps) {
    pdl_wait();
    if (steps) out += 3 * (*steps - 1);  // per-step series slot
    double e = 0.0, z = 0.0, d = 0.0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < S;
         q += (long long)gridDim.x * blockDim.x) {
        int ix[3];
        if (g.cm) {  // CM: q = ky * nx + kx
            ix[0] = (int)(q % g.m.n[0]);
            ix[1] = (int)(q / g.m.n[0]);
        } else {
            unflatten(g.m, q, ix);
        }
        const int il = ix[g.m.dims - 1];
        const double w = (il == 0 || il == g.m.nh - 1) ? 1.0 : 2.0;
        double ksq = 0.0;
        for (int ax = 0; ax < g.m.dims; ++ax) {
            const int si = ax == g.m.dims - 1 ? ix[ax] : signed_index(ix[ax], g.m.n[ax]);
            const double k = g.ks[ax] * si;
            ksq += k * k;
        }
        for (int v = 0; v < nvars; ++v) {
            cd x = f[v * S + q];
            const double nrm = x.x * x.x + x.y * x.y;
            if (g.solver2d) {
                if (ksq > 0.0) {
                    e += 0.5 * w * nrm / ksq;
                    d += 2.0 * g.nu * ksq * (0.5 * w * nrm / ksq);
                }
                z += 0.5 * w * nrm;
            } else {
                e += 0.5 * w * nrm;
                d += 2.0 * g.nu * ksq * (0.5 * w * nrm);
            }
        }
    }
    diag_accumulate(out, e, z, d);
}

struct DtGeo {
    int dims;
    int n[3];
    int ext[3];
    double ks[3];
    double nu;
};

// Simulation::compute_dt (CFL branch, simulation.cpp:463-476) and
// ExactLinStepper::refresh_exp (time_stepping.cpp:37-57) for the new dt.
__global__ void dt_update(DynStep* dyn, DevFlags* flags, double* etab, DtGeo g) {
    pdl_wait();
    if (flags->diverged) return;
    double dt = dyn->dt_max;
    for (int d = 0; d < g.dims; ++d) {
        const double vel = fmax(fabs(dyn->umax[d]), 1e-30);
        dt = fmin(dt, dyn->cfl * dyn->dx[d] / vel);
    }
    if (dyn->t_end >= 0.0) {
        const double remaining = dyn->t_end - dyn->t;
        if (remaining < dt) dt = remaining;
    }
    __syncthreads();  // every thread has read umax and t
    if (!(dt > 0.0)) {
        if (threadIdx.x == 0) {
            flags->bad_dt = 1;
            flags->div_step = flags->steps;
            flags->diverged = 1;  // stops the remaining kernels
        }
        return;
    }
    int per = 0;
    for (int d = 0; d < g.dims; ++d) per += g.ext[d];
    for (int q = threadIdx.x; q < 2 * per; q += blockDim.x) {
        const int which = q / per;
        int i = q % per, d = 0;
        while (i >= g.ext[d]) i -= g.ext[d++];
        const int si = d == g.dims - 1 ? i : signed_index(i, g.n[d]);
        const double kv = g.ks[d] * si;
        const double hdt = which == 0 ? 0.5 * dt : dt;
        etab[q] = exp(hdt * (-g.nu * (kv * kv)));
    }
    if (threadIdx.x == 0) {
        dyn->dt = dt;
        dyn->hdt = 0.5 * dt;
        dyn->sdt = dt / 6.0;
        dyn->last_dt = dt;
        dyn->t += dt;
        dyn->umax[0] = dyn->umax[1] = dyn->umax[2] = 0.0;
    }
}

MaskGeo make_geo(int dims, const int* n, const int* kc) {
    MaskGeo g{};
    g.dims = dims;
    for (int d = 0; d < dims; ++d) {
        g.n[d] = n[d];
        g.kc[d] = kc[d];
    }
    g.nh = n[dims - 1] / 2 + 1;
    return g;
}

// Pencil transposes: blockIdx.y = (f, x), the (y, z) plane of nz-long
// contiguous runs flattened over the threads (every lane busy whatever nz is),
// four independent 16-byte loads in flight per thread.
__global__ void __launch_bounds__(256) box_copy(BoxCopy b, int fence) {
    const unsigned x = blockIdx.y % b.nx, f = blockIdx.y / b.nx;
    const cd* __restrict__ s = b.src + f * b.sf + x * b.sx;
    cd* __restrict__ d = b.dst + f * b.df + x * b.dx;
    const unsigned nz = b.nz, total = (unsigned)b.ny * nz, stride = gridDim.x * 256u;
    unsigned i = blockIdx.x * 256u + threadIdx.x;
    for (; i + 3u * stride < total; i += 4u * stride) {
        cd v[4];
        size_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned idx = i + k * stride, y = idx / nz, z = idx - y * nz;
            v[k] = s[y * b.sy + z];
            o[k] = y * b.dy + z;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) d[o[k]] = v[k];
    }
    for (; i < total; i += stride) {
        const unsigned y = i / nz, z = i - y * nz;
        d[y * b.dy + z] = s[y * b.sy + z];
    }
    if (fence) __threadfence_system();
}

}  // namespace

cudaError_t launch_box_copy(const BoxCopy& b, bool fence, cudaStream_t s, long* launches) {
    const long long planes = (long long)b.nf * b.nx, per = (long long)b.ny * b.nz;
    if (planes == 0 || per == 0) return cudaSuccess;
    if (planes > 65535 || per >= (1ll << 31)) return cudaErrorInvalidValue;
    const int gx = (int)std::min<long long>((per + 1023) / 1024, 64);
    box_copy<<<dim3(gx, (unsigned)planes), 256, 0, s>>>(b, fence ? 1 : 0);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_transpose_c(const cd* in, cd* out, int rows, int cols, int, cudaStream_t s,
                               long* launches) {
    dim3 grid((cols + TD - 1) / TD, (rows + TD - 1) / TD);
    transpose_c<<<grid, dim3(TD, 8), 0, s>>>(in, out, rows, cols);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_count_masked(const cd* f, int dims, const int* n, const int* kc, int nvars,
                                long long S, unsigned long long* d_count, cudaStream_t s,
                                long* launches) {
    cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
    count_masked<<<592, 256, 0, s>>>(f, make_geo(dims, n, kc), nvars, S, d_count);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_grid_dump(int dims, const int* n, const int* kc, const double* kscale, int axis,
                             double* d_k, unsigned char* d_mask, cudaStream_t s, long* launches) {
    MaskGeo g = make_geo(dims, n, kc);
    long long S = 1;
    for (int d = 0; d < dims; ++d) S *= (d == dims - 1 ? g.nh : n[d]);
    grid_dump<<<592, 256, 0, s>>>(g, axis, kscale[axis], d_k, d_mask, S);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_dt_update(DynStep* dyn, DevFlags* flags, double* etab, int dims, const int* n,
                             const double* kscale, double nu, cudaStream_t s, long* launches) {
    DtGeo g{};
    g.dims = dims;
    for (int d = 0; d < dims; ++d) {
        g.n[d] = n[d];
        g.ext[d] = d == dims - 1 ? n[d] / 2 + 1 : n[d];
        g.ks[d] = kscale[d];
    }
    g.nu = nu;
    SKG_TRY(launch_pdl(dt_update, 1, 256, 0, s, dyn, flags, etab, g));
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_energy(const cd* f, int dims, const int* n, const double* kscale, int nvars,
                          int solver2d, double* d_out, cudaStream_t s, long* launches, double nu,
                          const int* steps, bool zero_first) {
    int kc[3] = {0, 0, 0};
    EnGeo g{};
    g.m = make_geo(dims, n, kc);
    for (int d = 0; d < dims; ++d) g.ks[d] = kscale[d];
    g.solver2d = solver2d != 0;  // 1: ns2d on the CM layout, 2: ns2d on the reference layout
    g.cm = solver2d == 1;
    g.nu = nu;
    long long S = 1;
    for (int d = 0; d < dims; ++d) S *= (d == dims - 1 ? g.m.nh : n[d]);
    if (zero_first) cudaMemsetAsync(d_out, 0, 3 * sizeof(double), s);
    SKG_TRY(launch_pdl(energy_kernel, 592, 256, 0, s, f, g, nvars, S, d_out, steps));
    ++*launches;
    return cudaGetLastError();
}

namespace {
constexpr size_t kGuard = 65536;
constexpr unsigned char kGuardByte = 0xA5;
std::mutex g_guard_mu;
std::map<void*, std::pair<void*, size_t>> g_guarded;  // user pointer -> (base, bytes)
}  // namespace

bool guards_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SKG_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}

cudaError_t dmalloc_raw(void** p, size_t bytes) {
    if (!guards_enabled()) return cudaMalloc(p, bytes);
    void* base = nullptr;
    SKG_TRY(cudaMalloc(&base, bytes + 2 * kGuard));
    char* b = static_cast<char*>(base);
    SKG_TRY(cudaMemset(b, kGuardByte, kGuard));
    SKG_TRY(cudaMemset(b + kGuard + bytes, kGuardByte, kGuard));
    SKG_TRY(cudaDeviceSynchronize());
    *p = b + kGuard;
    std::lock_guard<std::mutex> lock(g_guard_mu);
    g_guarded[*p] = {base, bytes};
    return cudaSuccess;
}

void dfree(void* p) {
    if (!p) return;
    if (guards_enabled()) {
        std::lock_guard<std::mutex> lock(g_guard_mu);
        auto it = g_guarded.find(p);
        if (it != g_guarded.end()) {
            cudaFree(it->second.first);
            g_guarded.erase(it);
            return;
        }
    }
    cudaFree(p);
}

long guard_violations() {
    if (!guards_enabled()) return 0;
    std::lock_guard<std::mutex> lock(g_guard_mu);
    std::vector<unsigned char> h(kGuard);
    long bad = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    for (const auto& kv : g_guarded) {
        const char* b = static_cast<const char*>(kv.second.first);
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, b) == cudaSuccess) cudaSetDevice(at.device);
        for (int side = 0; side < 2; ++side) {
            const char* g = side == 0 ? b : b + kGuard + kv.second.second;
            if (cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
            for (unsigned char v : h) bad += v != kGuardByte;
        }
    }
    cudaSetDevice(cur);
    return bad;
}

cudaError_t ensure_smem(const void* kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    SKG_TRY(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    size_t& d = done[{kernel, dev}];
    if (d >= bytes) return cudaSuccess;
    SKG_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    d = bytes;
    return cudaSuccess;
}

namespace {
__global__ void nsmid_probe(unsigned* out) {
    unsigned n;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
    *out = n;
}
}  // namespace

// Upper bound of %smid + 1 on `device` (the SM ids a CTA can observe are not
// guaranteed contiguous; %nsmid bounds them), at least the SM count.
int max_smid(int device) {
    static int cache[64] = {0};
    if (device >= 0 && device < 64 && cache[device]) return cache[device];
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    unsigned* d = nullptr;
    unsigned h = 0;
    if (dmalloc(&d, sizeof(unsigned)) != cudaSuccess) return sms > 256 ? sms : 256;
    nsmid_probe<<<1, 1>>>(d);
    if (cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) h = 256;
    dfree(d);
    const int r = (int)h > sms ? (int)h : sms;
    if (device >= 0 && device < 64) cache[device] = r;
    return r;
}

cudaError_t fp64_peak(int device, double* dfma_per_s) {
    SKG_TRY(cudaSetDevice(device));
    int sms = 0;
    SKG_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* d = nullptr;
    SKG_TRY(dmalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    SKG_TRY(cudaEventCreate(&e0));
    SKG_TRY(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    fp64_probe<<<blocks, threads>>>(d, 256, 0.999, 1e-3);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        SKG_TRY(cudaEventRecord(e0));
        fp64_probe<<<blocks, threads>>>(d, iters, 0.999, 1e-3);
        SKG_TRY(cudaEventRecord(e1));
        SKG_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        SKG_TRY(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(d);
    if (err != cudaSuccess) return err;
    *dfma_per_s = (double)blocks * threads * 8.0 * iters / (best * 1e-3);
    return cudaSuccess;
}

}  // namespace skg
