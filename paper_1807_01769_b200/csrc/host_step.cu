// host_step.cu -- step enqueueing of libskgpu (see host_ctx.h): the per-step
// launch sequences (fused 2D/3D paths, generic path, CUDA-graph replay),
// the adaptive-dt and forcing hooks, the slab all-to-all exchanges and the
// post-step divergence / time bookkeeping.
#include "host_ctx.h"

namespace skh {

// Simulation::refresh_forcing (simulation.cpp:482-533) before a step: the
// reference's generator fills the white noise on the host (one
// normal_distribution per variable, random_field grid.cpp:285-288), the rest
// runs on the device (forcing.cu).
int refresh_forcing(skg_ctx* c) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));  // the pinned noise buffer is reused
    const size_t P = (size_t)c->P;
    const cd* tw[3] = {c->tw[0], c->tw[1], c->tw[2]};
    for (int v = 0; v < c->nvars; ++v) {
        std::normal_distribution<double> gauss(0.0, 1.0);
        double* h = c->f_noise + v * P;
        for (size_t i = 0; i < P; ++i) h[i] = gauss(c->f_rng);
    }
    const skg::ForceGeo g = force_geo(c);
    for (int v = 0; v < c->nvars; ++v) {
        CUDA_TRY(cudaMemcpyAsync(c->phys, c->f_noise + v * P, sizeof(double) * P, cudaMemcpyHostToDevice,
                                 c->stream));
        CUDA_TRY(skg::fft_forward_dev(c->dims, c->n, c->phys, c->f_ref + (size_t)v * c->S, c->work, tw,
                                      c->stream, &c->launches));
    }
    CUDA_TRY(skg::forcing_shape(g, c->f_ref, c->stream, &c->launches));
    const cd* uref = c->u;
    if (c->f_cm) {  // ns2d fused kernels keep the state in CM layout
        int rc = store_state_to_io(c, c->u);
        if (rc) return rc;
        uref = c->io;
    }
    CUDA_TRY(skg::forcing_finish(g, uref, c->f_ref, c->f_rate, c->f_red, c->stream, &c->launches));
    if (c->f_cm)
        CUDA_TRY(skg::launch_transpose_c(c->f_ref, c->f_cm, c->n[0], c->nh, 0, c->stream, &c->launches));
    return SKG_OK;
}

int sync_and_check(skg_ctx* c, long nsteps, double dt) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    harvest(c);
    skg::DevFlags f;
    CUDA_TRY(cudaMemcpy(&f, c->flags, sizeof(f), cudaMemcpyDeviceToHost));
    if (c->forcing) {
        double r[8];
        CUDA_TRY(cudaMemcpy(r, c->f_red, sizeof(r), cudaMemcpyDeviceToHost));
        c->last_injection = r[6];
    }
    skg::DynStep dyn{};
    if (c->adaptive) {
        CUDA_TRY(cudaMemcpy(&dyn, c->d_dyn, sizeof(dyn), cudaMemcpyDeviceToHost));
        c->last_dt = dyn.last_dt;
    }
    if (f.bad_dt) {  // compute_dt gave dt <= 0 (past t_end): the step did not run
        c->it += f.div_step - 1;
        c->t = dyn.t;
        return fail(SKG_ECONFIG, "step: nonpositive dt (past t_end?)");
    }
    if (f.diverged) {
        const long done = f.div_step;
        if (c->adaptive) c->t = dyn.t;
        else
            for (long i = 0; i < done; ++i) c->t += dt;
        c->it += done;
        c->div_it = c->it;
        c->div_var = f.div_var;
        static const char* keys2[] = {"rot_fft"};
        static const char* keys3[] = {"vx_fft", "vy_fft", "vz_fft"};
        const char* key = c->solver == 2 ? keys2[0] : keys3[f.div_var >= 0 && f.div_var < 3 ? f.div_var : 0];
        return fail(SKG_EDIVERGENCE, std::string("non-finite value in field '") + key +
                                         "' at iteration " + std::to_string(c->it));
    }
    if (c->adaptive) {
        c->t = dyn.t;
    } else {
        for (long i = 0; i < nsteps; ++i) c->t += dt;
        if (nsteps > 0) c->last_dt = dt;
    }
    c->it += nsteps;
    return SKG_OK;
}

// All-to-all of the slab decomposition.  which = 0: x-inverse outputs
// (rows(q) x cols(r) from r to q), 1: product spectra (cols(q) x rows(r)).
// Single-process mode: device-to-device copies; otherwise NCCL send/recv
// on the context stream (grouped, one block per peer).
int exchange3(skg_ctx* c, int which, unsigned fmask = 0xffu, cudaStream_t st = nullptr);

int exchange(skg_ctx* c, int which) {
    if (c->solver == 3) return exchange3(c, which);
    if (c->p2p) {  // the producers already stored into the receive buffers
        if (c->comm) {  // cross-rank barrier: every rank's producer kernel has completed
            const ncclResult_t nr = nccl().AllReduce(c->d_barrier, c->d_barrier, 1, ncclDouble, ncclSum,
                                                     c->comm, c->stream);
            if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
        }
        return SKG_OK;
    }
    const int G = c->G;
    const size_t nrl = (size_t)c->nrl;
    auto ncol = [&](int q) { return c->cstart[q + 1] - c->cstart[q]; };
    auto npair = [&](int q) { return (size_t)(ncol(q) + 1) / 2; };
    // block (source r -> destination q): pointers and element count
    auto block = [&](const Part& src, const Part& dst, int f, cd** from, cd** to, size_t* cnt) {
        const int r = src.r, q = dst.r;
        if (which == 0) {
            *cnt = nrl * ncol(r);
            *from = src.sI[f] + (size_t)q * nrl * ncol(r);
            *to = dst.rI[f] + nrl * c->cstart[r];
        } else {
            *cnt = 2 * npair(q) * nrl;
            *from = src.sA[f] + (size_t)(c->cstart[q] / 2) * 2 * nrl;
            *to = dst.rA[f] + (size_t)r * 2 * npair(q) * nrl;
        }
    };
    const skg::LaunchHook hook = hook_of(c);
    hook.begin(4);
    double bytes = 0.0;
    if (c->comm == nullptr) {  // all partitions local
        for (const Part& src : c->parts)
            for (const Part& dst : c->parts)
                for (int f = 0; f < 2; ++f) {
                    cd *from, *to;
                    size_t cnt;
                    block(src, dst, f, &from, &to, &cnt);
                    if (cnt == 0) continue;
                    CUDA_TRY(cudaMemcpyAsync(to, from, cnt * sizeof(cd), cudaMemcpyDeviceToDevice, c->stream));
                    if (src.r != dst.r) bytes += cnt * sizeof(cd);
                }
    } else {
        const Part& me = c->parts[0];
        const int r = me.r;
        ncclResult_t nr = nccl().GroupStart();
        for (int q = 0; q < G && nr == ncclSuccess; ++q) {
            for (int f = 0; f < 2 && nr == ncclSuccess; ++f) {
                cd *sptr, *rptr;
                size_t scnt, rcnt;
                if (which == 0) {
                    sptr = me.sI[f] + (size_t)q * nrl * ncol(r);
                    scnt = nrl * ncol(r);
                    rptr = me.rI[f] + nrl * c->cstart[q];
                    rcnt = nrl * ncol(q);
                } else {
                    sptr = me.sA[f] + (size_t)(c->cstart[q] / 2) * 2 * nrl;
                    scnt = 2 * npair(q) * nrl;
                    rptr = me.rA[f] + (size_t)q * 2 * npair(r) * nrl;
                    rcnt = 2 * npair(r) * nrl;
                }
                if (q == r) {
                    if (scnt) CUDA_TRY(cudaMemcpyAsync(rptr, sptr, scnt * sizeof(cd), cudaMemcpyDeviceToDevice, c->stream));
                    continue;
                }
                if (scnt) nr = nccl().Send(sptr, 2 * scnt, ncclDouble, q, c->comm, c->stream);
                if (nr == ncclSuccess && rcnt) nr = nccl().Recv(rptr, 2 * rcnt, ncclDouble, q, c->comm, c->stream);
                bytes += scnt * sizeof(cd);
            }
        }
        ncclResult_t ne = nccl().GroupEnd();
        if (nr != ncclSuccess || ne != ncclSuccess)
            return fail(SKG_ENCCL, std::string("all-to-all: ") + nccl().GetErrorString(nr != ncclSuccess ? nr : ne));
    }
    hook.end(4, bytes);
    ++c->launches;
    return SKG_OK;
}

// ns3d all-to-alls.  which = 0: x-inverse outputs, 5 fields, block r -> q =
// rows(q) x lines(r) ([xl][kyl_r][kz_in]); 1: y-forward outputs, 3 fields,
// block r -> q = rows(r) x lines(q) ([xl][kyl_q][kz_o]).  fmask: the fields
// to exchange (bit f); st: the stream (default: the context stream).
int exchange3(skg_ctx* c, int which, unsigned fmask, cudaStream_t st) {
    if (!st) st = c->stream;
    const int G = c->G;
    if (G == 1) return SKG_OK;  // one partition: receive buffers alias the send buffers
    if (c->p2p) {  // producers stored into the receive buffers: a barrier remains
        if (c->comm) {
            const ncclResult_t nr = nccl().AllReduce(c->d_barrier, c->d_barrier, 1, ncclDouble, ncclSum,
                                                     c->comm, c->stream);
            if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
        }
        return SKG_OK;
    }
    const size_t nrl = (size_t)c->nrl;
    const int Pz = c->Pz;  // pencil: the exchange runs inside each group of equal pz
    auto nl = [&](int q) { return (size_t)(c->cstart[q + 1] - c->cstart[q]); };
    const int nf = which == 0 ? 5 : 3;
    // block from rank r (buffers src) to rank q (buffers dst), field f; kz: the
    // group's kz extent (kz_in = kz_o, pruned)
    auto src_ptr = [&](const Part& src, int q, int f) {
        const size_t kz = (size_t)src.nkz;
        return which == 0 ? src.A3 + f * src.fs + (size_t)q * nrl * nl(src.r) * kz
                          : src.sD3 + f * src.rfs + nrl * c->cstart[q] * kz;
    };
    auto dst_ptr = [&](const Part& dst, int r, int f) {
        const size_t kz = (size_t)dst.nkz;
        return which == 0 ? dst.rA3 + f * dst.rfs + nrl * c->cstart[r] * kz
                          : dst.B3 + f * dst.fs + (size_t)r * nrl * nl(dst.r) * kz;
    };
    auto count = [&](int r, int q, size_t kz) { return nrl * kz * (which == 0 ? nl(r) : nl(q)); };
    const skg::LaunchHook hook = hook_of(c);
    hook.begin(4);
    double bytes = 0.0;
    if (c->comm == nullptr) {
        for (const Part& src : c->parts)
            for (const Part& dst : c->parts)
                for (int f = 0; f < nf; ++f) {
                    if (src.pz != dst.pz) continue;
                    const size_t cnt = count(src.r, dst.r, (size_t)src.nkz);
                    if (!cnt || !(fmask >> f & 1u)) continue;
                    CUDA_TRY(cudaMemcpyAsync(dst_ptr(dst, src.r, f), src_ptr(src, dst.r, f),
                                             cnt * sizeof(cd), cudaMemcpyDeviceToDevice, st));
                    if (src.r != dst.r) bytes += cnt * sizeof(cd);
                }
    } else {
        const Part& me = c->parts[0];
        const int r = me.r;
        ncclResult_t nr = nccl().GroupStart();
        for (int q = 0; q < G && nr == ncclSuccess; ++q) {
            const int peer = q * Pz + me.pz;  // global rank of the group's member q
            for (int f = 0; f < nf && nr == ncclSuccess; ++f) {
                if (!(fmask >> f & 1u)) continue;
                const size_t scnt = count(r, q, (size_t)me.nkz), rcnt = count(q, r, (size_t)me.nkz);
                cd* sptr = src_ptr(me, q, f);
                cd* rptr = dst_ptr(me, q, f);
                if (q == r) {
                    if (scnt) CUDA_TRY(cudaMemcpyAsync(rptr, sptr, scnt * sizeof(cd), cudaMemcpyDeviceToDevice, st));
                    continue;
                }
                if (scnt) nr = nccl().Send(sptr, 2 * scnt, ncclDouble, peer, c->comm, st);
                if (nr == ncclSuccess && rcnt) nr = nccl().Recv(rptr, 2 * rcnt, ncclDouble, peer, c->comm, st);
                bytes += scnt * sizeof(cd);
            }
        }
        ncclResult_t ne = nccl().GroupEnd();
        if (nr != ncclSuccess || ne != ncclSuccess)
            return fail(SKG_ENCCL, std::string("all-to-all: ") + nccl().GetErrorString(nr != ncclSuccess ? nr : ne));
    }
    hook.end(4, bytes);
    ++c->launches;
    return SKG_OK;
}

// Pencil decomposition: the kz <-> y transposes inside each group of equal
// r (Pz members).  dir = 0, after the y-inverse: the six fields
// [xl][y][kz in the member's range] (B3) -> every member's z-pass input
// [xl][y in its rows][all kept kz] (Z3).  dir = 1, after the z pass: its three
// outputs [xl][yl][all kept kz] (A3, stride fsz) -> every member's y-forward
// input [xl][y][kz in its range] (fields 3..5 of B3).  All parts local, or the
// peer-memory route: ONE strided copy kernel per destination stores straight
// into the destination's layout (peer memory over NVLink across processes;
// no pack / unpack pass), then the barrier.  NCCL route: pack into one
// contiguous block per member, grouped send / recv, unpack.
int exchange_z(skg_ctx* c, int dir, cudaStream_t st) {
    if (!st) st = c->stream;
    const int Pz = c->Pz;
    if (Pz == 1) return SKG_OK;
    if (dir == 2) {  // the y-inverse stored into the members' Z3 already: the barrier remains
        const skg::LaunchHook hook = hook_of(c);
        double moved = 0.0;  // bytes its stores sent to other members
        for (const Part& s : c->parts)
            moved += (double)sizeof(cd) * 6 * c->nrl * c->nyl * s.nkz * (Pz - 1);
        hook.begin(4);
        hook.end(4, moved);
        if (c->comm) {
            const ncclResult_t nr = nccl().AllReduce(c->d_barrier, c->d_barrier, 1, ncclDouble, ncclSum, c->comm, st);
            if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
        }
        return SKG_OK;
    }
    const size_t nrl = (size_t)c->nrl, ny = (size_t)c->n[1], nyl = (size_t)c->nyl;
    const size_t kzf = (size_t)c->kc[2] + 1;
    const int nf = dir == 0 ? 6 : 3;
    const skg::LaunchHook hook = hook_of(c);
    hook.begin(4);
    double bytes = 0.0;
    // box from member `s` (kz range [skz0, skz0 + snkz), rows of member spz) to
    // member `d`: source and destination base pointers are the buffers' starts
    auto box = [&](const cd* sbuf, size_t sfs, int spz, int skz0, int snkz, cd* dbuf, size_t dfs_,
                   int dpz, int dkz0, int dnkz) {
        skg::BoxCopy b{};
        b.nf = nf;
        b.nx = (int)nrl;
        b.ny = (int)nyl;
        if (dir == 0) {  // B3 [xl][ny][snkz] rows of d -> Z3 [xl][nyl][kzf] at kz skz0
            b.nz = snkz;
            b.src = sbuf + (size_t)dpz * nyl * snkz;
            b.sf = sfs, b.sx = ny * snkz, b.sy = (size_t)snkz;
            b.dst = dbuf + skz0;
            b.df = dfs_, b.dx = nyl * kzf, b.dy = kzf;
        } else {  // A3 [xl][nyl][kzf] kz of d -> B3 fields 3.. [xl][ny][dnkz] rows of s
            b.nz = dnkz;
            b.src = sbuf + dkz0;
            b.sf = sfs, b.sx = nyl * kzf, b.sy = kzf;
            b.dst = dbuf + 3 * dfs_ + (size_t)spz * nyl * dnkz;
            b.df = dfs_, b.dx = ny * dnkz, b.dy = (size_t)dnkz;
        }
        return b;
    };
    if (c->comm == nullptr && !c->zpack) {  // all parts in this process
        for (const Part& s : c->parts)
            for (const Part& d : c->parts) {
                if (s.r != d.r) continue;
                const skg::BoxCopy b = dir == 0 ? box(s.B3, s.fs, s.pz, s.kz0, s.nkz, d.Z3, d.fsz, d.pz, d.kz0, d.nkz)
                                                : box(s.A3, s.fsz, s.pz, s.kz0, s.nkz, d.B3, d.fs, d.pz, d.kz0, d.nkz);
                CUDA_TRY(skg::launch_box_copy(b, false, st, &c->launches));
                if (s.pz != d.pz) bytes += (double)sizeof(cd) * b.nf * b.nx * b.ny * b.nz;
            }
    } else if (c->comm && c->p2p) {  // stores into the members' buffers, then the barrier
        const Part& s = c->parts[0];
        for (int z = 0; z < Pz; ++z) {
            const int peer = s.r * Pz + z;
            const int dkz0 = c->zstart[z], dnkz = c->zstart[z + 1] - c->zstart[z];
            // B3's and Z3's field strides are uniform over the ranks
            const skg::BoxCopy b = dir == 0 ? box(s.B3, s.fs, s.pz, s.kz0, s.nkz, c->peer_Z3[peer], s.fsz, z, dkz0, dnkz)
                                            : box(s.A3, s.fsz, s.pz, s.kz0, s.nkz, c->peer_B3[peer], s.fs, z, dkz0, dnkz);
            CUDA_TRY(skg::launch_box_copy(b, true, st, &c->launches));
            if (z != s.pz) bytes += (double)sizeof(cd) * b.nf * b.nx * b.ny * b.nz;
        }
        const ncclResult_t nr = nccl().AllReduce(c->d_barrier, c->d_barrier, 1, ncclDouble, ncclSum, c->comm, st);
        if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
    } else {  // NCCL (or its single-process stand-in): pack, send / recv, unpack
        const size_t plane = nrl * nyl;  // (x, y) rows of one block
        // member me's send block to member z / receive block from member z: offset, kz extent
        auto nkz_of = [&](int z) { return (size_t)(c->zstart[z + 1] - c->zstart[z]); };
        auto soff = [&](const Part& me, int z) {
            return dir == 0 ? (size_t)z * nf * plane * me.nkz : (size_t)nf * plane * c->zstart[z];
        };
        auto skz = [&](const Part& me, int z) { return dir == 0 ? (size_t)me.nkz : nkz_of(z); };
        auto roff = [&](const Part& me, int z) {
            return dir == 0 ? (size_t)nf * plane * c->zstart[z] : (size_t)z * nf * plane * me.nkz;
        };
        auto rkz = [&](const Part& me, int z) { return dir == 0 ? nkz_of(z) : (size_t)me.nkz; };
        for (Part& me : c->parts) {
            if (!me.sZ) {  // Pz blocks of up to max nkz modes (uneven kz ranges)
                size_t maxkz = 0;
                for (int z = 0; z < Pz; ++z) maxkz = std::max(maxkz, nkz_of(z));
                CUDA_TRY(skg::dmalloc(&me.sZ, sizeof(cd) * 6 * plane * Pz * maxkz));
                CUDA_TRY(skg::dmalloc(&me.rZ, sizeof(cd) * 6 * plane * Pz * maxkz));
            }
            for (int z = 0; z < Pz; ++z) {  // pack (the own block goes straight to its place)
                const int dkz0 = c->zstart[z], dnkz = (int)nkz_of(z);
                skg::BoxCopy b = dir == 0 ? box(me.B3, me.fs, me.pz, me.kz0, me.nkz, me.Z3, me.fsz, z, dkz0, dnkz)
                                          : box(me.A3, me.fsz, me.pz, me.kz0, me.nkz, me.B3, me.fs, z, dkz0, dnkz);
                if (z != me.pz) {  // contiguous [f][xl][yl][kz]
                    b.dst = me.sZ + soff(me, z);
                    b.dy = skz(me, z), b.dx = nyl * skz(me, z), b.df = plane * skz(me, z);
                }
                CUDA_TRY(skg::launch_box_copy(b, false, st, &c->launches));
            }
        }
        if (c->comm) {
            const Part& me = c->parts[0];
            ncclResult_t nr = nccl().GroupStart();
            for (int z = 0; z < Pz && nr == ncclSuccess; ++z) {
                if (z == me.pz) continue;
                const int peer = me.r * Pz + z;
                nr = nccl().Send(me.sZ + soff(me, z), 2 * nf * plane * skz(me, z), ncclDouble, peer, c->comm, st);
                if (nr == ncclSuccess)
                    nr = nccl().Recv(me.rZ + roff(me, z), 2 * nf * plane * rkz(me, z), ncclDouble, peer,
                                     c->comm, st);
                bytes += (double)sizeof(cd) * nf * plane * skz(me, z);
            }
            ncclResult_t ne = nccl().GroupEnd();
            if (nr != ncclSuccess || ne != ncclSuccess)
                return fail(SKG_ENCCL, std::string("pencil transpose: ") +
                                           nccl().GetErrorString(nr != ncclSuccess ? nr : ne));
        } else {  // the send / recv pairs as device copies
            for (const Part& sp : c->parts)
                for (const Part& dp : c->parts) {
                    if (sp.r != dp.r || sp.pz == dp.pz) continue;
                    const size_t cnt = nf * plane * skz(sp, dp.pz);
                    CUDA_TRY(cudaMemcpyAsync(dp.rZ + roff(dp, sp.pz), sp.sZ + soff(sp, dp.pz), cnt * sizeof(cd),
                                             cudaMemcpyDeviceToDevice, st));
                    bytes += (double)cnt * sizeof(cd);
                }
        }
        for (const Part& me : c->parts)
            for (int z = 0; z < Pz; ++z) {  // unpack the received blocks
                if (z == me.pz) continue;
                // as if member z had stored it: the box from z to me, read from the block
                skg::BoxCopy b = dir == 0 ? box(nullptr, 0, z, c->zstart[z], (int)nkz_of(z), me.Z3, me.fsz, me.pz, me.kz0, me.nkz)
                                          : box(nullptr, 0, z, c->zstart[z], (int)nkz_of(z), me.B3, me.fs, me.pz, me.kz0, me.nkz);
                b.src = me.rZ + roff(me, z);
                b.sy = rkz(me, z), b.sx = nyl * rkz(me, z), b.sf = plane * rkz(me, z);
                CUDA_TRY(skg::launch_box_copy(b, false, st, &c->launches));
            }
    }
    hook.end(4, bytes);
    return SKG_OK;
}

int dist_dt_update(skg_ctx* c, long* counter) {
    if (c->comm) {  // global max |u_d| over the ranks' x rows
        const ncclResult_t nr = nccl().AllReduce(c->d_dyn->umax, c->d_dyn->umax, 3, ncclDouble, ncclMax,
                                              c->comm, c->stream);
        if (nr != ncclSuccess) return fail(SKG_ENCCL, nccl().GetErrorString(nr));
    }
    CUDA_TRY(skg::launch_dt_update(c->d_dyn, c->flags, c->etab, c->dims, c->n, c->kscale, c->nu,
                                   c->stream, counter));
    return SKG_OK;
}

// One step of a slab-decomposed context.  ns2d: the x-forward of every stage
// runs fused with the next stage's x-inverse (first: the step opens the
// batch and runs its own stage-1 x-inverse; last: no next stage).
// ns3d slab step with the all-to-alls chunked per field on a second stream
// (copy / NCCL exchange): the x-inverse runs one velocity component per
// launch and the y-forward one field per launch, each followed by the
// exchange of the fields it produced on c->cstream, so the transfer of one
// overlaps the next one's pass; the compute stream joins the exchange stream
// before the consumers (y-inverse, x-forward) start.
int enqueue_dist_step3_chunked(skg_ctx* c, double dt, long* counter) {
    const int nst = c->scheme == SKG_RK2 ? 2 : 4;
    const skg::LaunchHook hook = hook_of(c);
    int rc;
    if (!c->cstream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        for (cudaEvent_t& e : c->xev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    auto run = [&](int pass, int st, int comp0, int ncomp) -> int {
        for (const Part& p : c->parts) {
            skg::Ns3dArgs a = args3d_part(c, dt, p);
            a.comp0 = comp0;
            a.ncomp = ncomp;
            CUDA_TRY(skg::ns3d_pass(a, pass, st, c->stream, counter, hook));
        }
        return SKG_OK;
    };
    auto fork = [&](int k, int which, unsigned fmask) -> int {
        CUDA_TRY(cudaEventRecord(c->xev[k], c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->cstream, c->xev[k], 0));
        int r2 = exchange3(c, which, fmask, c->cstream);
        ++*counter;
        return r2;
    };
    auto join = [&]() -> int {
        CUDA_TRY(cudaEventRecord(c->xev[6], c->cstream));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->xev[6], 0));
        return SKG_OK;
    };
    // fields of x-inverse component c: X[v_0]; X[v_1], X[kx v_1]; X[v_2], X[kx v_2]
    static const unsigned xfields[3] = {1u, 2u | 8u, 4u | 16u};
    for (int st = 1; st <= nst; ++st) {
        for (int comp = 0; comp < 3; ++comp)
            if ((rc = run(0, st, comp, 1)) || (rc = fork(comp, 0, xfields[comp]))) return rc;
        if ((rc = join()) || (rc = run(3, st, 0, 3))) return rc;
        for (int m = 0; m < 3; ++m)
            if ((rc = run(4, st, m, 1)) || (rc = fork(3 + m, 1, 1u << m))) return rc;
        if ((rc = join())) return rc;
        if (st == 1 && c->adaptive && (rc = dist_dt_update(c, counter))) return rc;
        if ((rc = run(2, st, 0, 3))) return rc;
    }
    return SKG_OK;
}

int enqueue_dist_step(skg_ctx* c, double dt, long* counter, bool first, bool last) {
    const int nst = c->scheme == SKG_RK2 ? 2 : 4;
    const skg::LaunchHook hook = hook_of(c);
    int rc;
    if (c->solver == 3 && !c->p2p && c->G > 1 && c->Pz == 1 && !c->timing && !c->no_overlap)
        return enqueue_dist_step3_chunked(c, dt, counter);
    if (c->solver == 3 && c->Pz > 1) {
        // pencil: x-inverse, all-to-all over the ky / x split, y-inverse,
        // kz -> y transpose, z pass on own (x, y) rows with all kept kz,
        // y -> kz transpose, y-forward, all-to-all back, x-forward + RK
        // kz -> y transpose fused into the y-inverse's stores wherever the
        // members' buffers are addressable (one process, or peer memory)
        const bool zfused = c->zfuse && (c->comm ? c->p2p : !c->zpack);
        auto run = [&](int pass, int st) -> int {
            for (const Part& p : c->parts) {
                skg::Ns3dArgs a = args3d_part(c, dt, p);
                if (pass == 6) {  // z pass: Z3 -> A3, nrl * nyl rows of all kept kz
                    a.B = p.Z3;
                    a.fstride = p.fsz;
                    a.ny = c->nyl;
                    a.kz_in = a.kz_o = c->kc[2] + 1;
                } else if (pass == 4) {  // y-forward input: fields 3..5 of B3
                    a.A = p.B3 + 3 * p.fs;
                } else if (pass == 5 && zfused) {  // y-inverse stores go to the members' Z3
                    a.zfused = 1;
                    a.nyl = c->nyl;
                    while ((1 << a.lg_nyl) < a.nyl) ++a.lg_nyl;
                    a.kzf = c->kc[2] + 1;
                    a.fsz = p.fsz;
                    for (int z = 0; z < c->Pz; ++z) {
                        if (c->comm) {
                            a.peer_Z[z] = c->peer_Z3[p.r * c->Pz + z];
                        } else {
                            for (const Part& q : c->parts)
                                if (q.r == p.r && q.pz == z) a.peer_Z[z] = q.Z3;
                        }
                    }
                }
                CUDA_TRY(skg::ns3d_pass(a, pass, st, c->stream, counter, hook));
            }
            return SKG_OK;
        };
        for (int st = 1; st <= nst; ++st) {
            if ((rc = run(0, st)) || (rc = exchange(c, 0))) return rc;
            if ((rc = run(5, st)) || (rc = exchange_z(c, zfused ? 2 : 0))) return rc;
            if ((rc = run(6, st)) || (rc = exchange_z(c, 1))) return rc;
            if ((rc = run(4, st)) || (rc = exchange(c, 1))) return rc;
            if (st == 1 && c->adaptive && (rc = dist_dt_update(c, counter))) return rc;
            if ((rc = run(2, st))) return rc;
        }
        return SKG_OK;
    }
    if (c->solver == 3) {
        for (int st = 1; st <= nst; ++st) {
            for (int pass = 0; pass < 3; ++pass) {
                for (const Part& p : c->parts) {
                    skg::Ns3dArgs a = args3d_part(c, dt, p);
                    CUDA_TRY(skg::ns3d_pass(a, pass, st, c->stream, counter, hook));
                }
                if (pass < 2 && (rc = exchange(c, pass))) return rc;
            }
            if (st == 1 && c->adaptive && (rc = dist_dt_update(c, counter))) return rc;
        }
        return SKG_OK;
    }
    auto run_pass = [&](int pass, int st, int next) -> int {
        for (const Part& p : c->parts) {
            skg::Ns2dArgs a = args2d_part(c, dt, p);
            a.lead = &p == c->parts.data() ? 1 : 0;
            CUDA_TRY(skg::ns2d_fast_pass(a, pass, st, c->stream, counter, hook, next));
        }
        return SKG_OK;
    };
    if (first) {
        if ((rc = run_pass(0, 1, 0)) || (rc = exchange(c, 0))) return rc;
    }
    for (int st = 1; st <= nst; ++st) {
        if ((rc = run_pass(1, st, 0)) || (rc = exchange(c, 1))) return rc;
        if (st == 1 && c->adaptive && (rc = dist_dt_update(c, counter))) return rc;
        const int next = st < nst || !last;
        if ((rc = run_pass(3, st, next))) return rc;
        if (next && (rc = exchange(c, 0))) return rc;
    }
    return SKG_OK;
}

int enqueue_steps(skg_ctx* c, double dt, long nsteps) {
    if (c->adaptive) dt = -1.0;  // device-resident: compute_dt per step
    else if (!(dt > 0.0)) return fail(SKG_ECONFIG, "step: nonpositive dt");
    if (nsteps < 0) return fail(SKG_ECONFIG, "step: negative step count");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->adaptive) {
        skg::DynStep d{};
        d.t = c->t;
        d.t_end = c->t_end;
        d.cfl = c->cfl;
        d.dt_max = c->dt_max;
        for (int k = 0; k < c->dims; ++k) d.dx[k] = c->L[k] / c->n[k];  // grid.cpp:50
        d.last_dt = c->last_dt;
        CUDA_TRY(cudaMemcpyAsync(c->d_dyn, &d, sizeof(d), cudaMemcpyHostToDevice, c->stream));
        c->cached_dt = -1.0;  // the device owns the factor tables now
    } else {
        int rc = refresh_exp(c, dt);
        if (rc) return rc;
    }
    skg::DevFlags init{0, std::numeric_limits<int>::max(), 0, 0};
    CUDA_TRY(cudaMemcpyAsync(c->flags, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    const int nst = c->scheme == SKG_RK2 ? 2 : 4;
    const skg::LaunchHook hook = hook_of(c);
    if (c->dist) {
        // first step eagerly, middle steps by replay of a captured step (the
        // NCCL calls and the exchange stream's fork/join are captured too),
        // the last step eagerly (ns2d: it closes the fused x-pass chain)
        long s = 0;
        if (nsteps > 0) {
            int rc2 = enqueue_dist_step(c, dt, &c->launches, true, nsteps == 1);
            if (rc2) return rc2;
            s = 1;
        }
        if (nsteps - s >= 3 && !c->timing && c->stream != nullptr) {
            if (c->gexec && (c->g_dt != dt || c->g_stream != c->stream || c->g_diag != c->diag ||
                             c->g_p2p != c->p2p)) {
                cudaGraphExecDestroy(c->gexec);
                c->gexec = nullptr;
            }
            if (!c->gexec) {
                cudaGraph_t graph;
                long dummy = 0;
                CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
                const int rc2 = enqueue_dist_step(c, dt, &dummy, false, false);
                cudaError_t e2 = cudaStreamEndCapture(c->stream, &graph);
                if (rc2) return rc2;
                CUDA_TRY(e2);
                CUDA_TRY(cudaGraphInstantiate(&c->gexec, graph, 0));
                cudaGraphDestroy(graph);
                c->g_launches = dummy;
                c->g_dt = dt;
                c->g_diag = c->diag;
                c->g_pruned = c->pruned;
                c->g_p2p = c->p2p;
                c->g_stream = c->stream;
            }
            for (; s < nsteps - 1; ++s) {
                CUDA_TRY(cudaGraphLaunch(c->gexec, c->stream));
                c->launches += c->g_launches;
            }
        }
        for (; s < nsteps; ++s) {
            int rc2 = enqueue_dist_step(c, dt, &c->launches, false, s == nsteps - 1);
            if (rc2) return rc2;
        }
        return SKG_OK;
    }
    // first: the step opens the batch; last: it closes it.  On the ns2d fast
    // path the x-forward of each stage is fused with the next stage's
    // x-inverse (across the step boundary too), so only the batch's first
    // step runs a standalone x-inverse and the last one no trailing one.
    auto one_step = [&](long* counter, bool first, bool last) -> cudaError_t {
        cudaError_t e = cudaSuccess;
        bool fused = false;
        auto dt_update = [&]() {
            return skg::launch_dt_update(c->d_dyn, c->flags, c->etab, c->dims, c->n, c->kscale, c->nu,
                                         c->stream, counter);
        };
        if (c->generic) {
            skg::GenArgs a = args_gen(c, dt);
            for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                e = skg::generic_stage(a, st, c->gs, c->stream, counter);
                if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
            }
        } else if (c->solver == 2) {
            skg::Ns2dArgs a = args2d(c, dt);
            fused = skg::ns2d_fast_ok(a);
            if (!fused) a.diag = nullptr;
            if (fused) {
                if (first) e = skg::ns2d_fast_pass(a, 0, 1, c->stream, counter, hook);
                for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                    e = skg::ns2d_fast_pass(a, 1, st, c->stream, counter, hook);
                    if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
                    if (e == cudaSuccess)
                        e = skg::ns2d_fast_pass(a, 3, st, c->stream, counter, hook, st < nst || !last);
                }
            } else {
                for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                    e = skg::ns2d_launch_stage(a, st, c->stream, counter, hook);
                    if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
                }
            }
        } else {
            skg::Ns3dArgs a = args3d(c, dt);
            fused = c->pruned;
            if (!fused) a.diag = nullptr;
            for (int st = 1; st <= nst && e == cudaSuccess; ++st) {
                e = skg::ns3d_launch_stage(a, st, c->stream, counter, hook);
                if (st == 1 && c->adaptive && e == cudaSuccess) e = dt_update();
            }
        }
        if (e == cudaSuccess && c->diag && !fused)  // unfused paths: one reduction per step
            e = skg::launch_energy(c->u, c->dims, c->n, c->kscale, c->nvars, energy_mode(c),
                                   c->diag, c->stream, counter, c->nu, &c->flags->steps, false);
        return e;
    };
    long s = 0;
    if (c->forcing) {  // host noise every step: no graph replay
        for (; s < nsteps; ++s) {
            int rc2 = refresh_forcing(c);
            if (rc2) return rc2;
            CUDA_TRY(one_step(&c->launches, s == 0, s == nsteps - 1));
        }
        return SKG_OK;
    }
    if (nsteps > 0) {  // first step eagerly (also sets kernel attributes)
        CUDA_TRY(one_step(&c->launches, true, nsteps == 1));
        s = 1;
    }
    // middle steps: replay of a captured step; the last step eagerly
    if (nsteps - s >= 3 && !c->timing && c->stream != nullptr) {
        if (c->gexec && (c->g_dt != dt || c->g_pruned != c->pruned || c->g_stream != c->stream ||
                         c->g_diag != c->diag || c->g_p2p != c->p2p)) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        if (!c->gexec) {
            cudaGraph_t graph;
            long dummy = 0;
            CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = one_step(&dummy, false, false);
            cudaError_t e2 = cudaStreamEndCapture(c->stream, &graph);
            CUDA_TRY(e);
            CUDA_TRY(e2);
            CUDA_TRY(cudaGraphInstantiate(&c->gexec, graph, 0));
            cudaGraphDestroy(graph);
            c->g_launches = dummy;
            c->g_dt = dt;
            c->g_diag = c->diag;
            c->g_pruned = c->pruned;
            c->g_p2p = c->p2p;
            c->g_stream = c->stream;
        }
        for (; s < nsteps - 1; ++s) {
            CUDA_TRY(cudaGraphLaunch(c->gexec, c->stream));
            c->launches += c->g_launches;
        }
    }
    for (; s < nsteps; ++s) CUDA_TRY(one_step(&c->launches, false, s == nsteps - 1));
    return SKG_OK;
}

}  // namespace skh
