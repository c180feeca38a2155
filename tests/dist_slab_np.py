"""numpy model of the ns2d slab decomposition of libskgpu (csrc/skgpu.cu
create_impl / exchange, csrc/ns2d.cu fast-path kernels): the same column /
row partitions and the same pair-interleaved send/receive block layouts,
exchanged with torch.distributed.all_to_all_single.  Used by
tests/test_dist_cpu.py (gloo, world_size 2 and 4) to check the host-side
decomposition logic against the undecomposed oracle tendency.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import spectral_np as O


def partition(Kc, nx, G):
    PP = (Kc + 1) // 2
    cstart = [2 * (q * PP // G) for q in range(G)] + [Kc]
    return cstart, nx // G


def _a2a(send_blocks, recv_sizes, group=None):
    """all_to_all_single of complex blocks (lists indexed by peer; group: the
    sub-communicator of a pencil row / column, default the world)."""
    s = torch.from_numpy(np.concatenate([b.view(np.float64) for b in send_blocks]))
    r = torch.empty(2 * sum(recv_sizes), dtype=torch.float64)
    dist.all_to_all_single(r, s, output_split_sizes=[2 * x for x in recv_sizes],
                           input_split_sizes=[b.size * 2 for b in send_blocks], group=group)
    out, o = [], 0
    rn = r.numpy().view(np.complex128)
    for x in recv_sizes:
        out.append(rn[o:o + x])
        o += x
    return out


def slab_tendency(w_full, n, rank, G):
    """Dealiased-path tendency of the full state, computed on the slab of
    `rank`; returns this rank's kept columns of N_hat (CM layout [kyl][kx])."""
    nx, ny = n
    kx, ky = O.k_axes(n)
    kcx = int(np.abs(kx[O.dealias_mask((nx, ny))[:, 0].astype(bool)]).max())
    Kc = int(O.dealias_mask(n)[0].sum())
    cstart, nrl = partition(Kc, nx, G)
    c0, c1 = cstart[rank], cstart[rank + 1]
    ncols = c1 - c0
    # x-inverse of psi and kx psi on own columns (CM: column ky over kx)
    W = w_full[0][:, c0:c1]                               # (nx, ncols)
    KX = kx[:, None]
    KY = ky[None, c0:c1]
    ksq = KX ** 2 + KY ** 2
    psi = np.where(ksq == 0, 0, W / np.where(ksq == 0, 1, ksq))
    X0 = np.fft.ifft(psi, axis=0) * nx                    # (x, kyl)
    X1 = np.fft.ifft(KX * psi, axis=0) * nx
    # send block to q: rows(q) x own cols, ((xl/4) ncols + kyl) 4 + xl%4
    def pack_I(X, q):
        blk = X[q * nrl:(q + 1) * nrl, :]                 # (xl, kyl)
        return blk.reshape(nrl // 4, 4, ncols).transpose(0, 2, 1).reshape(-1).copy()
    rs = [nrl * (cstart[q + 1] - cstart[q]) for q in range(G)]
    R0 = _a2a([pack_I(X0, q) for q in range(G)], rs)
    R1 = _a2a([pack_I(X1, q) for q in range(G)], rs)
    # y pass on own rows: assemble rows over all kept ky from the owners
    def unpack_rows(R):
        cols = []
        for q in range(G):
            nc = cstart[q + 1] - cstart[q]
            cols.append(R[q].reshape(nrl // 4, nc, 4).transpose(0, 2, 1).reshape(nrl, nc))
        return np.concatenate(cols, axis=1)               # (xl, Kc)
    P0, P1 = unpack_rows(R0), unpack_rows(R1)
    kyk = ky[:Kc][None, :]
    uh = 1j * kyk * P0                                    # u: i ky X[psi]
    vh = -1j * P1                                         # v: -i X[kx psi]
    def c2r_rows(h):
        full = np.zeros((nrl, ny // 2 + 1), complex)
        full[:, :Kc] = h
        full[:, 0] = full[:, 0].real
        return np.fft.irfft(full, n=ny, axis=1) * ny
    u, v = c2r_rows(uh), c2r_rows(vh)
    A = np.fft.rfft(v * v - u * u, axis=1)[:, :Kc] / (nx * ny)
    B = np.fft.rfft(u * v, axis=1)[:, :Kc] / (nx * ny)
    # send to q: cols(q) x own rows, ((k/2) nrl + xl) 2 + k%2 in pair order
    def pack_A(M, q):
        a, b = cstart[q], cstart[q + 1]
        np_q = (b - a + 1) // 2
        blk = np.zeros((nrl, 2 * np_q), complex)
        blk[:, :b - a] = M[:, a:b]
        return blk.reshape(nrl, np_q, 2).transpose(1, 0, 2).reshape(-1).copy()
    npair_r = (ncols + 1) // 2
    RA = _a2a([pack_A(A, q) for q in range(G)], [2 * npair_r * nrl] * G)
    RB = _a2a([pack_A(B, q) for q in range(G)], [2 * npair_r * nrl] * G)
    def unpack_cols(R):
        rows = [R[q].reshape(npair_r, nrl, 2).transpose(1, 0, 2).reshape(nrl, 2 * npair_r)[:, :ncols]
                for q in range(G)]
        return np.concatenate(rows, axis=0)               # (x, kyl)
    Ah, Bh = np.fft.fft(unpack_cols(RA), axis=0), np.fft.fft(unpack_cols(RB), axis=0)
    N = KX * KY * Ah + (KX ** 2 - KY ** 2) * Bh
    keep = np.abs(kx)[:, None] <= kcx
    N = np.where(keep, N, 0)
    if c0 == 0:
        N[0, 0] = 0
    return N, c0, c1


# ------------------------------------------------------------------ ns3d
def partition3(Kyc, nx, G):
    """Compact kept ky lines [kstart[q], kstart[q+1]) and x rows nx / G of
    rank q (csrc/skgpu.cu create_impl, ns3d branch)."""
    return [q * Kyc // G for q in range(G + 1)], nx // G


def slab3d_tendency(v_full, n, rank, G):
    """Dealiased-path ns3d tendency computed on the slab of `rank` with the
    block layouts of csrc/skgpu.cu exchange3 and csrc/ns3d.cu (send blocks of
    the x-inverse [xl][kyl_r][kz], of the y-forward [xl][kyl_q][kz]); returns
    this rank's lines (3, nx, nkyl, kzc) and their global ky indices."""
    nx, ny, nz = n
    kx, ky, kz = O.k_axes(n)
    mask = O.dealias_mask(n).astype(bool)
    kcy = int(np.abs(ky[mask[0, :, 0]]).max() / (ky[1] - ky[0]) + 0.5)
    kcz = int(mask[0, 0].sum()) - 1
    Kyc, kzc = 2 * kcy + 1, kcz + 1
    gky = np.array(list(range(kcy + 1)) + list(range(ny - kcy, ny)))   # compact -> global
    kstart, nrl = partition3(Kyc, nx, G)
    c0, c1 = kstart[rank], kstart[rank + 1]
    nl = [kstart[q + 1] - kstart[q] for q in range(G)]
    V = v_full[:, :, gky[c0:c1], :kzc]                     # (3, nx, nkyl, kzc)
    KX = kx[:, None, None]
    # x-inverse: vx, vy, vz, kx vy, kx vz
    F = [V[0], V[1], V[2], KX * V[1], KX * V[2]]
    X = [np.fft.ifft(f, axis=0) * nx for f in F]           # (x, kyl, kz)
    sizes = [nrl * nl[q] * kzc for q in range(G)]
    R = [_a2a([x[q * nrl:(q + 1) * nrl].reshape(-1).copy() for q in range(G)], sizes) for x in X]
    def lines(Rf):   # (xl, Kyc, kz) from the owners' blocks
        return np.concatenate([Rf[q].reshape(nrl, nl[q], kzc) for q in range(G)], axis=1)
    P = [lines(Rf) for Rf in R]
    KY = ky[gky][None, :, None]
    KZ = kz[:kzc][None, None, :]
    spec = [P[0], P[1], P[2],
            1j * KY * P[2] - 1j * KZ * P[1],               # wx
            1j * KZ * P[0] - 1j * P[4],                    # wy = i kz vx - i kx vz
            1j * P[3] - 1j * KY * P[0]]                    # wz = i kx vy - i ky vx
    def to_phys(h):
        full = np.zeros((nrl, ny, nz // 2 + 1), complex)
        full[:, gky, :kzc] = h
        y = np.fft.ifft(full, axis=1) * ny
        y[..., 0] = y[..., 0].real
        y[..., -1] = y[..., -1].real
        return np.fft.irfft(y, n=nz, axis=2) * nz
    ux, uy, uz, ox, oy, oz = (to_phys(h) for h in spec)
    cross = [uy * oz - uz * oy, uz * ox - ux * oz, ux * oy - uy * ox]
    def to_spec(c):
        s = np.fft.fft(np.fft.rfft(c, axis=2)[..., :kzc], axis=1)[:, gky, :] / (nx * ny * nz)
        return s                                            # (xl, Kyc, kz)
    D = [to_spec(c) for c in cross]
    sizes = [nrl * nl[rank] * kzc] * G
    RD = [_a2a([d[:, kstart[q]:kstart[q + 1]].reshape(-1).copy() for q in range(G)], sizes) for d in D]
    out = [np.fft.fft(np.concatenate([r[q].reshape(nrl, nl[rank], kzc) for q in range(G)], axis=0), axis=0)
           for r in RD]
    KYl = ky[gky[c0:c1]][None, :, None]
    ksq = KX ** 2 + KYl ** 2 + KZ ** 2
    nzm = ksq != 0
    s = (KX * out[0] + KYl * out[1] + KZ * out[2]) / np.where(nzm, ksq, 1.0)
    out = [np.where(nzm, out[0] - KX * s, out[0]), np.where(nzm, out[1] - KYl * s, out[1]),
           np.where(nzm, out[2] - KZ * s, out[2])]
    keep = mask[:, gky[c0:c1], :kzc]
    out = np.stack([np.where(keep, o, 0) for o in out])
    if c0 == 0:
        out[:, 0, 0, 0] = 0
    return out, gky[c0:c1], kzc


# ------------------------------------------------------------------ ns3d pencil
def pencil_groups(py, pz):
    """Sub-communicators of the py x pz process grid (global rank = r_y pz +
    r_z, csrc/skgpu.cu skg_create_pencil): for every rank its ky / x group
    (equal r_z, py members) and its kz / y group (equal r_y, pz members).
    Collective: every rank creates all groups in the same order."""
    gy = [dist.new_group([q * pz + z for q in range(py)]) for z in range(pz)]
    gz = [dist.new_group([r * pz + z for z in range(pz)]) for r in range(py)]
    return gy, gz


def pencil3d_tendency(v_full, n, rank, py, pz, groups):
    """Dealiased-path ns3d tendency on part (r_y, r_z) of the pencil layout
    with the block layouts of csrc/host_step.cu exchange3 (inside the ky / x
    group, per-part kz range) and exchange_z (the kz <-> y transposes, NCCL
    route: contiguous [xl][yl][kz] blocks per member).  Returns this part's
    lines (3, nx, nkyl, nkz), their global ky indices and the kz range."""
    nx, ny, nz = n
    ry, rz = divmod(rank, pz)
    gy, gz = groups[0][rz], groups[1][ry]
    kx, ky, kz = O.k_axes(n)
    mask = O.dealias_mask(n).astype(bool)
    kcy = int(np.abs(ky[mask[0, :, 0]]).max() / (ky[1] - ky[0]) + 0.5)
    kzc = int(mask[0, 0].sum())
    Kyc = 2 * kcy + 1
    gky = np.array(list(range(kcy + 1)) + list(range(ny - kcy, ny)))
    kstart, nrl = partition3(Kyc, nx, py)
    zstart = [z * kzc // pz for z in range(pz + 1)]
    nkzs = [zstart[z + 1] - zstart[z] for z in range(pz)]
    k0, k1 = zstart[rz], zstart[rz + 1]
    nkz, nyl = k1 - k0, ny // pz
    c0, c1 = kstart[ry], kstart[ry + 1]
    nl = [kstart[q + 1] - kstart[q] for q in range(py)]
    V = v_full[:, :, gky[c0:c1], k0:k1]                    # (3, nx, nkyl, nkz)
    KX = kx[:, None, None]
    X = [np.fft.ifft(f, axis=0) * nx for f in (V[0], V[1], V[2], KX * V[1], KX * V[2])]
    sizes = [nrl * nl[q] * nkz for q in range(py)]
    R = [_a2a([x[q * nrl:(q + 1) * nrl].reshape(-1).copy() for q in range(py)], sizes, gy) for x in X]
    P = [np.concatenate([Rf[q].reshape(nrl, nl[q], nkz) for q in range(py)], axis=1) for Rf in R]
    KY = ky[gky][None, :, None]
    KZ = kz[k0:k1][None, None, :]
    spec = [P[0], P[1], P[2], 1j * KY * P[2] - 1j * KZ * P[1], 1j * KZ * P[0] - 1j * P[4],
            1j * P[3] - 1j * KY * P[0]]
    def y_inverse(h):                                      # (xl, ny, nkz)
        full = np.zeros((nrl, ny, nkz), complex)
        full[:, gky, :] = h
        return np.fft.ifft(full, axis=1) * ny
    def kz_to_y(f):                                        # -> (xl, nyl, kzc)
        rs = [nrl * nyl * nkzs[z] for z in range(pz)]
        got = _a2a([f[:, z * nyl:(z + 1) * nyl, :].reshape(-1).copy() for z in range(pz)], rs, gz)
        return np.concatenate([got[z].reshape(nrl, nyl, nkzs[z]) for z in range(pz)], axis=2)
    def c2r_z(h):
        full = np.zeros((nrl, nyl, nz // 2 + 1), complex)
        full[..., :kzc] = h
        full[..., 0] = full[..., 0].real
        return np.fft.irfft(full, n=nz, axis=2) * nz
    ux, uy, uz, ox, oy, oz = (c2r_z(kz_to_y(y_inverse(h))) for h in spec)
    cross = [uy * oz - uz * oy, uz * ox - ux * oz, ux * oy - uy * ox]
    def y_to_kz(c):                                        # (xl, nyl, kzc) -> (xl, ny, nkz)
        rs = [nrl * nyl * nkz] * pz
        got = _a2a([c[:, :, zstart[z]:zstart[z + 1]].reshape(-1).copy() for z in range(pz)], rs, gz)
        return np.concatenate([got[z].reshape(nrl, nyl, nkz) for z in range(pz)], axis=1)
    D = [np.fft.fft(y_to_kz(np.fft.rfft(c, axis=2)[..., :kzc] / (nx * ny * nz)), axis=1)[:, gky, :]
         for c in cross]                                   # (xl, Kyc, nkz)
    sizes = [nrl * nl[ry] * nkz] * py
    RD = [_a2a([d[:, kstart[q]:kstart[q + 1]].reshape(-1).copy() for q in range(py)], sizes, gy) for d in D]
    out = [np.fft.fft(np.concatenate([r[q].reshape(nrl, nl[ry], nkz) for q in range(py)], axis=0), axis=0)
           for r in RD]
    KYl = ky[gky[c0:c1]][None, :, None]
    ksq = KX ** 2 + KYl ** 2 + KZ ** 2
    nzm = ksq != 0
    s = (KX * out[0] + KYl * out[1] + KZ * out[2]) / np.where(nzm, ksq, 1.0)
    out = [np.where(nzm, out[0] - KX * s, out[0]), np.where(nzm, out[1] - KYl * s, out[1]),
           np.where(nzm, out[2] - KZ * s, out[2])]
    keep = mask[:, gky[c0:c1], k0:k1]
    out = np.stack([np.where(keep, o, 0) for o in out])
    if c0 == 0 and k0 == 0:
        out[:, 0, 0, 0] = 0
    return out, gky[c0:c1], (k0, k1)
