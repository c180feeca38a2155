"""Seeded synthetic initial conditions for the BASELINE configs.

The reference has no such IC (its own bench uses ``random_field`` unit-phase
noise, proj/src/grid.cpp:276-306); BASELINE.json's configs ask for complex
Gaussian noise shaped to an energy spectrum, Hermitian-symmetric, zero mean,
dealiased and normalised.  These stand in for the paper's runs (DESIGN.md
"Synthetic inputs").  Generated on the host with numpy's PCG64 so that the
oracle and the GPU consume byte-identical inputs.

Recipe:
  ns2d: omega_hat = g(|k|) * (complex Gaussian), g = sqrt(k E(k)),
        E(k) = k^4 exp(-2 (k/6)^2) (peak at |k| = 6, inside 4 <= |k| <= 8),
        Hermitian planes symmetrised, dealiased, mean 0, rescaled to
        E = sum w |w_hat|^2 / (2|k|^2) = 1 (unit rms velocity per component).
  ns3d: per component g = sqrt(E(k))/k, E(k) = k^4 exp(-2 (k/k0)^2), k0 = 4,
        Leray-projected, dealiased, mean 0, rescaled to E = 1.5.
"""
from __future__ import annotations

import numpy as np

K_TWO_PI = 6.283185307179586476925286766559


def _k_axes(n):
    ks = []
    d = len(n)
    for a in range(d):
        if a == d - 1:
            idx = np.arange(n[a] // 2 + 1)
        else:
            i = np.arange(n[a])
            idx = np.where(i <= n[a] // 2, i, i - n[a])
        ks.append((K_TWO_PI / K_TWO_PI) * idx.astype(np.float64))
    return ks


def _mask(n, coef=2.0 / 3.0):
    ks = _k_axes(n)
    d = len(n)
    keep = None
    for a in range(d):
        kcut = coef * 1.0 * float(n[a] // 2)
        shape = [1] * d
        shape[a] = ks[a].size
        ok = (np.abs(ks[a]) <= kcut).reshape(shape)
        keep = ok if keep is None else keep & ok
    return keep


def _ksq(n):
    ks = _k_axes(n)
    d = len(n)
    out = 0.0
    for a in range(d):
        shape = [1] * d
        shape[a] = ks[a].size
        out = out + (ks[a] * ks[a]).reshape(shape)
    return out


def _hermitian_planes(f, n):
    """Make the self-conjugate planes (last-axis index 0 and Nyquist) of a
    half-stored spectrum Hermitian: f(-k) = conj(f(k)) over the full axes."""
    d = len(n)
    for j in (0, n[-1] // 2):
        plane = f[..., j]
        flipped = plane
        for a in range(d - 1):
            flipped = np.roll(np.flip(flipped, axis=a), 1, axis=a)
        f[..., j] = 0.5 * (plane + np.conj(flipped))
    return f


def _noise(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def ns2d_ic(n, seed=1234, energy=1.0, kp=6.0):
    n = tuple(int(x) for x in n)
    rng = np.random.default_rng(seed)
    ksq = _ksq(n)
    k = np.sqrt(ksq)
    E = k ** 4 * np.exp(-2.0 * (k / kp) ** 2)
    g = np.sqrt(k * E)
    w = _noise(rng, ksq.shape) * g
    w = _hermitian_planes(w, n)
    w = np.where(_mask(n), w, 0.0)
    w[0, 0] = 0.0
    # energy = sum w_k |w_hat|^2 / (2|k|^2)   (proj/src/solvers.cpp:211-218)
    pw = np.full(n[-1] // 2 + 1, 2.0)
    pw[0] = pw[-1] = 1.0
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.where(ksq > 0, 0.5 * pw * np.abs(w) ** 2 / np.where(ksq > 0, ksq, 1.0), 0.0).sum()
    w *= np.sqrt(energy / e)
    return w[None].astype(np.complex128)


def ns3d_ic(n, seed=1234, energy=1.5, k0=4.0):
    n = tuple(int(x) for x in n)
    rng = np.random.default_rng(seed)
    ksq = _ksq(n)
    k = np.sqrt(ksq)
    E = k ** 4 * np.exp(-2.0 * (k / k0) ** 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        g = np.where(k > 0, np.sqrt(E) / np.where(k > 0, k, 1.0), 0.0)
    v = np.stack([_hermitian_planes(_noise(rng, ksq.shape) * g, n) for _ in range(3)])
    kx, ky, kz = _k_axes(n)
    KX, KY, KZ = kx[:, None, None], ky[None, :, None], kz[None, None, :]
    nz = ksq != 0
    s = (KX * v[0] + KY * v[1] + KZ * v[2]) / np.where(nz, ksq, 1.0)
    v[0] = np.where(nz, v[0] - KX * s, v[0])
    v[1] = np.where(nz, v[1] - KY * s, v[1])
    v[2] = np.where(nz, v[2] - KZ * s, v[2])
    v = np.where(_mask(n)[None], v, 0.0)
    v[:, 0, 0, 0] = 0.0
    pw = np.full(n[-1] // 2 + 1, 2.0)
    pw[0] = pw[-1] = 1.0
    e = (0.5 * pw * np.abs(v) ** 2).sum()
    v *= np.sqrt(energy / e)
    return v.astype(np.complex128)


def initial_state(solver, n, seed=1234):
    return ns2d_ic(n, seed) if solver == "ns2d" else ns3d_ic(n, seed)


def cfl_dt(solver, n, state, cfl=0.5, dt_max=0.1):
    """dt = min(dt_max, cfl * min_d dx_d / max|u_d|) from the IC, as
    compute_cfl_dt (proj/src/time_stepping.cpp:15-26) with max|u_d| from
    max_velocity_per_axis (proj/src/solvers.cpp:176-194, 341-357)."""
    n = tuple(n)
    if solver == "ns2d":
        kx, ky = _k_axes(n)
        ksq = _ksq(n)
        with np.errstate(divide="ignore", invalid="ignore"):
            psi = np.where(ksq == 0, 0.0, state[0] / np.where(ksq == 0, 1.0, ksq))
        comps = [1j * ky[None, :] * psi, -1j * kx[:, None] * psi]
    else:
        comps = list(state)
    dt = dt_max
    dx = K_TWO_PI / n[0]
    for a, c in enumerate(comps):
        u = np.fft.irfftn(c, s=n, axes=tuple(range(len(n))), norm="forward")
        vel = max(float(np.abs(u).max()), 1e-30)
        dt = min(dt, cfl * (K_TWO_PI / n[a]) / vel)
    return dt


def embed(v, n):
    """Spectral embedding of a dealiased half-spectrum state v (vars, n0, ..,
    n_last//2+1) of a coarser grid into grid n: the same modes (same signed
    indices) with zeros elsewhere.  The physical field is the same
    band-limited function sampled finer (1/N-forward convention), so the
    BASELINE recipe at a large n is generated at a coarse grid holding all of
    its spectral energy (E(k) ~ k^4 exp(-2 (k/k0)^2) is below 1e-200 of its
    peak beyond |k| = 64) and embedded."""
    small = v.shape[1:-1] + (2 * (v.shape[-1] - 1),)
    d = len(n)
    out = np.zeros((v.shape[0],) + tuple(n[:-1]) + (n[-1] // 2 + 1,), np.complex128)
    idx = []
    for a in range(d - 1):
        i = np.arange(small[a])
        si = np.where(i <= small[a] // 2, i, i - small[a])
        keep = np.abs(si) < small[a] // 2          # the coarse Nyquist is masked anyway
        idx.append((i[keep], np.where(si[keep] >= 0, si[keep], si[keep] + n[a])))
    kz = small[-1] // 2                            # coarse Nyquist plane excluded
    if d == 2:
        out[:, idx[0][1][:, None], np.arange(kz)[None, :]] = v[:, idx[0][0][:, None], np.arange(kz)[None, :]]
    else:
        src = v[:, idx[0][0]][:, :, idx[1][0], :kz]
        out[:, idx[0][1][:, None], idx[1][1][None, :], :kz] = src
    return out
