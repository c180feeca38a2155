"""numpy restatement of the reference hot path (CPU oracle, secondary).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import it.

Independent of oracle/_ref (the compiled reference): the transforms here are
numpy's pocketfft, so agreement between this module and oracle/_ref also pins
oracle/fft_shim.c.  Each function cites the reference lines it restates
(paths relative to /root/reference/proj).
"""
from __future__ import annotations

import numpy as np

K_TWO_PI = 6.283185307179586476925286766559  # src/grid.cpp:11


# ----------------------------------------------------------------- grid
def k_axes(n, L=None):
    """k_axis per axis, src/grid.cpp:49-63: spacing*signed_i on full axes
    (Nyquist -> +n/2), spacing*i on the half-stored last axis."""
    d = len(n)
    L = [K_TWO_PI] * d if L is None else list(L)
    ks = []
    for a in range(d):
        spacing = K_TWO_PI / L[a]
        if a == d - 1:
            idx = np.arange(n[a] // 2 + 1)
        else:
            i = np.arange(n[a])
            idx = np.where(i <= n[a] // 2, i, i - n[a])
        ks.append(spacing * idx.astype(np.float64))
    return ks


def dealias_mask(n, L=None, coef=2.0 / 3.0):
    """uint8 mask, src/grid.cpp:78-100: keep iff |k_d| <= coef*(2pi/L_d)*(n_d/2)
    for every axis (same left-to-right double arithmetic)."""
    d = len(n)
    L = [K_TWO_PI] * d if L is None else list(L)
    ks = k_axes(n, L)
    keep = None
    for a in range(d):
        kcut = coef * (K_TWO_PI / L[a]) * float(n[a] // 2)
        ok = np.abs(ks[a]) <= kcut
        shape = [1] * d
        shape[a] = ks[a].size
        ok = ok.reshape(shape)
        keep = ok if keep is None else keep & ok
    return keep.astype(np.uint8)


def k_sq(n, L=None):
    """|k|^2 per stored mode, src/grid.cpp:84-86 (k0*k0 + k1*k1 + k2*k2 order)."""
    ks = k_axes(n, L)
    d = len(n)
    pad = [np.zeros(1)] * (3 - d) + ks
    k0 = pad[0][:, None, None]
    k1 = pad[1][None, :, None]
    k2 = pad[2][None, None, :]
    return (k0 * k0 + k1 * k1 + k2 * k2).reshape(tuple(x.size for x in ks))


def parseval_w(n):
    """1 on last-axis index 0 and Nyquist, else 2 (src/grid.cpp:96-98)."""
    h = n[-1] // 2 + 1
    w = np.full(h, 2.0)
    w[0] = 1.0
    w[-1] = 1.0
    return np.broadcast_to(w, tuple(n[:-1]) + (h,))


# ------------------------------------------------------------ transforms
def forward(u):
    """FftPlan::forward, src/fft.cpp:92-98: unnormalised r2c, then *= 1/N."""
    return np.fft.rfftn(u) * (1.0 / u.size)


def inverse(uhat, shape):
    """FftPlan::inverse, src/fft.cpp:100-106: unnormalised c2r."""
    return np.fft.irfftn(uhat, s=tuple(shape), axes=tuple(range(len(shape))), norm="forward")


# ------------------------------------------------------------- tendencies
def tendency_ns2d(w, n):
    """Ns2dSolver::tendency, src/solvers.cpp:133-174 (input not dealiased)."""
    w = w[0]
    kx, ky = k_axes(n)
    KX = kx[:, None]
    KY = ky[None, :]
    ksq = k_sq(n)
    with np.errstate(divide="ignore", invalid="ignore"):
        psi = np.where(ksq == 0.0, 0.0, w / np.where(ksq == 0.0, 1.0, ksq))  # grid.cpp:262-270
    ux_h = 1j * KY * psi                      # i ky psi  (grid.cpp:271)
    uy_h = -1j * KX * psi                     # -i kx psi (grid.cpp:272)
    ux = inverse(ux_h, n)
    uy = inverse(uy_h, n)
    dwx = inverse(1j * KX * w, n)             # gradient_component axis 0 (grid.cpp:124-143)
    dwy = inverse(1j * KY * w, n)
    prod = -(ux * dwx + uy * dwy)             # solvers.cpp:160-164
    out = forward(prod)
    out = out * dealias_mask(n)               # grid.cpp:112-118 (exact zero where masked)
    out[0, 0] = 0.0                           # solvers.cpp:172
    return out[None]


def tendency_ns3d(v, n):
    """Ns3dSolver::tendency, src/solvers.cpp:299-339."""
    kx, ky, kz = k_axes(n)
    KX = kx[:, None, None]
    KY = ky[None, :, None]
    KZ = kz[None, None, :]
    vx, vy, vz = v
    wx = 1j * KY * vz - 1j * KZ * vy          # curl3d, grid.cpp:195-203
    wy = 1j * KZ * vx - 1j * KX * vz
    wz = 1j * KX * vy - 1j * KY * vx
    ux, uy, uz = (inverse(a, n) for a in (vx, vy, vz))
    ox, oy, oz = (inverse(a, n) for a in (wx, wy, wz))
    cx = uy * oz - uz * oy                    # solvers.cpp:321-325
    cy = uz * ox - ux * oz
    cz = ux * oy - uy * ox
    out = np.stack([forward(c) for c in (cx, cy, cz)])
    ksq = k_sq(n)
    nz = ksq != 0.0
    s = (KX * out[0] + KY * out[1] + KZ * out[2]) / np.where(nz, ksq, 1.0)  # grid.cpp:227-249
    out[0] = np.where(nz, out[0] - KX * s, out[0])
    out[1] = np.where(nz, out[1] - KY * s, out[1])
    out[2] = np.where(nz, out[2] - KZ * s, out[2])
    out = out * dealias_mask(n)[None]
    out[:, 0, 0, 0] = 0.0                     # solvers.cpp:337
    return out


TENDENCY = {"ns2d": tendency_ns2d, "ns3d": tendency_ns3d}


# --------------------------------------------------------------- stepper
def rk4_step(u, dt, nu, n, solver):
    """ExactLinStepper::step RK4 branch, src/time_stepping.cpp:121-193, with
    sigma = -nu |k|^2 (src/simulation.cpp:147-157) and E1/E2 from
    refresh_exp (time_stepping.cpp:37-57)."""
    f = TENDENCY[solver]
    if nu == 0.0:
        hdt = 0.5 * dt
        k1 = f(u, n)
        k2 = f(u + hdt * k1, n)
        k3 = f(u + hdt * k2, n)
        k4 = f(u + dt * k3, n)
        sdt = dt / 6.0
        delta = sdt * (k1 + 2.0 * (k2 + k3) + k4)
        return np.where(delta != 0.0, u + delta, u)
    sigma = -nu * k_sq(n)
    e1 = np.exp(0.5 * dt * sigma)
    e2 = np.exp(dt * sigma)
    hdt = 0.5 * dt
    k1 = f(u, n)
    k2 = f(e1 * (u + hdt * k1), n)
    k3 = f(e1 * u + hdt * k2, n)
    k4 = f(e2 * u + dt * e1 * k3, n)
    sdt = dt / 6.0
    return e2 * u + sdt * (e2 * k1 + 2.0 * e1 * (k2 + k3) + k4)


def rk2_step(u, dt, nu, n, solver):
    """ExactLinStepper::step RK2 branch, src/time_stepping.cpp:82-119."""
    f = TENDENCY[solver]
    hdt = 0.5 * dt
    if nu == 0.0:
        k1 = f(u, n)
        k2 = f(u + hdt * k1, n)
        delta = dt * k2
        return np.where(delta != 0.0, u + delta, u)
    sigma = -nu * k_sq(n)
    e1 = np.exp(0.5 * dt * sigma)
    e2 = np.exp(dt * sigma)
    k1 = f(u, n)
    k2 = f(e1 * (u + hdt * k1), n)
    return e2 * u + dt * e1 * k2


# ----------------------------------------------------------- diagnostics
def energy(u, n, solver):
    """Simulation::energy via mode_energy (solvers.cpp:211-218 for ns2d;
    Solver::mode_energy default 0.5*w*|u|^2 summed over variables for ns3d)."""
    w = parseval_w(n)
    if solver == "ns2d":
        ksq = k_sq(n)
        e = np.where(ksq > 0.0, 0.5 * w * np.abs(u[0]) ** 2 / np.where(ksq > 0, ksq, 1.0), 0.0)
        return float(e.sum())
    return float(sum((0.5 * w * np.abs(x) ** 2).sum() for x in u))


def rel_l2(a, b):
    """Parity metric of SURVEY 8(c): ||a - b||_2 / ||b||_2 over stored modes."""
    nb = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0))
