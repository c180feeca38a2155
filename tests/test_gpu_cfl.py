"""Adaptive (CFL) time step on the device vs the reference with
time_stepping.fixed_dt = 0 (Simulation::compute_dt, simulation.cpp:463-476;
compute_cfl_dt, time_stepping.cpp:15-26; reference defaults cfl_coef 0.5,
dt_max 0.1, simulation.cpp:93-94).  The max |u_d| comes from the stage-1
physical pass of each step (no extra transforms); the reference runs 2 (ns2d)
or 3 (ns3d) extra c2r per step for it."""
import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
PARITY = 1e-10


def per_field(a, b):
    return max(O.rel_l2(a[v], b[v]) for v in range(a.shape[0]))


def _noise(n, nvars, seed):
    rng = np.random.default_rng(seed)
    return np.stack([O.forward(rng.standard_normal(n)) for _ in range(nvars)])


CASES = [
    ("ns2d", (64, 64), "ic", {}),
    ("ns2d", (256, 128), "ic", {}),
    ("ns2d", (32, 32), "noise", {}),          # general (not dealiased) path
    ("ns3d", (32, 32, 32), "ic", {}),
    ("ns3d", (16, 16, 16), "noise", {}),
    ("ns3d", (32, 32, 32), "ic", {"compact": True}),
    ("ns3d", (32, 64, 32), "ic", {"world": 2}),
    ("ns2d", (128, 128), "ic", {"world": 4}),
]


@pytest.mark.parametrize("solver,n,kind,kw", CASES,
                         ids=[f"{c[0]}-{'x'.join(map(str, c[1]))}-{c[2]}-{'-'.join(c[3]) or 'one'}"
                              for c in CASES])
def test_cfl_steps_match_reference(ref_lib, solver, n, kind, kw):
    nv = 1 if solver == "ns2d" else 3
    if kind == "ic":
        u0 = ic.initial_state(solver, n, seed=21)
    else:
        u0 = _noise(n, nv, 5) * (0.05 if solver == "ns2d" else 1.0)
    nu = 1e-3
    r = ref_lib.RefSimulation(solver, n, nu, 0.0)  # fixed_dt = 0: CFL 0.5, dt_max 0.1
    r.set_state(u0)
    g = api.Simulation(solver, n, nu, 0.0, **kw)
    g.set_cfl(0.5, 0.1)
    g.set_state(u0)
    for _ in range(3):
        r.step(2)
        g.step(2)
        assert abs(g.t - r.t) <= 1e-12 * r.t
        assert g.iteration == r.iteration
    assert per_field(g.get_state(), r.get_state()) < PARITY
    assert g.last_dt > 0


def test_cfl_dt_max_binds_and_graph_replay():
    n = (64, 64)
    u0 = ic.ns2d_ic(n, seed=3) * 1e-6   # tiny velocity: dt = dt_max
    g = api.Simulation("ns2d", n, 1e-3, 0.0)
    g.set_cfl(0.5, 2e-3)
    g.set_state(u0)
    g.step(7)                           # first step eager, the rest replayed
    assert g.last_dt == 2e-3
    assert abs(g.t - 7 * 2e-3) < 1e-15
    g.set_cfl(0.0)                      # back to a fixed dt
    g.step(2, dt=1e-3)
    assert g.last_dt == 1e-3
    assert abs(g.t - (7 * 2e-3 + 2e-3)) < 1e-15


@pytest.mark.parametrize("solver,n", [("ns2d", (64, 64)), ("ns3d", (16, 16, 16))])
def test_cfl_t_end_clamp(solver, n):
    u0 = ic.initial_state(solver, n, seed=4)
    g = api.Simulation(solver, n, 1e-3, 0.0)
    g.set_cfl(0.5, 0.05, t_end=0.12)
    g.set_state(u0)
    with pytest.raises(api.ConfigError):
        g.step(100)                     # stops at t_end: the next dt is 0
    assert g.t == pytest.approx(0.12, abs=1e-15)
    it = g.iteration
    assert it >= 3
    with pytest.raises(api.ConfigError):
        g.step(1)
    assert g.iteration == it


@pytest.mark.parametrize("solver,n,kind", [("ns2d", (64, 64), "ic"), ("ns2d", (32, 32), "noise"),
                                            ("ns3d", (16, 16, 16), "ic")])
def test_max_velocity_matches_physical_fields(solver, n, kind):
    """skg_max_velocity == max |u_d| of the c2r velocity components."""
    nv = 1 if solver == "ns2d" else 3
    u0 = ic.initial_state(solver, n, seed=2) if kind == "ic" else _noise(n, nv, 3)
    g = api.Simulation(solver, n, 1e-3, 1e-3)
    m = g.max_velocity(u0)
    if solver == "ns2d":
        kx, ky = O.k_axes(n)
        ksq = O.k_sq(n)
        psi = np.where(ksq == 0, 0, u0[0] / np.where(ksq == 0, 1, ksq))
        comps = [1j * ky[None, :] * psi, -1j * kx[:, None] * psi]
    else:
        comps = list(u0)
    ref = [np.abs(O.inverse(c, n)).max() for c in comps]
    assert np.allclose(m, ref, rtol=1e-13, atol=0)
