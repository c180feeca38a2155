"""The Python mirror of the reference's Simulation binding
(python/src/bindings.cpp:93-140): parameter-tree construction, stopping
rules, compute_dt, diagnostics, get_phys/set_phys."""
import math

import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu


def per_field(a, b):
    return max(O.rel_l2(a[v], b[v]) for v in range(a.shape[0]))


@pytest.mark.parametrize("solver,n", [("ns2d", (64, 32)), ("ns3d", (16, 16, 32)), ("ns2d", (24, 24))])
def test_get_set_phys(solver, n):
    u0 = ic.initial_state(solver, n, seed=3)
    g = api.Simulation(solver, n, 1e-3, 1e-3)
    g.set_state(u0)
    assert g.state_keys == (["rot"] if solver == "ns2d" else ["vx", "vy", "vz"])
    for i, key in enumerate(g.state_keys):
        assert np.abs(g.get_phys(key) - O.inverse(u0[i], n)).max() < 1e-12
    kx, ky = O.k_axes(n)[:2]
    if solver == "ns2d":
        ksq = O.k_sq(n)
        psi = np.where(ksq == 0, 0, u0[0] / np.where(ksq == 0, 1, ksq))
        assert np.abs(g.get_phys("ux") - O.inverse(1j * ky[None, :] * psi, n)).max() < 1e-12
        assert np.abs(g.get_phys("uy") - O.inverse(-1j * kx[:, None] * psi, n)).max() < 1e-12
    else:
        rz = 1j * kx[:, None, None] * u0[1] - 1j * ky[None, :, None] * u0[0]
        assert np.abs(g.get_phys("rotz") - O.inverse(rz, n)).max() < 1e-12
    with pytest.raises(api.ConfigError):
        g.get_phys("nope")
    # load_phys: forward transform of the values replaces one variable
    phys = g.get_phys(g.state_keys[0])
    g.set_phys(g.state_keys[0], 2.0 * phys)
    assert np.abs(g.get_state()[0] - 2.0 * u0[0]).max() < 1e-12
    with pytest.raises(api.ShapeError):
        g.set_phys(g.state_keys[0], np.zeros(4))


def test_from_params_cfl_run_matches_reference(ref_lib):
    n = (64, 64)
    u0 = ic.ns2d_ic(n, seed=8)
    params = {"solver": "ns2d", "nu_2": 1e-3, "oper.nx": 64, "oper.ny": 64,
              "time_stepping.fixed_dt": 0.0, "time_stepping.n_iters": 5, "time_stepping.t_end": -1.0}
    g = api.Simulation.from_params(params)
    g.set_state(u0)
    assert math.isclose(g.compute_dt(), ic.cfl_dt("ns2d", n, u0), rel_tol=1e-12)
    summary = g.run()
    assert summary["iterations"] == 5 and summary["means"].shape == (5, 3)
    r = ref_lib.RefSimulation("ns2d", n, 1e-3, 0.0)
    r.set_state(u0)
    r.step(5)
    assert abs(summary["t_final"] - r.t) <= 1e-12 * r.t
    assert per_field(g.get_state(), r.get_state()) < 1e-10
    e, z, eps = g.diagnostics()
    assert abs(e - r.energy) <= 1e-12 * r.energy and abs(z - r.enstrophy) <= 1e-12 * r.enstrophy
    assert abs(g.dissipation_rate() - eps) <= 1e-13 * eps  # atomic summation order
    assert abs(summary["means"][-1, 2] - eps) <= 1e-12 * eps


def test_params_rules():
    with pytest.raises(api.ConfigError):  # both stopping rules
        api.Simulation.from_params({"solver": "ns2d", "time_stepping.n_iters": 3,
                                    "time_stepping.t_end": 1.0})
    with pytest.raises(api.ConfigError):
        api.Simulation.from_params({"solver": "ns9d"})


@pytest.mark.parametrize("solver,n", [("ns2d", (32, 32)), ("ns3d", (16, 16, 16))])
def test_t_end_with_fixed_dt(solver, n):
    """compute_dt clamps the last step to t_end (simulation.cpp:471-474)."""
    u0 = ic.initial_state(solver, n, seed=2)
    dt = 1e-3
    g = api.Simulation(solver, n, 1e-3, dt)
    g.set_state(u0)
    g.set_t_end(5.5 * dt)
    summary = g.run()
    assert summary["iterations"] == 6
    assert abs(g.t - 5.5 * dt) < 1e-15
    h = api.Simulation(solver, n, 1e-3, dt)
    h.set_state(u0)
    h.step(5)
    h.step(1, dt=5.5 * dt - h.t)
    assert per_field(g.get_state(), h.get_state()) == 0.0
    assert g.run()["iterations"] == 0  # already at t_end


@pytest.mark.parametrize("solver,n", [("ns2d", (32, 32)), ("ns2d", (24, 40)), ("ns3d", (16, 16, 16)),
                                      ("ns3d", (12, 12, 12))])
def test_sanitize_state(solver, n):
    """Solver::sanitize_state (solvers.cpp:263-267, 377-381) on the device."""
    nv = 1 if solver == "ns2d" else 3
    rng = np.random.default_rng(6)
    v = np.stack([O.forward(rng.standard_normal(n)) for _ in range(nv)])
    g = api.Simulation(solver, n, 1e-3, 1e-3)
    g.set_state(v)
    assert not g.pruned
    g.sanitize_state()
    mask = O.dealias_mask(n)
    if solver == "ns2d":
        ref = v * mask[None]
        ref[0, 0, 0] = 0.0
    else:
        kx, ky, kz = O.k_axes(n)
        K = [kx[:, None, None], ky[None, :, None], kz[None, None, :]]
        ksq = O.k_sq(n)
        s = (K[0] * v[0] + K[1] * v[1] + K[2] * v[2]) / np.where(ksq == 0, 1.0, ksq)
        ref = np.stack([np.where(ksq == 0, v[c], v[c] - K[c] * s) for c in range(3)]) * mask[None]
    out = g.get_state()
    assert np.abs(out - ref).max() <= 1e-15 * np.abs(ref).max()
    assert g.pruned or n[0] % 2  # masked modes are now exactly zero


@pytest.mark.parametrize("solver,n", [("ns2d", (64, 64)), ("ns2d", (24, 40)), ("ns3d", (16, 16, 16))])
def test_spectra_match_reference_definitions(ref_lib, solver, n):
    """OutputManager's shell spectra (output.cpp:231-257) from the GPU state and
    tendency vs the same binning of the reference's tendency (numpy)."""
    u0 = ic.initial_state(solver, n, seed=5)
    nu = 1e-3
    g = api.Simulation(solver, n, nu, 1e-3)
    g.set_state(u0)
    sp = g.spectra()
    nl = ref_lib.RefSimulation(solver, n, nu, 1e-3).tendency(u0)
    ksq = O.k_sq(n)
    w = O.parseval_w(n)
    dk = 1.0
    shell = np.rint(np.sqrt(ksq) / dk).astype(int)
    nsh = int(np.rint(np.sqrt(ksq).max() / dk)) + 1
    if solver == "ns2d":
        s = np.where(ksq > 0, w / np.where(ksq > 0, ksq, 1.0), 0.0)
        e = 0.5 * s * np.abs(u0[0]) ** 2
        t = s * (u0[0].real * nl[0].real + u0[0].imag * nl[0].imag)
    else:
        e = 0.5 * w * sum(np.abs(u0[c]) ** 2 for c in range(3))
        t = w * sum(u0[c].real * nl[c].real + u0[c].imag * nl[c].imag for c in range(3))
    E = np.bincount(shell.ravel(), e.ravel(), nsh) / dk
    T = np.bincount(shell.ravel(), t.ravel(), nsh)
    D = np.bincount(shell.ravel(), (-2 * nu * ksq * e).ravel(), nsh)
    assert len(sp["k"]) == nsh and np.allclose(sp["k"], np.arange(nsh) * dk)
    assert np.abs(sp["E"] - E).max() <= 1e-12 * np.abs(E).max()
    assert np.abs(sp["T"] - T).max() <= 1e-10 * np.abs(T).max()
    assert np.abs(sp["D"] - D).max() <= 1e-12 * np.abs(D).max()


def test_fld_roundtrip(tmp_path):
    n = (32, 16)
    u0 = ic.ns2d_ic(n, seed=4)
    g = api.Simulation("ns2d", n, 1e-3, 1e-3)
    g.set_state(u0)
    g.step(3)
    p = tmp_path / "state_phys.fld"
    g.save_fld(p, digest="abc")
    head = p.read_bytes().split(b"\n")[:6]
    assert head[0] == b"spectralkit-fld 1" and head[2] == b"shape=32x16" and head[3] == b"vars=rot"
    assert head[4] == b"digest=abc" and head[5] == b""
    h = api.Simulation("ns2d", n, 1e-3, 1e-3)
    hdr = h.load_fld(p)
    assert hdr["time"] == g.t and h.t == g.t
    assert np.abs(h.get_state() - g.get_state()).max() < 1e-14


@pytest.mark.parametrize("solver,n", [("ns2d", (64, 64)), ("ns3d", (16, 16, 16))])
def test_restart_equals_uninterrupted(solver, n, tmp_path):
    """test_simulation.cpp:361-396: a run continued from its own snapshot
    matches the uninterrupted run (the physical round trip costs ~1e-16)."""
    u0 = ic.initial_state(solver, n, seed=10)
    dt = 0.5 * ic.cfl_dt(solver, n, u0)
    a = api.Simulation(solver, n, 1e-3, dt)
    a.set_state(u0)
    a.step(4)
    a.save_fld(tmp_path / "snap.fld")
    a.step(4)
    b = api.Simulation(solver, n, 1e-3, dt)
    b.load_fld(tmp_path / "snap.fld")
    b.step(4)
    assert per_field(b.get_state(), a.get_state()) < 1e-12
    assert abs(b.t - a.t) < 1e-15
