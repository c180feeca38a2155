"""GPU parity tests, ns3d (rotational form), through the C ABI.

Known answers restated from the reference's own tests
(proj/tests/unit/test_solvers.cpp:194-291) plus oracle parity on the
BASELINE configs (1e-10 relative L2 per field after the stated steps)."""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
PARITY = 1e-10


def per_field(a, b):
    return max(O.rel_l2(a[v], b[v]) for v in range(a.shape[0]))


@pytest.mark.parametrize("n", [(8, 8, 8), (16, 8, 32), (128, 128, 128), (512, 512, 512)])
def test_grid_bit_exact(ref_lib, n):
    g = api.Simulation("ns3d", n, 0.0, 0.1)
    ks, mask = g.grid()
    r = ref_lib.RefSimulation("ns3d", n, 0.0, 0.1)
    rks, rmask = r.grid()
    for a, b in zip(ks, rks):
        assert a.tobytes() == b.tobytes()
    assert mask.tobytes() == rmask.tobytes()
    g.close()


@pytest.mark.parametrize("n", [(16, 16, 16), (32, 32, 32), (16, 8, 32), (32, 64, 16), (64, 64, 64)])
def test_tendency_matches_reference(ref_lib, n):
    u0 = ic.ns3d_ic(n, seed=3)
    r = ref_lib.RefSimulation("ns3d", n, 1e-3, 1e-3)
    g = api.Simulation("ns3d", n, 1e-3, 1e-3)
    t_ref = r.tendency(u0)
    t_gpu = g.compute_tendency(u0)
    assert per_field(t_gpu, t_ref) < 1e-11
    mask = O.dealias_mask(n).astype(bool)
    for v in range(3):
        assert np.all(t_gpu[v][~mask] == 0)
    assert np.all(t_gpu[:, 0, 0, 0] == 0)


@pytest.mark.parametrize("n", [(16, 16, 16), (8, 16, 32)])
def test_tendency_of_non_dealiased_input(ref_lib, n):
    rng = np.random.default_rng(9)
    v = np.stack([O.forward(rng.standard_normal(n)) for _ in range(3)])
    r = ref_lib.RefSimulation("ns3d", n, 0.0, 0.1)
    g = api.Simulation("ns3d", n, 0.0, 0.1)
    assert per_field(g.compute_tendency(v), r.tendency(v)) < 1e-11


@pytest.mark.parametrize("path", sorted(GOLD.glob("ns3d*.npz")), ids=lambda p: p.stem)
def test_golden_fixtures(path):
    f = np.load(path)
    n = tuple(int(x) for x in f["n"])
    g = api.Simulation("ns3d", n, float(f["nu"]), float(f["dt"]), scheme=str(f["scheme"]))
    assert per_field(g.compute_tendency(f["u0"]), f["tendency"]) < 1e-11
    g.set_state(f["u0"])
    assert g.pruned
    g.step(int(f["steps"]))
    assert per_field(g.get_state(), f["final"]) < PARITY


def test_baseline_config_128(ref_lib):
    """configs[2] of BASELINE.json: ns3d 128^3, nu 1e-3, dt from CFL 0.5, 10 RK4 steps."""
    n = (128, 128, 128)
    u0 = ic.ns3d_ic(n, seed=1234)
    dt = ic.cfl_dt("ns3d", n, u0)
    ref_lib.set_workers(8)
    r = ref_lib.RefSimulation("ns3d", n, 1e-3, dt)
    r.set_state(u0)
    r.step(10)
    g = api.Simulation("ns3d", n, 1e-3, dt)
    g.set_state(u0)
    g.step(10)
    s = g.get_state()
    assert per_field(s, r.get_state()) < PARITY
    e, _ = g.energy_enstrophy()
    assert abs(e - r.energy) < 1e-12 * r.energy


def test_unpruned_step_matches_reference(ref_lib):
    n = (16, 16, 16)
    rng = np.random.default_rng(4)
    v = np.stack([O.forward(rng.standard_normal(n)) for _ in range(3)])
    r = ref_lib.RefSimulation("ns3d", n, 1e-2, 1e-3)
    r.set_state(v)
    r.step(3)
    g = api.Simulation("ns3d", n, 1e-2, 1e-3)
    g.set_state(v)
    assert not g.pruned
    g.step(3)
    assert per_field(g.get_state(), r.get_state()) < PARITY


def _sample3d(n, f):
    x = np.arange(n[0]) * (2 * math.pi / n[0])
    y = np.arange(n[1]) * (2 * math.pi / n[1])
    z = np.arange(n[2]) * (2 * math.pi / n[2])
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    return f(X, Y, Z)


def test_beltrami_zero_tendency_and_decay():
    # test_solvers.cpp:194-224 (zero nonlinear term); exact viscous decay
    n = (32, 32, 32)
    vx = _sample3d(n, lambda x, y, z: np.sin(z) + np.cos(y))
    vy = _sample3d(n, lambda x, y, z: np.sin(x) + np.cos(z))
    vz = _sample3d(n, lambda x, y, z: np.sin(y) + np.cos(x))
    v = np.stack([O.forward(a) for a in (vx, vy, vz)])
    nu, dt = 0.01, 0.01
    g = api.Simulation("ns3d", n, nu, dt)
    assert np.abs(g.compute_tendency(v)).max() < 1e-13
    g.set_state(v)
    g.step(10)
    assert np.abs(g.get_state() - v * math.exp(-nu * 10 * dt)).max() < 1e-11


def test_zero_state_zero_tendency():
    g = api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3)
    z = np.zeros((3, 16, 16, 9), complex)
    assert np.all(g.compute_tendency(z) == 0)


def test_energy_neutral_and_divergence_free():
    # test_solvers.cpp:239-291
    n = (32, 32, 32)
    v = ic.ns3d_ic(n, seed=5)
    g = api.Simulation("ns3d", n, 1e-3, 5e-3)
    t = g.compute_tendency(v)
    w = O.parseval_w(n)
    terms = sum(w * (v[c].real * t[c].real + v[c].imag * t[c].imag) for c in range(3))
    assert abs(terms.sum()) < 1e-10 * np.abs(terms).sum()
    kx, ky, kz = O.k_axes(n)
    g.set_state(v)
    for _ in range(10):
        g.step(1)
        s = g.get_state()
        div = 1j * (kx[:, None, None] * s[0] + ky[None, :, None] * s[1] + kz[None, None, :] * s[2])
        dn = np.sqrt((w * np.abs(div) ** 2).sum())
        vn = np.sqrt(sum((w * np.abs(s[c]) ** 2).sum() for c in range(3)))
        assert dn / vn < 1e-12


def test_divergence_error_field_name():
    n = (16, 16, 16)
    u0 = ic.ns3d_ic(n, seed=1)
    u0[1, 2, 3, 1] = np.inf
    g = api.Simulation("ns3d", n, 1e-3, 1e-3)
    g.set_state(u0)
    with pytest.raises(api.DivergenceError) as ei:
        g.step(4)
    assert ei.value.iteration == 1
    assert ei.value.field in ("vx_fft", "vy_fft", "vz_fft")


@pytest.mark.parametrize("noise", [False, True])
def test_run_series_matches_reference(ref_lib, noise):
    n = (32, 32, 32)
    if noise:
        rng = np.random.default_rng(3)
        u0 = np.stack([O.forward(rng.standard_normal(n)) for _ in range(3)])
    else:
        u0 = ic.ns3d_ic(n, seed=8)
    nu, dt, steps = 1e-2, 2e-3, 4
    r = ref_lib.RefSimulation("ns3d", n, nu, dt)
    r.set_state(u0)
    g = api.Simulation("ns3d", n, nu, dt)
    g.set_state(u0)
    series = g.run(steps)
    ksq = O.k_sq(n)
    w = O.parseval_w(n)
    for i in range(steps):
        r.step(1)
        s = r.get_state()
        eps = float(sum((2 * nu * ksq * 0.5 * w * np.abs(s[c]) ** 2).sum() for c in range(3)))
        assert abs(series[i, 0] - r.energy) < 1e-12 * r.energy
        assert series[i, 1] == 0.0
        assert abs(series[i, 2] - eps) < 1e-11 * eps


def test_xforward_scratch_slots_match_in_place_write_back():
    """k4_3d parks the transformed components 0 and 1 in per-SM scratch slots
    (claimed through a bit mask); SKG_XSCR=0 selects the in-place
    write-back the kernel falls back to when no slot is free.  Same
    arithmetic: the states after 3 RK4 steps are bit-identical (dealiased and
    non-dealiased, 16-element and 8-element lines, a non-cubic grid)."""
    import os
    import subprocess
    import sys

    root = Path(__file__).resolve().parents[1]
    code = (
        "import sys, hashlib; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from paper_1807_01769_b200 import api, ic\n"
        "for n, dealiased in (((64, 64, 64), True), ((32, 64, 16), True), ((512, 16, 16), True), ((32, 32, 32), False)):\n"
        "    u0 = ic.initial_state('ns3d', n, seed=5)\n"
        "    if not dealiased:\n"
        "        rng = np.random.default_rng(2)\n"
        "        u0 = u0 + 1e-3 * (rng.standard_normal(u0.shape) + 1j * rng.standard_normal(u0.shape))\n"
        "        u0[..., 0].imag = 0; u0[..., -1].imag = 0\n"
        "    s = api.Simulation('ns3d', n, 1e-3, 1e-3)\n"
        "    s.set_state(u0); s.step(3)\n"
        "    print('H', n, hashlib.sha256(s.get_state().tobytes()).hexdigest())\n"
        "    s.close()\n" % str(root))
    outs = []
    for flag in ("1", "0"):  # slots forced on (default: from nx = 256) / off
        env = dict(os.environ)
        env.pop("SKG_NO_XSCR", None)
        env["SKG_XSCR"] = flag
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        outs.append([l for l in r.stdout.splitlines() if l.startswith("H ")])
    assert len(outs[0]) == 4 and outs[0] == outs[1]
