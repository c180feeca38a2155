"""GPU parity tests, ns2d + transform operators, through the C ABI.

Bars (BASELINE.json north_star): wavenumbers and dealias masks bit-exact;
states within 1e-10 relative L2 per field after the stated steps; transforms
within the reference's own test tolerances (test_fft.cpp).
"""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
PARITY = 1e-10


def rel(a, b):
    return O.rel_l2(a, b)


@pytest.mark.parametrize("n", [(8, 8), (64, 32), (32, 128), (1024, 1024), (4096, 4096)])
def test_grid_bit_exact(ref_lib, n):
    g = api.Simulation("ns2d", n, 0.0, 0.1)
    ks, mask = g.grid()
    r = ref_lib.RefSimulation("ns2d", n, 0.0, 0.1)
    rks, rmask = r.grid()
    for a, b in zip(ks, rks):
        assert a.tobytes() == b.tobytes()
    assert mask.tobytes() == rmask.tobytes()


@pytest.mark.parametrize("shape", [(8,), (8, 6), (6, 4, 8), (64, 64), (16, 16, 16), (16, 12, 8),
                                   (1024, 1024), (4096, 64), (32, 4096), (128, 64, 32)])
def test_fft_operators_match_reference(ref_lib, shape):
    rng = np.random.default_rng(11)
    u = rng.uniform(-1, 1, size=shape)
    uh = api.fft_forward(u)
    ruh = ref_lib.fft_forward(u)
    assert np.abs(uh - ruh).max() < 1e-13  # test_fft.cpp:122
    back = api.fft_inverse(uh, shape)
    assert np.abs(back - u).max() / np.abs(u).max() < 1e-12  # test_fft.cpp:141-155
    assert np.abs(back - ref_lib.fft_inverse(ruh, shape)).max() < 1e-12


def test_fft_known_answers():
    u = np.cos(2 * math.pi * np.arange(8) / 8)
    uh = api.fft_forward(u)
    assert abs(uh[1] - 0.5) < 1e-15
    uh = api.fft_forward(np.full((16, 16), 3.0))
    assert abs(uh[0, 0] - 3.0) < 1e-14 and np.abs(uh.ravel()[1:]).max() < 1e-14
    h = np.zeros(5, complex)
    h[1] = 0.5
    assert np.allclose(api.fft_inverse(h, (8,)), np.cos(2 * math.pi * np.arange(8) / 8),
                       rtol=0, atol=1e-15)
    # the inverse leaves its input intact (test_fft.cpp:157-168)
    rng = np.random.default_rng(5)
    uh = api.fft_forward(rng.uniform(-1, 1, (16, 16)))
    keep = uh.copy()
    api.fft_inverse(uh, (16, 16))
    assert np.array_equal(uh, keep)


def test_context_fft_matches_plan(ref_lib):
    g = api.Simulation("ns2d", (256, 128), 0.0, 0.1)
    rng = np.random.default_rng(2)
    u = rng.standard_normal((256, 128))
    assert np.abs(g.fft_forward(u) - ref_lib.fft_forward(u)).max() < 1e-14
    uh = ref_lib.fft_forward(u)
    assert np.abs(g.fft_inverse(uh) - u).max() < 1e-12


@pytest.mark.parametrize("n", [(16, 16), (32, 32), (64, 32), (32, 64), (256, 256), (1024, 1024)])
def test_tendency_matches_reference(ref_lib, n):
    u0 = ic.ns2d_ic(n, seed=3)
    r = ref_lib.RefSimulation("ns2d", n, 1e-3, 1e-3)
    g = api.Simulation("ns2d", n, 1e-3, 1e-3)
    t_ref = r.tendency(u0)
    t_gpu = g.compute_tendency(u0)
    # one tendency evaluation: FP64 FFT rounding, O(eps log N); the dealiased
    # fast path evaluates the mathematically identical Basdevant form
    assert rel(t_gpu, t_ref) < 1e-11
    # dealiased output: masked modes exactly zero, mean zero
    mask = O.dealias_mask(n).astype(bool)
    assert np.all(t_gpu[0][~mask] == 0)
    assert t_gpu[0, 0, 0] == 0


@pytest.mark.parametrize("n", [(16, 16), (64, 32), (128, 128)])
def test_tendency_of_non_dealiased_input(ref_lib, n):
    # the reference's tendency does not dealias its input (solvers.cpp:133-174):
    # the unpruned path must see every mode
    rng = np.random.default_rng(9)
    w = O.forward(rng.standard_normal(n))[None]
    r = ref_lib.RefSimulation("ns2d", n, 0.0, 0.1)
    g = api.Simulation("ns2d", n, 0.0, 0.1)
    assert rel(g.compute_tendency(w), r.tendency(w)) < 1e-12


@pytest.mark.parametrize("path", sorted(GOLD.glob("ns2d*.npz")), ids=lambda p: p.stem)
def test_golden_fixtures(path):
    f = np.load(path)
    n = tuple(int(x) for x in f["n"])
    g = api.Simulation("ns2d", n, float(f["nu"]), float(f["dt"]), scheme=str(f["scheme"]))
    assert rel(g.compute_tendency(f["u0"]), f["tendency"]) < 1e-11
    g.set_state(f["u0"])
    assert g.pruned
    g.step(int(f["steps"]))
    assert rel(g.get_state(), f["final"]) < PARITY
    assert g.iteration == int(f["steps"])


@pytest.mark.parametrize("n,steps,nu,dt", [((1024, 1024), 10, 1e-4, 1e-3), ((512, 256), 10, 1e-4, 2e-3)])
def test_baseline_config_parity(ref_lib, n, steps, nu, dt):
    """configs[0] of BASELINE.json: ns2d 1024^2, nu 1e-4, dt 1e-3, 10 RK4 steps."""
    u0 = ic.ns2d_ic(n, seed=1234)
    ref_lib.set_workers(8)
    r = ref_lib.RefSimulation("ns2d", n, nu, dt)
    r.set_state(u0)
    r.step(steps)
    g = api.Simulation("ns2d", n, nu, dt)
    g.set_state(u0)
    g.step(steps)
    assert rel(g.get_state(), r.get_state()) < PARITY
    e, z = g.energy_enstrophy()
    assert abs(e - r.energy) < 1e-12 * max(1.0, r.energy)
    assert abs(z - r.enstrophy) < 1e-10 * max(1.0, r.enstrophy)


def test_unpruned_step_matches_reference(ref_lib):
    # a state with energy in masked-out modes takes the full (unpruned) path
    n = (64, 64)
    rng = np.random.default_rng(4)
    w = O.forward(rng.standard_normal(n))[None] * 5.0
    w[0, 0, 0] = 0.3
    r = ref_lib.RefSimulation("ns2d", n, 1e-2, 1e-3)
    r.set_state(w)
    r.step(5)
    g = api.Simulation("ns2d", n, 1e-2, 1e-3)
    g.set_state(w)
    assert not g.pruned
    g.step(5)
    assert rel(g.get_state(), r.get_state()) < PARITY


def test_taylor_green_known_answers():
    # test_solvers.cpp:62-80 (zero nonlinear term) and 164-192 (exact decay)
    n = (64, 64)
    x = np.arange(64) * (2 * math.pi / 64)
    w = 2.0 * np.sin(x)[:, None] * np.sin(x)[None, :]
    wh = O.forward(w)[None]
    nu, dt = 0.01, 0.01
    g = api.Simulation("ns2d", n, nu, dt)
    assert np.abs(g.compute_tendency(wh)).max() < 1e-13
    g.set_state(wh)
    assert abs(g.energy() - 0.25) < 1e-12 and abs(g.enstrophy() - 0.5) < 1e-12
    g.step(20)
    decay = math.exp(-2 * nu * 20 * dt)
    assert np.abs(g.get_state() - wh * decay).max() < 1e-11


def test_zero_state_gives_zero_tendency():
    g = api.Simulation("ns2d", (32, 32), 1e-3, 1e-3)
    z = np.zeros((1, 32, 17), complex)
    assert np.all(g.compute_tendency(z) == 0)


def test_divergence_error():
    # NaN injection -> DivergenceError(iteration, field), state frozen (simulation.cpp:557-563)
    n = (32, 32)
    u0 = ic.ns2d_ic(n, seed=1)
    u0[0, 3, 2] = np.nan
    g = api.Simulation("ns2d", n, 1e-3, 1e-3)
    g.set_state(u0)
    with pytest.raises(api.DivergenceError) as ei:
        g.step(5)
    assert ei.value.iteration == 1
    assert ei.value.field == "rot_fft"
    assert g.iteration == 1


def test_bad_dt():
    g = api.Simulation("ns2d", (32, 32), 1e-3, 0.0)
    with pytest.raises(api.ConfigError):
        g.step(1)


def test_state_shape_error():
    g = api.Simulation("ns2d", (32, 32), 1e-3, 1e-3)
    with pytest.raises(api.ShapeError):
        g.set_state(np.zeros((1, 32, 16), complex))


@pytest.mark.parametrize("n,noise", [((256, 256), False), ((64, 64), True)])
def test_run_series_matches_reference(ref_lib, n, noise):
    """Simulation::run's per-step means (output.cpp:204-214): E, Z, eps after
    every step, fused on the dealiased path, a device reduction otherwise."""
    if noise:
        rng = np.random.default_rng(3)
        u0 = O.forward(rng.standard_normal(n))[None]
    else:
        u0 = ic.ns2d_ic(n, seed=8)
    nu, dt, steps = 1e-3, 1e-3, 6
    r = ref_lib.RefSimulation("ns2d", n, nu, dt)
    r.set_state(u0)
    g = api.Simulation("ns2d", n, nu, dt)
    g.set_state(u0)
    series = g.run(steps)
    ksq = O.k_sq(n)
    w = O.parseval_w(n)
    for i in range(steps):
        r.step(1)
        s = r.get_state()[0]
        eps = float((np.where(ksq > 0, nu * w * np.abs(s) ** 2, 0.0)).sum())
        assert abs(series[i, 0] - r.energy) < 1e-12 * r.energy
        assert abs(series[i, 1] - r.enstrophy) < 1e-11 * r.enstrophy
        assert abs(series[i, 2] - eps) < 1e-11 * eps
    assert O.rel_l2(g.get_state(), r.get_state()) < PARITY


def test_8192_generic_step(ref_lib):
    """8192 x 8192, beyond the fused kernels' range (their general path does
    not fit shared memory there): the generic step and the transform
    operators, 2 RK4 steps vs the reference (multi-threaded CPU oracle)."""
    n = (8192, 8192)
    u0 = ic.ns2d_ic(n, seed=5)
    dt = ic.cfl_dt("ns2d", n, u0)
    g = api.Simulation("ns2d", n, 1e-4, dt)
    g.set_state(u0)
    g.step(2)
    ref_lib.set_workers(16)
    r = ref_lib.RefSimulation("ns2d", n, 1e-4, dt)
    r.set_state(u0)
    r.step(2)
    assert O.rel_l2(g.get_state()[0], r.get_state()[0]) < 1e-10
    u = np.random.default_rng(1).standard_normal((8192,))
    assert np.abs(api.fft_forward(u) - np.fft.rfft(u) / u.size).max() < 1e-14


@pytest.mark.parametrize("scheme,lo,hi,k0", [("RK4", 3.7, 4.3, 20), ("RK2", 1.8, 2.2, 80)])
def test_temporal_order(scheme, lo, hi, k0):
    """Measured global order of the GPU stepper on the nonlinear ns2d problem
    (the property test_time_stepping.cpp:108-139 checks on scalar ODEs),
    against a 16x finer run of the same code."""
    n = (64, 64)
    u0 = ic.ns2d_ic(n, seed=13) * 2.0
    nu, T = 1e-3, 0.2

    def run(nsteps):
        g = api.Simulation("ns2d", n, nu, T / nsteps, scheme=scheme)
        g.set_state(u0)
        g.step(nsteps)
        return g.get_state()

    ref = run(32 * k0)
    e1, e2, e3 = (np.linalg.norm(run(k) - ref) for k in (k0, 2 * k0, 4 * k0))
    o1, o2 = np.log2(e1 / e2), np.log2(e2 / e3)
    assert lo < o1 < hi and lo < o2 < hi, (o1, o2)


def test_exp_factors_follow_dt_changes():
    """time_stepping.cpp:160-166: a pure-decay mode (zero nonlinearity) with a
    dt change decays by exp(-nu k^2 (dt1 + dt2)) to round-off."""
    n = (32, 32)
    x = np.arange(32) * 2 * math.pi / 32
    w = np.cos(3 * x)[:, None] * np.ones((1, 32))       # kx = 3: u . grad w = 0
    s = O.forward(w)[None]
    nu = 0.05
    g = api.Simulation("ns2d", n, nu, 0.01)
    g.set_state(s)
    g.step(1, dt=0.01)
    g.step(1, dt=0.03)
    assert np.abs(g.get_state() - s * math.exp(-nu * 9 * 0.04)).max() < 1e-15
