"""The generic step (csrc/generic.cu) for extents outside the fused kernels'
range -- any even n >= 4 the reference accepts (grid.cpp:34-44), e.g. the
3 x 2^k grids common in spectral codes -- against the compiled reference."""
import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
PARITY = 1e-10


def per_field(a, b):
    return max(O.rel_l2(a[v], b[v]) for v in range(a.shape[0]))


def _noise(n, nv, seed):
    rng = np.random.default_rng(seed)
    return np.stack([O.forward(rng.standard_normal(n)) for _ in range(nv)])


@pytest.mark.parametrize("solver,n,nu,scheme,steps", [
    ("ns2d", (12, 20), 1e-2, "RK4", 10),
    ("ns2d", (96, 96), 1e-4, "RK4", 10),
    ("ns2d", (48, 80), 0.0, "RK4", 6),
    ("ns2d", (24, 36), 1e-3, "RK2", 8),
    ("ns3d", (12, 12, 12), 1e-2, "RK4", 5),
    ("ns3d", (12, 16, 20), 1e-3, "RK4", 4),
    ("ns3d", (4, 8, 8), 1e-2, "RK2", 4),
    ("ns3d", (24, 24, 24), 0.0, "RK4", 3),
])
def test_generic_steps_match_reference(ref_lib, solver, n, nu, scheme, steps):
    u0 = ic.initial_state(solver, n, seed=31)
    dt = ic.cfl_dt(solver, n, u0)
    r = ref_lib.RefSimulation(solver, n, nu, dt, scheme=scheme)
    r.set_state(u0)
    r.step(steps)
    g = api.Simulation(solver, n, nu, dt, scheme=scheme)
    g.set_state(u0)
    g.step(steps)
    assert per_field(g.get_state(), r.get_state()) < PARITY
    e, z = g.energy_enstrophy()
    assert abs(e - r.energy) <= 1e-12 * abs(r.energy)


@pytest.mark.parametrize("solver,n", [("ns2d", (12, 20)), ("ns2d", (36, 36)), ("ns3d", (12, 12, 20))])
def test_generic_tendency_of_noise(ref_lib, solver, n):
    nv = 1 if solver == "ns2d" else 3
    v = _noise(n, nv, 4)
    r = ref_lib.RefSimulation(solver, n, 1e-3, 1e-3)
    g = api.Simulation(solver, n, 1e-3, 1e-3)
    assert per_field(g.compute_tendency(v), r.tendency(v)) < 1e-11


@pytest.mark.parametrize("solver,n", [("ns2d", (24, 24)), ("ns3d", (12, 12, 12))])
def test_generic_cfl_and_series(ref_lib, solver, n):
    u0 = ic.initial_state(solver, n, seed=6)
    r = ref_lib.RefSimulation(solver, n, 1e-3, 0.0)   # fixed_dt = 0: CFL
    r.set_state(u0)
    g = api.Simulation(solver, n, 1e-3, 0.0)
    g.set_cfl(0.5, 0.1)
    g.set_state(u0)
    series = g.run(4)
    r.step(4)
    assert abs(g.t - r.t) <= 1e-12 * r.t
    assert per_field(g.get_state(), r.get_state()) < PARITY
    assert abs(series[-1, 0] - r.energy) <= 1e-12 * r.energy


def test_generic_divergence_error():
    n = (12, 12)
    u0 = ic.ns2d_ic(n, seed=2)
    u0[0, 1, 2] = np.nan
    g = api.Simulation("ns2d", n, 1e-3, 1e-3)
    g.set_state(u0)
    with pytest.raises(api.DivergenceError) as ei:
        g.step(3)
    assert ei.value.iteration == 1 and ei.value.field == "rot_fft"


def test_generic_rejects_slab():
    with pytest.raises(api.UnsupportedError):
        api.Simulation("ns2d", (96, 96), 1e-3, 1e-3, world=2)
    with pytest.raises(api.UnsupportedError):
        api.Simulation("ns3d", (12, 12, 12), 1e-3, 1e-3, compact=True)


@pytest.mark.parametrize("shape", [(6,), (96,), (1000,), (3000,), (5000,), (96, 160), (12, 20, 36)])
def test_non_pow2_transforms(shape):
    """Bluestein (n <= 4096) and direct-DFT (larger) line transforms against
    numpy: FftPlan::forward = rfftn / N, inverse = irfftn * N."""
    rng = np.random.default_rng(11)
    u = rng.standard_normal(shape)
    uh = api.fft_forward(u)
    ref = np.fft.rfftn(u) / u.size
    assert np.abs(uh - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    back = api.fft_inverse(uh, shape)
    assert np.abs(back - u).max() < 1e-12


def test_generic_384_is_fast(ref_lib):
    """A 3 x 2^7 grid through the generic path: parity and a sane step time."""
    import time
    n = (384, 384)
    u0 = ic.ns2d_ic(n, seed=3)
    dt = ic.cfl_dt("ns2d", n, u0)
    g = api.Simulation("ns2d", n, 1e-4, dt)
    g.set_state(u0)
    g.step(2)
    t0 = time.perf_counter()
    g.step(10)
    ms = (time.perf_counter() - t0) / 10 * 1e3
    r = ref_lib.RefSimulation("ns2d", n, 1e-4, dt)
    r.set_state(u0)
    r.step(12)
    assert per_field(g.get_state(), r.get_state()) < PARITY
    assert ms < 50.0, ms
