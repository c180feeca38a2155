"""3D pencil decomposition (BASELINE configs[4]) on ONE GPU: all
py x pz parts of the ns3d state run in one process, with device copies standing
in for the two all-to-alls per 3D FFT (the same kernels, layouts and blocks as
the multi-process path).  The result must reproduce the single-partition path
bit for bit and the reference within the 1e-10 bar."""
import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu


def run_pair(n, grid, steps=3, nu=1e-3, seed=7, p2p=False, packed=False, unfused=False):
    u0 = ic.ns3d_ic(n, seed=seed)
    dt = ic.cfl_dt("ns3d", n, u0)
    one = api.Simulation("ns3d", n, nu, dt)
    one.set_state(u0)
    one.step(steps)
    d = api.Simulation("ns3d", n, nu, dt, pencil=grid)
    if p2p:
        d.enable_p2p()
    if packed:
        d.set_overlap(2)
    if unfused:
        d.set_overlap(3)
    d.set_state(u0)
    d.step(steps)
    return d, one


@pytest.mark.parametrize("n,grid", [((32, 32, 32), (2, 2)), ((64, 64, 64), (2, 4)),
                                    ((64, 32, 128), (4, 2)), ((128, 128, 128), (2, 4)),
                                    ((64, 64, 64), (1, 4)), ((64, 64, 64), (4, 1)),
                                    ((32, 64, 16), (2, 2)), ((128, 128, 128), (4, 4))])
def test_pencil_matches_single_partition(n, grid):
    d, one = run_pair(n, grid)
    a, b = d.get_state(), one.get_state()
    for v in range(3):  # same kernels and arithmetic per element
        assert O.rel_l2(a[v], b[v]) < 1e-14
    assert d.iteration == 3
    mask = O.dealias_mask(n).astype(bool)
    assert np.all(a[:, ~mask] == 0)
    ea, _ = d.energy_enstrophy()
    eb, _ = one.energy_enstrophy()
    assert abs(ea - eb) <= 1e-13 * eb


@pytest.mark.parametrize("n,grid", [((64, 64, 64), (2, 2)), ((128, 64, 64), (2, 4))])
def test_pencil_matches_reference(ref_lib, n, grid):
    u0 = ic.ns3d_ic(n, seed=9)
    dt = ic.cfl_dt("ns3d", n, u0)
    r = ref_lib.RefSimulation("ns3d", n, 1e-3, dt)
    r.set_state(u0)
    r.step(10)
    d = api.Simulation("ns3d", n, 1e-3, dt, pencil=grid)
    d.set_state(u0)
    d.step(10)
    s, rs = d.get_state(), r.get_state()
    assert max(O.rel_l2(s[v], rs[v]) for v in range(3)) < 1e-10


@pytest.mark.parametrize("n,grid", [((32, 32, 32), (2, 2)), ((64, 64, 64), (2, 4)), ((128, 128, 128), (4, 2))])
def test_pencil_peer_and_packed_routes_match(n, grid):
    """The exchange routes agree bit for bit: the kz -> y transpose from the
    y-inverse kernel's own stores into the members' buffers (the default with
    all parts in one process) or as a separate strided-copy kernel, the
    peer-memory route of the ky / x all-to-all (producers store into the
    owners' blocks), and the NCCL route's pack -> block transfer -> unpack with
    copies as send / recv."""
    a, one = run_pair(n, grid, steps=4)
    b, _ = run_pair(n, grid, steps=4, p2p=True)
    c, _ = run_pair(n, grid, steps=4, packed=True)
    e, _ = run_pair(n, grid, steps=4, unfused=True)
    sa = a.get_state()
    assert np.array_equal(sa, b.get_state())
    assert np.array_equal(sa, c.get_state())
    assert np.array_equal(sa, e.get_state())
    # switching the route between calls re-captures the step graph
    e.set_overlap(1)
    e.step(4)
    a.step(4)
    assert np.array_equal(a.get_state(), e.get_state())
    r = one.get_state()
    for v in range(3):
        assert O.rel_l2(sa[v], r[v]) < 1e-14


def test_pencil_run_series_cfl_and_divergence():
    n, grid = (32, 32, 32), (2, 2)
    u0 = ic.ns3d_ic(n, seed=4)
    one = api.Simulation("ns3d", n, 1e-2, 1e-3)
    one.set_state(u0)
    d = api.Simulation("ns3d", n, 1e-2, 1e-3, pencil=grid)
    d.set_state(u0)
    a, b = d.run(6), one.run(6)  # fused per-step E / eps over the parts (graph replay in the middle)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    d.set_cfl(0.5, 0.1)
    one.set_cfl(0.5, 0.1)
    d.step(5)
    one.step(5)
    assert abs(d.t - one.t) <= 1e-15 * one.t
    s, r = d.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(s[v], r[v]) < 1e-13
    bad = u0.copy()
    bad[2, 1, 1, 1] = np.nan
    d.set_state(bad)
    with pytest.raises(api.DivergenceError) as ei:
        d.step(3)
    assert ei.value.iteration == d.iteration


def test_pencil_rk2():
    n, grid = (32, 32, 32), (2, 2)
    u0 = ic.ns3d_ic(n, seed=5)
    one = api.Simulation("ns3d", n, 1e-3, 1e-3, scheme="RK2")
    one.set_state(u0)
    one.step(4)
    d = api.Simulation("ns3d", n, 1e-3, 1e-3, scheme="RK2", pencil=grid)
    d.set_state(u0)
    d.step(4)
    assert np.array_equal(d.get_state(), one.get_state())


def test_pencil_config_errors():
    with pytest.raises(api.ConfigError):
        api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3, pencil=(2, 3))    # ny % (2 pz)
    with pytest.raises(api.ConfigError):
        api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3, pencil=(3, 2))    # nx % py
    with pytest.raises(api.ConfigError):
        api.Simulation("ns3d", (64, 64, 64), 1e-3, 1e-3, pencil=(8, 4))    # > 16 ranks
    with pytest.raises(api.ConfigError):
        api.Simulation("ns3d", (64, 64, 16), 1e-3, 1e-3, pencil=(1, 8))    # 6 kept kz < 8 ranks
    with pytest.raises(api.UnsupportedError):
        api.Simulation("ns2d", (64, 64), 1e-3, 1e-3, pencil=(2, 2))
    d = api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3, pencil=(2, 2))
    rng = np.random.default_rng(2)
    v = np.stack([O.forward(rng.standard_normal((16, 16, 16))) for _ in range(3)])
    with pytest.raises(api.UnsupportedError):
        d.set_state(v)  # needs a dealiased state


def a2a_bytes_per_gpu_step(sim, world, nsteps=2):
    sim.reset_stats()
    sim.set_timing(True)
    sim.step(nsteps)
    sim.set_timing(False)
    return sim.kernel_stats()["exchange"][2] / world / nsteps


@pytest.mark.parametrize("n,grid", [((128, 128, 128), (2, 4)), ((128, 128, 128), (2, 2))])
def test_pencil_exchange_volume_matches_model(n, grid):
    """Measured bytes crossing parts per GPU per RK4 step = the kept-mode
    pencil model: per stage, 8 fields through the ky / x all-to-all
    (nx K kz/pz 16 B (py-1)/py^2 each) and 9 fields through the kz / y
    transposes (6 in: nxl ny kz, 3 out; (pz-1)/pz^2 of the group's volume)."""
    py, pz = grid
    u0 = ic.ns3d_ic(n, seed=1)
    dt = ic.cfl_dt("ns3d", n, u0)
    d = api.Simulation("ns3d", n, 1e-3, dt, pencil=grid)
    d.set_state(u0)
    got = a2a_bytes_per_gpu_step(d, py * pz)
    nx, ny, nz = n
    K, kz = 2 * (ny // 3) + 1, nz // 3 + 1
    assert (K, kz) == (85, 43)
    # totals over all parts, then per GPU
    t1 = 8 * nx * K * kz * 16 * (py - 1) / py
    t2 = 9 * nx * ny * kz * 16 * (pz - 1) / pz
    model = 4 * (t1 + t2) / (py * pz)
    assert abs(got - model) <= 1e-9 * model


@pytest.mark.slow
def test_real_split_ns3d_512_pencil_2x4():
    """BASELINE configs[3]'s grid on the 2 x 4 process grid of configs[4]
    (8 parts on one GPU): equals one partition; measured exchange volume per
    GPU = the kept-mode pencil model."""
    n, grid = (512, 512, 512), (2, 4)
    py, pz = grid
    u0 = ic.ns3d_ic(n, seed=1234)
    dt = ic.cfl_dt("ns3d", n, u0)
    one = api.Simulation("ns3d", n, 2e-4, dt)
    one.set_state(u0)
    one.step(3)
    ref = one.get_state()
    one.close()
    d = api.Simulation("ns3d", n, 2e-4, dt, pencil=grid)
    d.set_state(u0)
    d.step(3)
    s = d.get_state()
    for v in range(3):
        assert O.rel_l2(s[v], ref[v]) < 1e-14
    del s
    K, kz = 341, 171
    t1 = 8 * n[0] * K * kz * 16 * (py - 1) / py
    t2 = 9 * n[0] * n[1] * kz * 16 * (pz - 1) / pz
    model = 4 * (t1 + t2) / (py * pz)
    got = a2a_bytes_per_gpu_step(d, py * pz, 1)
    assert abs(got - model) <= 1e-9 * model
    d.close()
