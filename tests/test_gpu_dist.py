"""Slab decomposition on ONE GPU: all `world` partitions of the ns2d / ns3d state
run in one process with device copies standing in for the NCCL all-to-all
(the same kernels and block layouts as the multi-process NCCL path).  The
result must reproduce the single-partition path and the reference."""
import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,world", [((256, 256), 2), ((256, 256), 4), ((512, 256), 8),
                                     ((1024, 1024), 8), ((128, 512), 2)])
def test_slab_matches_single_partition(n, world):
    u0 = ic.ns2d_ic(n, seed=7)
    dt = ic.cfl_dt("ns2d", n, u0)
    one = api.Simulation("ns2d", n, 1e-4, dt)
    one.set_state(u0)
    one.step(5)
    d = api.Simulation("ns2d", n, 1e-4, dt, world=world)
    d.set_state(u0)
    d.step(5)
    a, b = d.get_state(), one.get_state()
    # same kernels and arithmetic per element: expected bit-identical
    assert O.rel_l2(a, b) < 1e-14
    assert d.iteration == 5
    ea, za = d.energy_enstrophy()
    eb, zb = one.energy_enstrophy()
    assert abs(ea - eb) <= 1e-13 * eb and abs(za - zb) <= 1e-13 * zb


def test_slab_matches_reference(ref_lib):
    n = (256, 256)
    u0 = ic.ns2d_ic(n, seed=9)
    dt = ic.cfl_dt("ns2d", n, u0)
    r = ref_lib.RefSimulation("ns2d", n, 1e-4, dt)
    r.set_state(u0)
    r.step(10)
    d = api.Simulation("ns2d", n, 1e-4, dt, world=4)
    d.set_state(u0)
    d.step(10)
    assert O.rel_l2(d.get_state(), r.get_state()) < 1e-10


def test_slab_needs_dealiased_state():
    n = (64, 64)
    rng = np.random.default_rng(2)
    w = O.forward(rng.standard_normal(n))[None]
    d = api.Simulation("ns2d", n, 1e-3, 1e-3, world=2)
    with pytest.raises(api.UnsupportedError):
        d.set_state(w)


def test_slab_config_errors():
    with pytest.raises(api.ConfigError):
        api.Simulation("ns2d", (64, 64), 1e-3, 1e-3, world=64)   # 64 % (2*64) != 0
    with pytest.raises(api.ConfigError):
        api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3, world=3)  # nx % world
    with pytest.raises(api.ConfigError):
        api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3, world=16)  # 11 kept ky lines


@pytest.mark.parametrize("n,world", [((32, 32, 32), 2), ((64, 64, 64), 4), ((64, 32, 128), 8),
                                     ((128, 128, 128), 8), ((16, 64, 32), 16)])
def test_slab3d_matches_single_partition(n, world):
    u0 = ic.ns3d_ic(n, seed=7)
    dt = ic.cfl_dt("ns3d", n, u0)
    one = api.Simulation("ns3d", n, 1e-3, dt)
    one.set_state(u0)
    one.step(3)
    d = api.Simulation("ns3d", n, 1e-3, dt, world=world)
    d.set_state(u0)
    d.step(3)
    a, b = d.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(a[v], b[v]) < 1e-14
    assert d.iteration == 3


def test_slab3d_matches_reference(ref_lib):
    n = (64, 64, 64)
    u0 = ic.ns3d_ic(n, seed=9)
    dt = ic.cfl_dt("ns3d", n, u0)
    r = ref_lib.RefSimulation("ns3d", n, 1e-3, dt)
    r.set_state(u0)
    r.step(10)
    d = api.Simulation("ns3d", n, 1e-3, dt, world=4)
    d.set_state(u0)
    d.step(10)
    s, rs = d.get_state(), r.get_state()
    assert max(O.rel_l2(s[v], rs[v]) for v in range(3)) < 1e-10


def test_slab3d_run_series_and_divergence():
    n = (32, 32, 32)
    u0 = ic.ns3d_ic(n, seed=4)
    one = api.Simulation("ns3d", n, 1e-2, 1e-3)
    one.set_state(u0)
    d = api.Simulation("ns3d", n, 1e-2, 1e-3, world=2)
    d.set_state(u0)
    a, b = d.run(4), one.run(4)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    bad = u0.copy()
    bad[2, 1, 1, 1] = np.nan
    d.set_state(bad)
    with pytest.raises(api.DivergenceError) as ei:
        d.step(3)
    assert ei.value.iteration == d.iteration


def test_slab_run_series():
    n = (256, 256)
    u0 = ic.ns2d_ic(n, seed=4)
    one = api.Simulation("ns2d", n, 1e-3, 1e-3)
    one.set_state(u0)
    d = api.Simulation("ns2d", n, 1e-3, 1e-3, world=4)
    d.set_state(u0)
    a, b = d.run(5), one.run(5)
    assert np.allclose(a, b, rtol=1e-12, atol=0)


@pytest.mark.parametrize("n", [(32, 32, 32), (64, 32, 16), (16, 64, 128), (128, 128, 128)])
def test_compact_layout_matches_full(n):
    """ns3d compact single-GPU layout (skg_create_dist, world 1)."""
    u0 = ic.ns3d_ic(n, seed=11)
    dt = ic.cfl_dt("ns3d", n, u0)
    one = api.Simulation("ns3d", n, 1e-3, dt)
    one.set_state(u0)
    c = api.Simulation("ns3d", n, 1e-3, dt, compact=True)
    c.set_state(u0)
    a, b = c.run(3), one.run(3)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    s, r = c.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(s[v], r[v]) < 1e-14
    mask = O.dealias_mask(n).astype(bool)
    assert np.all(s[:, ~mask] == 0)
    e1, _ = c.energy_enstrophy()
    e2, _ = one.energy_enstrophy()
    assert abs(e1 - e2) <= 1e-13 * e2


def test_compact_layout_rejects_undealiased_state():
    n = (16, 16, 16)
    rng = np.random.default_rng(2)
    v = np.stack([O.forward(rng.standard_normal(n)) for _ in range(3)])
    c = api.Simulation("ns3d", n, 1e-3, 1e-3, compact=True)
    with pytest.raises(api.UnsupportedError):
        c.set_state(v)


def test_nccl_single_rank_communicator():
    """The NCCL plumbing on one GPU: a 1-rank communicator (ncclCommInitRank,
    the all-reduce of the state gather and of the CFL maxima) on the compact
    ns3d layout; ranks that wait on each other are never co-located."""
    n = (32, 32, 32)
    u0 = ic.ns3d_ic(n, seed=12)
    one = api.Simulation("ns3d", n, 1e-3, 1e-3)
    one.set_state(u0)
    one.step(3)
    d = api.Simulation("ns3d", n, 1e-3, 1e-3, world=1, rank=0, nccl_id=api.nccl_unique_id(),
                       compact=True)
    d.set_state(u0)
    d.step(3)
    a, b = d.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(a[v], b[v]) < 1e-14
    d.set_cfl(0.5, 0.1)
    one.set_cfl(0.5, 0.1)
    d.step(2)
    one.step(2)
    assert d.t == one.t
    s, r = d.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(s[v], r[v]) < 1e-14


@pytest.mark.parametrize("n,world", [((256, 256), 2), ((512, 256), 8), ((1024, 1024), 4)])
def test_slab_peer_exchange_matches(n, world):
    """Peer-memory exchange (producers store into the owners' receive
    buffers; skg_dist_p2p) reproduces the copy-based all-to-all exactly."""
    u0 = ic.ns2d_ic(n, seed=3)
    dt = ic.cfl_dt("ns2d", n, u0)
    a = api.Simulation("ns2d", n, 1e-4, dt, world=world)
    a.set_state(u0)
    a.step(4)
    b = api.Simulation("ns2d", n, 1e-4, dt, world=world)
    b.enable_p2p()
    b.set_state(u0)
    b.step(4)
    assert np.array_equal(a.get_state(), b.get_state())
    ra, rb = a.run(3), b.run(3)
    assert np.allclose(ra, rb, rtol=1e-13, atol=0)


@pytest.mark.parametrize("n,world", [((32, 32, 32), 2), ((64, 64, 64), 4), ((128, 128, 128), 8)])
def test_slab3d_peer_exchange_matches(n, world):
    u0 = ic.ns3d_ic(n, seed=3)
    dt = ic.cfl_dt("ns3d", n, u0)
    a = api.Simulation("ns3d", n, 1e-3, dt, world=world)
    a.set_state(u0)
    a.step(3)
    b = api.Simulation("ns3d", n, 1e-3, dt, world=world)
    b.enable_p2p()
    b.set_state(u0)
    b.step(3)
    assert np.array_equal(a.get_state(), b.get_state())


@pytest.mark.gpu
def test_exchange_mode_switch_between_calls():
    """Toggling the peer exchange between skg_step calls re-captures the
    per-step CUDA graph (its key includes the exchange mode): the trajectory
    equals the copy path's with the same call boundaries (a batch ends with
    an unfused x-forward, so the boundaries themselves change the last bits)."""
    n, world = (256, 256), 4
    u0 = ic.ns2d_ic(n, seed=5)
    dt = ic.cfl_dt("ns2d", n, u0)
    a = api.Simulation("ns2d", n, 1e-4, dt, world=world)
    a.set_state(u0)
    for _ in range(3):
        a.step(5)
    b = api.Simulation("ns2d", n, 1e-4, dt, world=world)
    b.set_state(u0)
    b.step(5)
    b.enable_p2p()
    b.step(5)
    b.disable_p2p()
    b.step(5)
    assert np.array_equal(a.get_state(), b.get_state())


@pytest.mark.parametrize("n,world", [((64, 64, 64), 4), ((128, 64, 32), 8)])
def test_slab3d_overlapped_exchange_matches_serial(n, world):
    """ns3d copy exchange chunked per field on a second stream (the
    NCCL path's overlap, skg_dist_overlap: per-component x-inverse and
    per-field y-forward launches, fork/join events) equals the serial
    exchange bit for bit, with the middle steps replayed from the captured
    CUDA graph of the dist step; and both equal one partition."""
    u0 = ic.ns3d_ic(n, seed=6)
    dt = ic.cfl_dt("ns3d", n, u0)
    a = api.Simulation("ns3d", n, 1e-3, dt, world=world)
    a.set_overlap(False)
    a.set_state(u0)
    a.step(6)
    b = api.Simulation("ns3d", n, 1e-3, dt, world=world)
    b.set_state(u0)
    b.step(6)
    assert np.array_equal(a.get_state(), b.get_state())
    one = api.Simulation("ns3d", n, 1e-3, dt)
    one.set_state(u0)
    one.step(6)
    s, r = b.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(s[v], r[v]) < 1e-14
    # CFL steps through the overlapped path (all-reduced max |u_d| per step)
    b.set_cfl(0.5, 0.1)
    one.set_cfl(0.5, 0.1)
    b.step(5)
    one.step(5)
    assert abs(b.t - one.t) <= 1e-15 * one.t
    s, r = b.get_state(), one.get_state()
    for v in range(3):
        assert O.rel_l2(s[v], r[v]) < 1e-13


def a2a_bytes_per_gpu_step(sim, world, nsteps=2):
    """Measured all-to-all bytes per GPU per RK4 step (exchange class of the
    per-kernel stats: bytes that cross partitions)."""
    sim.reset_stats()
    sim.set_timing(True)
    sim.step(nsteps)
    sim.set_timing(False)
    return sim.kernel_stats()["exchange"][2] / world / nsteps


@pytest.mark.slow
def test_real_split_ns2d_4096_world8():
    """BASELINE configs[1]'s grid at its 8-GPU split (8 slab partitions on one
    GPU): copy and peer-memory exchanges equal one partition; the measured
    all-to-all volume per GPU is the kept-column model
    4 stages x 2 exchanges x 2 fields x nx Kc 16 B (G-1)/G^2 (SURVEY 8(d)'s
    unpruned 4-inverse+1-forward model: 20 F (G-1)/G^2)."""
    n, world = (4096, 4096), 8
    u0 = ic.ns2d_ic(n, seed=1234)
    dt = ic.cfl_dt("ns2d", n, u0)
    one = api.Simulation("ns2d", n, 1e-4, dt)
    one.set_state(u0)
    one.step(5)
    ref = one.get_state()
    one.close()
    for p2p in (False, True):
        d = api.Simulation("ns2d", n, 1e-4, dt, world=world)
        if p2p:
            d.enable_p2p()
        d.set_state(u0)
        d.step(5)
        assert O.rel_l2(d.get_state(), ref) < 1e-14
        if not p2p:
            kc = 1365 + 1
            model = 4 * 2 * 2 * n[0] * kc * 16 * (world - 1) / world ** 2
            got = a2a_bytes_per_gpu_step(d, world)
            assert abs(got - model) <= 1e-9 * model
            F = 16 * n[0] * (n[1] // 2 + 1)
            assert got < 20 * F * (world - 1) / world ** 2
        d.close()


@pytest.mark.slow
def test_real_split_ns3d_512_world8():
    """BASELINE configs[3]'s grid at its 8-GPU split: the overlapped copy
    exchange and the peer-memory exchange equal one partition; measured
    all-to-all volume per GPU = 4 stages x 8 fields x nx K kz 16 B (G-1)/G^2
    (K = 341 kept ky lines, kz = 171 kept kz; SURVEY 8(d) unpruned 32 F (G-1)/G^2)."""
    n, world = (512, 512, 512), 8
    u0 = ic.ns3d_ic(n, seed=1234)
    dt = ic.cfl_dt("ns3d", n, u0)
    one = api.Simulation("ns3d", n, 2e-4, dt)
    one.set_state(u0)
    one.step(4)
    ref = one.get_state()
    one.close()
    for p2p in (False, True):
        d = api.Simulation("ns3d", n, 2e-4, dt, world=world)
        if p2p:
            d.enable_p2p()
        d.set_state(u0)
        d.step(4)
        s = d.get_state()
        for v in range(3):
            assert O.rel_l2(s[v], ref[v]) < 1e-14
        del s
        if not p2p:
            model = 4 * 8 * n[0] * 341 * 171 * 16 * (world - 1) / world ** 2
            got = a2a_bytes_per_gpu_step(d, world, 1)
            assert abs(got - model) <= 1e-9 * model
            F = 16 * n[0] * n[1] * (n[2] // 2 + 1)
            assert got < 32 * F * (world - 1) / world ** 2
        d.close()
