"""Slab decomposition on ONE GPU: all `world` partitions of the ns2d state
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
    with pytest.raises(api.UnsupportedError):
        api.Simulation("ns3d", (16, 16, 16), 1e-3, 1e-3, world=2)


def test_slab_run_series():
    n = (256, 256)
    u0 = ic.ns2d_ic(n, seed=4)
    one = api.Simulation("ns2d", n, 1e-3, 1e-3)
    one.set_state(u0)
    d = api.Simulation("ns2d", n, 1e-3, 1e-3, world=4)
    d.set_state(u0)
    a, b = d.run(5), one.run(5)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
