"""Random band forcing (forcing.enable) against the reference with the same
band, rate and seed: the reference's own generator feeds both, so the
forced trajectories must agree to the parity bar."""
import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
PARITY = 1e-10


def per_field(a, b):
    return max(O.rel_l2(a[v], b[v]) for v in range(a.shape[0]))


@pytest.mark.parametrize("solver,n,nu,band,rate", [
    ("ns2d", (64, 64), 1e-3, (2.0, 4.0), 1.0),        # fused dealiased path
    ("ns2d", (32, 32), 1e-2, (3.0, 6.0), 0.5),        # general path (n < 64)
    ("ns2d", (48, 48), 1e-3, (2.0, 5.0), 2.0),        # generic step
    ("ns3d", (16, 16, 16), 1e-2, (2.0, 4.0), 1.0),
    ("ns3d", (12, 12, 12), 1e-2, (1.0, 3.0), 0.3),    # generic step
])
def test_forced_steps_match_reference(ref_lib, solver, n, nu, band, rate):
    u0 = ic.initial_state(solver, n, seed=17)
    dt = ic.cfl_dt(solver, n, u0)
    r = ref_lib.RefSimulation(solver, n, nu, dt, forcing=(band[0], band[1], rate, 99))
    r.set_state(u0)
    g = api.Simulation(solver, n, nu, dt)
    g.set_forcing(band[0], band[1], rate, seed=99)
    g.set_state(u0)
    for _ in range(3):
        r.step(2)
        g.step(2)
        assert abs(g.last_injection - r.last_injection) <= 1e-12 * abs(r.last_injection)
    assert per_field(g.get_state(), r.get_state()) < PARITY
    e, _ = g.energy_enstrophy()
    assert abs(e - r.energy) <= 1e-11 * r.energy


def test_forcing_fallback_zero_state(ref_lib):
    """No state energy in the band: unit-energy fallback (simulation.cpp:500-516)."""
    n = (32, 32)
    z = np.zeros((1, 32, 17), complex)
    r = ref_lib.RefSimulation("ns2d", n, 1e-3, 1e-3, forcing=(2.0, 4.0, 1.0, 5))
    r.set_state(z)
    r.step(3)
    g = api.Simulation("ns2d", n, 1e-3, 1e-3)
    g.set_forcing(2.0, 4.0, 1.0, seed=5)
    g.set_state(z)
    g.step(3)
    assert per_field(g.get_state(), r.get_state()) < PARITY
    assert abs(g.last_injection - r.last_injection) <= 1e-11 * max(1.0, abs(r.last_injection))


def test_forcing_config_errors():
    g = api.Simulation("ns2d", (32, 32), 1e-3, 1e-3)
    with pytest.raises(api.ConfigError):
        g.set_forcing(4.0, 2.0)
    with pytest.raises(api.UnsupportedError):
        g.set_forcing(0.0, 3.0)          # mean shell in the band
    with pytest.raises(api.UnsupportedError):
        g.set_forcing(2.0, 11.0)         # above the dealiasing cut (32/3)
    g.set_forcing(enable=False)
