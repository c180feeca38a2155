"""BASELINE.json's full single-GPU grids (configs[1] ns2d 4096^2, configs[3]
ns3d 512^3) on the B200 against the compiled reference (oracle/_ref, all host
threads), plus size-independent properties where the reference's CPU step is
too slow for a test (ns3d 512^3: ~40 s per step).

Bar (north_star): <= 1e-10 relative L2 per field.  These take a few minutes
(the reference's CPU steps dominate).
"""
import os

import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
PARITY = 1e-10


def per_field(a, b):
    return max(O.rel_l2(a[v], b[v]) for v in range(a.shape[0]))


def test_configs1_ns2d_4096_20_steps(ref_lib):
    """configs[1]: ns2d 4096^2, nu 1e-4, dt from CFL 0.5 on the IC, 20 RK4 steps."""
    n = (4096, 4096)
    u0 = ic.ns2d_ic(n, seed=1234)
    dt = ic.cfl_dt("ns2d", n, u0)
    ref_lib.set_workers(os.cpu_count() or 1)
    r = ref_lib.RefSimulation("ns2d", n, 1e-4, dt)
    r.set_state(u0)
    r.step(20)
    g = api.Simulation("ns2d", n, 1e-4, dt)
    g.set_state(u0)
    assert g.pruned
    g.step(20)
    s, ref = g.get_state(), r.get_state()
    r.close()
    assert per_field(s, ref) < PARITY
    # dealias mask: the masked modes stay exactly zero (grid.cpp:112-122)
    mask = O.dealias_mask(n)
    assert not np.any(s[0][~mask.astype(bool)])


def test_configs3_ns3d_512_one_step_and_properties(ref_lib):
    """configs[3]: ns3d 512^3, nu 2e-4, dt from CFL 0.5.  One RK4 step against
    the reference, then 10 GPU steps: divergence-free to round-off, masked modes
    exactly zero, viscous energy decay, and the device energy equal to the
    reference's energy formula on the final state."""
    n = (512, 512, 512)
    u0 = ic.ns3d_ic(n, seed=1234)
    dt = ic.cfl_dt("ns3d", n, u0)
    ref_lib.set_workers(os.cpu_count() or 1)
    r = ref_lib.RefSimulation("ns3d", n, 2e-4, dt)
    r.set_state(u0)
    r.step(1)
    ref1 = r.get_state()
    r.close()
    g = api.Simulation("ns3d", n, 2e-4, dt)
    g.set_state(u0)
    assert g.pruned
    g.step(1)
    s = g.get_state()
    assert per_field(s, ref1) < PARITY
    del ref1
    e1, _ = g.energy_enstrophy()
    g.step(9)
    s = g.get_state()
    e10, _ = g.energy_enstrophy()
    assert np.all(np.isfinite(s.view(np.float64)))
    assert 0.0 < e10 < e1
    w = O.parseval_w(n)
    # energy: Sum w |v|^2 / 2 over the three components (simulation.cpp:163-170)
    e_host = 0.5 * sum(float((w * (s[c].real ** 2 + s[c].imag ** 2)).sum()) for c in range(3))
    assert abs(e_host - e10) < 1e-12 * e10
    kx, ky, kz = O.k_axes(n)
    div = kx[:, None, None] * s[0]
    div += ky[None, :, None] * s[1]
    div += kz[None, None, :] * s[2]
    dn = np.sqrt((w * np.abs(div) ** 2).sum())
    vn = np.sqrt(2.0 * e_host)
    assert dn / vn < 1e-12
    del div
    mask = O.dealias_mask(n).astype(bool)
    for c in range(3):
        assert not np.any(s[c][~mask])


@pytest.mark.parametrize("n", [(4096, 4096), (512, 512, 512)])
def test_transform_round_trip_full_size(n):
    """FftPlan::inverse(FftPlan::forward(u)) == u (fft.cpp:92-106; test_fft.cpp:141-191)
    and Parseval at the full BASELINE grids."""
    rng = np.random.default_rng(7)
    u = rng.standard_normal(n)
    uh = api.fft_forward(u)
    back = api.fft_inverse(uh, n)
    assert O.rel_l2(back, u) < 1e-12
    w = O.parseval_w(n)
    # Parseval with the forward's 1/N: mean(u^2) == Sum w |uh|^2
    lhs = float((u * u).mean())
    rhs = float((w * (uh.real ** 2 + uh.imag ** 2)).sum())
    assert abs(lhs - rhs) < 1e-12 * lhs
