"""The chained y-inverse -> z -> y-forward pass of ns3d (one persistent launch
with per-x-plane dataflow counters, ns3d.cu k_yzy_chain) against the same
tiles run as three separate launches (SKG_CHAIN=0, in a subprocess: the
switch is read once per process): bit-identical states, including the
adaptive-dt (CFL max reduced inside the z tiles) and RK2 variants, and the
self-resetting counters across many launches (graph replays)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_1807_01769_b200 import api, ic
def run(n, steps, cfl, scheme):
    u0 = ic.ns3d_ic(n, seed=21)
    dt = ic.cfl_dt("ns3d", n, u0)
    s = api.Simulation("ns3d", n, 2e-4, dt, scheme=scheme)
    s.set_state(u0)
    if cfl:
        s.set_cfl(0.5, 0.1)
    s.step(steps)
    return s.get_state(), s.t
'''


def run_here(n, steps, cfl, scheme):
    ns = {}
    exec(SCRIPT.format(root=str(ROOT)), ns)
    return ns["run"](n, steps, cfl, scheme)


@pytest.mark.parametrize("n,steps,cfl,scheme", [((256, 256, 256), 7, False, "RK4"),
                                                ((256, 256, 256), 4, True, "RK4"),
                                                ((512, 512, 512), 2, False, "RK2"),
                                                ((512, 256, 256), 3, False, "RK4")])
def test_chain_equals_separate_launches(tmp_path, n, steps, cfl, scheme):
    out = tmp_path / "sep.npz"
    code = SCRIPT.format(root=str(ROOT)) + (
        f"s, t = run({n!r}, {steps}, {cfl}, {scheme!r})\n"
        f"np.savez({str(out)!r}, s=s, t=t)\n")
    env = dict(os.environ, SKG_CHAIN="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    ref = np.load(out)
    s, t = run_here(n, steps, cfl, scheme)
    assert t == float(ref["t"])
    assert np.array_equal(s, ref["s"])
