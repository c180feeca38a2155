"""Evidence run (not a unit test: the reference needs ~40 s per 512^3 step):
BASELINE.json configs[1] (ns2d 4096^2, 20 RK4 steps) and configs[3] (ns3d
512^3, 10 RK4 steps) on the B200 against the compiled reference on all host
threads, same seeded IC; prints the per-field relative L2 errors (bar 1e-10).

    python tools/parity_fullsize.py [ns2d] [ns3d] > profiles/parity_fullsize.txt
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import ref  # noqa: E402
from oracle import spectral_np as O  # noqa: E402
from paper_1807_01769_b200 import api, ic  # noqa: E402

CASES = {"ns2d": ((4096, 4096), 1e-4, 20), "ns3d": ((512, 512, 512), 2e-4, 10)}
threads = os.cpu_count() or 1
ref.set_workers(threads)
for solver in (sys.argv[1:] or ["ns2d", "ns3d"]):
    n, nu, steps = CASES[solver]
    u0 = ic.initial_state(solver, n, seed=1234)
    dt = ic.cfl_dt(solver, n, u0)
    t0 = time.perf_counter()
    r = ref.RefSimulation(solver, n, nu, dt)
    r.set_state(u0)
    r.step(steps)
    sr = r.get_state()
    e_ref = r.energy
    r.close()
    t_ref = time.perf_counter() - t0
    g = api.Simulation(solver, n, nu, dt)
    g.set_state(u0)
    g.step(steps)
    sg = g.get_state()
    e_gpu, _ = g.energy_enstrophy()
    g.close()
    errs = [O.rel_l2(sg[v], sr[v]) for v in range(sg.shape[0])]
    names = ["rot"] if solver == "ns2d" else ["vx", "vy", "vz"]
    print(f"{solver} {'x'.join(map(str, n))} nu={nu} dt={dt:.6g} (CFL 0.5) {steps} RK4 steps, seed 1234; "
          f"reference {threads} threads {t_ref:.0f} s")
    for nm, e in zip(names, errs):
        print(f"  rel L2 {nm}: {e:.3e}  {'PASS' if e <= 1e-10 else 'FAIL'} (bar 1e-10)")
    print(f"  energy: gpu {e_gpu:.15e} ref {e_ref:.15e} rel diff {abs(e_gpu - e_ref) / e_ref:.2e}")
    sys.stdout.flush()
