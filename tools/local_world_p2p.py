"""Single-GPU emulation of the ns2d slab: copy-based all-to-all vs the
peer-memory exchange (producers store into the owners' receive buffers)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1807_01769_b200 import api, ic
n = (4096, 4096)
u0 = ic.ns2d_ic(n, seed=1)
dt = ic.cfl_dt("ns2d", n, u0)
for world in (1, 2, 4, 8):
    for p2p in ((False, True) if world > 1 else (False,)):
        s = api.Simulation("ns2d", n, 1e-4, dt, world=world) if world > 1 else api.Simulation("ns2d", n, 1e-4, dt)
        if p2p:
            s.enable_p2p()
        s.set_state(u0)
        s.step(3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.step(30)
        ms = (time.perf_counter() - t0) / 30 * 1e3
        print(f"world {world} p2p {p2p}: {ms:.3f} ms/step (all partitions on one GPU)")
        s.close()
