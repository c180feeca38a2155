"""Quick device timing of ns2d steps at several sizes (A/B of library variants):
    SKG_LIB_VARIANT=x python tools/time_ns2d.py 512 1024 2048"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1807_01769_b200 import api  # noqa: E402
from paper_1807_01769_b200 import ic  # noqa: E402

for n in map(int, sys.argv[1:]):
    u0 = ic.ns2d_ic((n, n), seed=1234)
    sim = api.Simulation("ns2d", (n, n), 1e-4, 1e-4, device=0)
    sim.set_state(u0)
    st = torch.cuda.Stream()
    sim.set_stream(st.cuda_stream)
    sim.step(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 200
    torch.cuda.synchronize()
    e0.record(st)
    sim.step_async(steps)
    e1.record(st)
    torch.cuda.synchronize()
    sim.sync()
    print(f"n={n} pruned={sim.pruned} ms/step {e0.elapsed_time(e1) / steps:.4f}", flush=True)
    sim.close()
