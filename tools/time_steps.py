"""Quick device timing of RK4 steps at several cubic/square sizes (A/B of
library variants):  SKG_LIB_VARIANT=x python tools/time_steps.py ns2d 512 1024"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1807_01769_b200 import api  # noqa: E402
from paper_1807_01769_b200 import ic  # noqa: E402

solver = sys.argv[1]
for n in map(int, sys.argv[2:]):
    shape = (n,) * (2 if solver == "ns2d" else 3)
    u0 = ic.initial_state(solver, shape, seed=1234)
    sim = api.Simulation(solver, shape, 1e-4, 1e-4, device=0)
    sim.set_state(u0)
    st = torch.cuda.Stream()
    sim.set_stream(st.cuda_stream)
    sim.step(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 100 if n ** len(shape) <= 1 << 22 else 10
    torch.cuda.synchronize()
    e0.record(st)
    sim.step_async(steps)
    e1.record(st)
    torch.cuda.synchronize()
    sim.sync()
    print(f"{solver} n={n} pruned={sim.pruned} ms/step {e0.elapsed_time(e1) / steps:.4f}", flush=True)
    sim.close()
