import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_1807_01769_b200 import api, ic
from oracle import ref, spectral_np as O
n = (8192, 8192)
u0 = ic.ns2d_ic(n, seed=5)
dt = ic.cfl_dt("ns2d", n, u0)
g = api.Simulation("ns2d", n, 1e-4, dt)
g.set_state(u0)
g.step(2)
import torch
torch.cuda.synchronize()
t0 = time.perf_counter(); g.step(20); print("8192^2 ms/step", (time.perf_counter() - t0) / 20 * 1e3)
ref.set_workers(16)
r = ref.RefSimulation("ns2d", n, 1e-4, dt)
r.set_state(u0)
r.step(22)
print("rel l2", O.rel_l2(g.get_state()[0], r.get_state()[0]))
