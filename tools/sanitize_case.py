"""Small step runs for compute-sanitizer (tools/sanitize.sh): every kernel
class of the step once or twice on tiny grids, incl. slab emulation with the
copy, overlapped-copy and peer-memory exchanges.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py <case>
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle import spectral_np as O  # noqa: E402
from paper_1807_01769_b200 import api, ic  # noqa: E402

CASES = {
    # name: solver, n, world, p2p
    "ns2d_32": ("ns2d", (32, 32), 1, False),      # general kernels
    "ns2d_64": ("ns2d", (64, 64), 1, False),      # dealiased fast path
    "ns2d_64_w2_p2p": ("ns2d", (128, 64), 2, True),
    "ns2d_64_w4": ("ns2d", (256, 64), 4, False),
    "ns3d_16": ("ns3d", (16, 16, 16), 1, False),
    "ns3d_32_w2_p2p": ("ns3d", (32, 32, 32), 2, True),
    "ns3d_32_w4": ("ns3d", (32, 32, 32), 4, False),   # overlapped copy exchange
    # pencil grids (world = (py, pz)): fused kz -> y stores, packed (NCCL-route) blocks,
    # peer-memory ky / x exchange; uneven kz ranges (11 kept kz over 4 and 3... ranks)
    "ns3d_32_p2x2": ("ns3d", (32, 32, 32), (2, 2), False),
    "ns3d_32_p2x4_p2p": ("ns3d", (32, 32, 32), (2, 4), True),
    "ns3d_p1x4_packed": ("ns3d", (16, 64, 32), (1, 4), "packed"),
    "ns3d_p4x2_unfused": ("ns3d", (64, 32, 32), (4, 2), "unfused"),
}


def main(name):
    solver, n, world, p2p = CASES[name]
    u0 = ic.initial_state(solver, n, seed=3)
    dt = ic.cfl_dt(solver, n, u0)
    pencil = isinstance(world, tuple)
    kw = {"pencil": world} if pencil else {"world": world} if world > 1 else {}
    s = api.Simulation(solver, n, 1e-3, dt, **kw)
    if p2p is True:
        s.enable_p2p()
    elif p2p == "packed":
        s.set_overlap(2)
    elif p2p == "unfused":
        s.set_overlap(3)
    if pencil:
        world = world[0] * world[1]
    s.set_state(u0)
    s.step(2)
    if world == 1:
        s.set_cfl(0.5, 0.1)
        s.step(2)
        # non-dealiased input through the general kernels
        rng = np.random.default_rng(1)
        raw = np.stack([O.forward(rng.standard_normal(n)) for _ in range(u0.shape[0])])
        s.compute_tendency(raw)
    out = s.get_state()
    assert np.all(np.isfinite(out.view(np.float64)))
    s.close()
    print(name, "ok")


if __name__ == "__main__":
    for c in sys.argv[1:] or sorted(CASES):
        main(c)
