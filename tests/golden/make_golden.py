"""Generate the committed golden fixtures from the compiled reference.

Run here (needs /root/reference to build oracle/_ref):
    make -C oracle && python tests/golden/make_golden.py
Each fixture holds the synthetic IC, the reference's tendency of it and the
reference state after `steps` RK4 steps, all produced by the UNMODIFIED
reference core (oracle/_ref/libskref.so = proj/src/*.cpp + oracle/fft_shim.c).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_1807_01769_b200 import ic  # noqa: E402

CASES = [
    # name, solver, n, nu, steps, scheme, seed
    ("ns2d_32", "ns2d", (32, 32), 1e-3, 10, "RK4", 11),
    ("ns2d_64x32", "ns2d", (64, 32), 1e-3, 5, "RK4", 12),
    ("ns2d_128_inviscid", "ns2d", (128, 128), 0.0, 5, "RK4", 13),
    ("ns2d_64_rk2", "ns2d", (64, 64), 1e-3, 5, "RK2", 14),
    ("ns3d_16", "ns3d", (16, 16, 16), 1e-3, 5, "RK4", 15),
    ("ns3d_16x8x32", "ns3d", (16, 8, 32), 2e-3, 3, "RK4", 16),
    # viscous RK4 at grids on the dealiased fast kernels' path (smoke())
    ("ns2d_128", "ns2d", (128, 128), 1e-3, 10, "RK4", 17),
    ("ns3d_32", "ns3d", (32, 32, 32), 1e-3, 5, "RK4", 18),
]


def main(only=None):
    """only: fixture names to (re)generate; None = all."""
    out = Path(__file__).resolve().parent
    for name, solver, n, nu, steps, scheme, seed in CASES:
        if only and name not in only:
            continue
        u0 = ic.initial_state(solver, n, seed)
        dt = ic.cfl_dt(solver, n, u0)
        r = ref.RefSimulation(solver, n, nu, dt, scheme=scheme)
        r.set_state(u0)
        tend = r.tendency(u0)
        r.step(steps)
        np.savez_compressed(out / f"{name}.npz", u0=u0, tendency=tend, final=r.get_state(),
                            n=np.array(n), nu=nu, dt=dt, steps=steps, scheme=scheme,
                            solver=solver, seed=seed, energy=r.energy)
        print(name, "dt", dt, "E", r.energy)
    if only:
        return
    # FFT known answers on the reference's own test shapes (test_fft.cpp:111-124)
    fx = {}
    rng = np.random.default_rng(11)
    for shape in [(8,), (8, 6), (6, 4, 8), (64, 64), (16, 16, 16), (16, 12, 8)]:
        u = rng.uniform(-1, 1, size=shape)
        key = "x".join(map(str, shape))
        fx[f"u_{key}"] = u
        fx[f"uhat_{key}"] = ref.fft_forward(u)
    np.savez_compressed(out / "fft.npz", **fx)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
