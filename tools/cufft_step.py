"""Library baseline (comparison only, never on the product path): the same
ns2d RK4 step written with cuFFT (torch.fft, FP64) and torch elementwise ops,
in the Basdevant form the fused path uses (2 inverse + 2 forward real 2D FFTs
per stage, 2/3 mask, integrating factors), timed with CUDA events at the
BASELINE grids and checked against libskgpu after a few steps.

    python tools/cufft_step.py [4096 1024]       ->  one JSON line per grid
    python tools/cufft_step.py ns3d [128 512]   (rotational form, Leray projection)
"""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1807_01769_b200 import api, ic  # noqa: E402


def make_step(n, nu, dt, dev):
    nx, ny = n
    kx = torch.fft.fftfreq(nx, 1.0 / nx, dtype=torch.float64, device=dev)[:, None]
    ky = torch.arange(ny // 2 + 1, dtype=torch.float64, device=dev)[None, :]
    k2 = kx * kx + ky * ky
    inv_k2 = torch.where(k2 > 0, 1.0 / torch.where(k2 > 0, k2, 1.0), torch.zeros_like(k2))
    kc = [(2.0 / 3.0) * (nx // 2), (2.0 / 3.0) * (ny // 2)]
    mask = ((kx.abs() <= kc[0]) & (ky.abs() <= kc[1])).to(torch.float64)
    mask[0, 0] = 0.0  # mean of the tendency
    sig = -nu * k2
    e1, e2 = torch.exp(0.5 * dt * sig), torch.exp(dt * sig)
    N = nx * ny

    def tend(w):
        psi = w * inv_k2
        u = torch.fft.irfft2(1j * ky * psi, s=n) * N
        v = torch.fft.irfft2(-1j * kx * psi, s=n) * N
        a = torch.fft.rfft2(v * v - u * u) / N
        b = torch.fft.rfft2(u * v) / N
        return (kx * ky * a + (kx * kx - ky * ky) * b) * mask

    def step(w):
        k1 = tend(w)
        k2_ = tend(e1 * (w + 0.5 * dt * k1))
        k3 = tend(e1 * w + 0.5 * dt * k2_)
        k4 = tend(e2 * w + dt * e1 * k3)
        return e2 * w + dt / 6.0 * (e2 * k1 + 2.0 * e1 * (k2_ + k3) + k4)

    return step


def make_step3(n, nu, dt, dev):
    """ns3d rotational form (solvers.cpp:299-339): curl, 6 c2r, u x w, 3 r2c,
    Leray projection, 2/3 mask, mean 0; integrating-factor RK4."""
    nx, ny, nz = n
    kx = torch.fft.fftfreq(nx, 1.0 / nx, dtype=torch.float64, device=dev)[:, None, None]
    ky = torch.fft.fftfreq(ny, 1.0 / ny, dtype=torch.float64, device=dev)[None, :, None]
    kz = torch.arange(nz // 2 + 1, dtype=torch.float64, device=dev)[None, None, :]
    k2 = kx * kx + ky * ky + kz * kz
    inv_k2 = torch.where(k2 > 0, 1.0 / torch.where(k2 > 0, k2, 1.0), torch.zeros_like(k2))
    kc = [(2.0 / 3.0) * (m // 2) for m in n]
    mask = ((kx.abs() <= kc[0]) & (ky.abs() <= kc[1]) & (kz <= kc[2])).to(torch.float64)
    mask[0, 0, 0] = 0.0
    sig = -nu * k2
    e1, e2 = torch.exp(0.5 * dt * sig), torch.exp(dt * sig)
    N = nx * ny * nz
    inv = lambda f: torch.fft.irfftn(f, s=n) * N  # noqa: E731
    fwd = lambda f: torch.fft.rfftn(f) / N  # noqa: E731

    def tend(v):
        vx, vy, vz = v[0], v[1], v[2]
        ux, uy, uz = inv(vx), inv(vy), inv(vz)
        ox = inv(1j * (ky * vz - kz * vy))
        oy = inv(1j * (kz * vx - kx * vz))
        oz = inv(1j * (kx * vy - ky * vx))
        cx, cy, cz = fwd(uy * oz - uz * oy), fwd(uz * ox - ux * oz), fwd(ux * oy - uy * ox)
        kdot = (kx * cx + ky * cy + kz * cz) * inv_k2
        return torch.stack([(cx - kx * kdot) * mask, (cy - ky * kdot) * mask, (cz - kz * kdot) * mask])

    def step(w):
        k1 = tend(w)
        k2_ = tend(e1 * (w + 0.5 * dt * k1))
        k3 = tend(e1 * w + 0.5 * dt * k2_)
        k4 = tend(e2 * w + dt * e1 * k3)
        return e2 * w + dt / 6.0 * (e2 * k1 + 2.0 * e1 * (k2_ + k3) + k4)

    return step


def main3(n, nu):
    dev = torch.device("cuda", 0)
    n3 = (n, n, n)
    u0 = ic.ns3d_ic(n3, seed=1234)
    dt = ic.cfl_dt("ns3d", n3, u0)
    step = make_step3(n3, nu, dt, dev)
    x = step(torch.from_numpy(u0).to(dev))
    sim = api.Simulation("ns3d", n3, nu, dt, device=0)
    sim.set_state(u0)
    sim.step(1)
    ref = torch.from_numpy(sim.get_state()).to(dev)
    rel = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
    sim.close()
    del ref
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 3
    s.record()
    for _ in range(steps):
        x = step(x)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    print(json.dumps({"grid": f"{n}^3", "impl": "cuFFT (torch.fft) + torch elementwise, FP64",
                      "ms_per_step": ms, "Gpts_steps_per_s": n ** 3 / ms / 1e6,
                      "rel_l2_vs_libskgpu_after_1_step": rel}), flush=True)


def main():
    dev = torch.device("cuda", 0)
    for n in [int(x) for x in (sys.argv[1:] or ["4096", "1024"])]:
        n2 = (n, n)
        u0 = ic.ns2d_ic(n2, seed=1234)
        dt = ic.cfl_dt("ns2d", n2, u0)
        step = make_step(n2, 1e-4, dt, dev)
        w = torch.from_numpy(u0[0]).to(dev)
        # validity: 3 steps against libskgpu
        x = w
        for _ in range(3):
            x = step(x)
        sim = api.Simulation("ns2d", n2, 1e-4, dt, device=0)
        sim.set_state(u0)
        sim.step(3)
        ref = torch.from_numpy(sim.get_state()[0]).to(dev)
        rel = float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))
        sim.close()
        for _ in range(3):
            x = step(x)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 20
        s.record()
        for _ in range(steps):
            x = step(x)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        print(json.dumps({"grid": f"{n}x{n}", "impl": "cuFFT (torch.fft) + torch elementwise, FP64",
                          "ms_per_step": ms, "Gpts_steps_per_s": n * n / ms / 1e6,
                          "rel_l2_vs_libskgpu_after_3_steps": rel}), flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["ns3d"]:
        for m in (sys.argv[2:] or ["128", "512"]):
            main3(int(m), 1e-3 if int(m) <= 128 else 2e-4)
    else:
        main()
