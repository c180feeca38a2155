"""Cross-check of FFT throughput: cuFFT (via torch.fft) batched FP64 C2C /
C2R / R2C of the lengths the hot path uses, timed with CUDA events.  cuFFT
is a comparison point only; it is never on the product path."""
import json
import sys

import torch


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


out = {}
for n, batch in [(4096, 8192), (512, 65536), (128, 131072)]:
    x = torch.randn(batch, n, dtype=torch.complex128, device="cuda")
    ms = t(lambda: torch.fft.fft(x, dim=-1))
    out[f"c2c_{n}x{batch}"] = {"ms": ms, "ns_per_fft": ms * 1e6 / batch,
                               "GBps": 2 * x.numel() * 16 / ms / 1e6}
    r = torch.randn(batch, n, dtype=torch.float64, device="cuda")
    ms = t(lambda: torch.fft.rfft(r, dim=-1))
    out[f"r2c_{n}x{batch}"] = {"ms": ms, "ns_per_line": ms * 1e6 / batch}
    del x, r
x = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
ms = t(lambda: torch.fft.fft(x, dim=0))
out["c2c_4096_strided_columns"] = {"ms": ms, "ns_per_fft": ms * 1e6 / 4096}
print(json.dumps(out, indent=1))
