"""CPU test of the device FFT code itself: fft_block.cuh compiled for the host
(tests/host_emu/fft_block_emu.cpp emulates one thread block with std::thread
and a std::barrier) and compared with numpy.fft on every power-of-two length
the kernels instantiate."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "host_emu" / "fft_block_emu.cpp"
HDR = ROOT / "paper_1807_01769_b200" / "csrc" / "fft_block.cuh"


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    d = tmp_path_factory.mktemp("emu")
    hdr = d / "fft_block_host.cuh"
    hdr.write_text(HDR.read_text().replace("#include <cuda_runtime.h>", ""))
    exe = d / "emu"
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-pthread",
                        f'-DFFT_BLOCK_HEADER="{hdr}"', str(SRC), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
@pytest.mark.parametrize("sign", [-1, 1])
@pytest.mark.parametrize("split", [0, 1, 2, 3])
def test_block_fft_matches_numpy(emu, n, sign, split):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    inp = "\n".join(f"{c.real:.17g} {c.imag:.17g}" for c in x)
    r = subprocess.run([str(emu), str(n), str(sign), str(split)], input=inp, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0
    y = np.array([complex(*map(float, l.split())) for l in r.stdout.splitlines()])
    ref = np.fft.fft(x) if sign < 0 else np.fft.ifft(x) * n
    assert np.abs(y - ref).max() / np.abs(ref).max() < 1e-14
