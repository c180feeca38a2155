"""CPU tests of the C-ABI boundary: the sm_100a library loads, exports
every entry point include/skgpu.h declares, and fails loudly without a GPU
(there is no CPU fallback)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1807_01769_b200 import api

HEADER = Path(__file__).resolve().parents[1] / "include" / "skgpu.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(skg_[a-z0-9_]+)\s*\(", text)))


def test_header_lists_the_python_exports():
    assert set(declared()) == set(api.EXPORTS)


def test_library_exports_every_declared_symbol(gpu_lib):
    for name in declared():
        assert hasattr(gpu_lib, name), name


def test_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(api.lib_path())],
                       capture_output=True, text=True)
    assert r.returncode == 0
    assert "sm_100a" in r.stdout


def test_version(gpu_lib):
    assert b"sm_100a" in gpu_lib.skg_version()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    with pytest.raises(api.CudaError):
        api.Simulation("ns2d", (32, 32), 1e-3, 1e-3)
    with pytest.raises(api.CudaError):
        api.fft_forward(np.zeros((8, 8)))
    with pytest.raises(api.CudaError):
        api.fp64_peak(0)


def test_argument_validation_before_device():
    # same rules as make_grid / plan_fft (grid.cpp:26-38, fft.cpp:34-44)
    with pytest.raises(api.ConfigError):
        api.Simulation("ns4d", (32, 32))
    with pytest.raises(api.ConfigError):
        api.Simulation("ns2d", (31, 32))
    with pytest.raises(api.ConfigError):
        api.Simulation("ns2d", (2, 32))
    with pytest.raises(api.ConfigError):
        api.Simulation("ns2d", (32, 32), nu=-1.0)
    with pytest.raises(api.ConfigError):
        api.Simulation("ns2d", (32, 32), dealias_coef=1.5)
    with pytest.raises(api.ShapeError):
        api.fft_forward(np.zeros((7,)))
    with pytest.raises(api.ShapeError):
        api.fft_forward(np.zeros((2, 2, 2, 2)))
