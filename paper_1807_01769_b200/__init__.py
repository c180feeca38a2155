"""paper_1807_01769_b200 -- B200-native RK4 step of the pseudo-spectral
Navier-Stokes solvers (ns2d vorticity form, ns3d rotational form).

The compute path is ``_lib/libskgpu.so`` (hand-written sm_100a CUDA behind the
C ABI of ``include/skgpu.h``); this package is the host-side mirror of the
reference's solver/operator interface (spectralkit: ``Simulation``,
``FftPlan``, ``Solver::tendency``).  There is no CPU fallback:
if the library or a GPU is missing, every call raises.
"""
from .api import (  # noqa: F401
    ConfigError,
    CudaError,
    DivergenceError,
    ShapeError,
    SkgError,
    Simulation,
    UnsupportedError,
    fft_forward,
    fft_inverse,
    fp64_peak,
    lib_path,
    load_library,
    nccl_unique_id,
)

__all__ = [
    "Simulation",
    "fft_forward",
    "fft_inverse",
    "SkgError",
    "ConfigError",
    "ShapeError",
    "DivergenceError",
    "CudaError",
    "UnsupportedError",
    "load_library",
    "lib_path",
]
