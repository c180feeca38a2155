"""The reference's OWN Simulation / ExactLinStepper driving the GPU tendency
through the plugin of integration/skgpu_solver.cpp: the
solver registered as "ns2d_gpu"/"ns3d_gpu" must reproduce "ns2d"/"ns3d"."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import ic

PLUGIN = Path(__file__).resolve().parents[1] / "integration" / "_build" / "libskgpu_plugin.so"


def _lib():
    if not PLUGIN.exists():
        pytest.skip("integration plugin not built (needs /root/reference at build time)")
    L = C.CDLL(str(PLUGIN))
    L.skgi_run.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int), C.c_double, C.c_double,
                           C.c_void_p, C.c_long, C.c_void_p]
    L.skgi_last_error.restype = C.c_char_p
    return L


def _run(L, name, n, nu, dt, u0, steps):
    out = np.empty_like(u0)
    cn = (C.c_int * len(n))(*n)
    rc = L.skgi_run(name.encode(), len(n), cn, nu, dt, C.c_void_p(u0.ctypes.data), steps,
                    C.c_void_p(out.ctypes.data))
    assert rc == 0, L.skgi_last_error()
    return out


def test_plugin_library_loads():
    _lib()


@pytest.mark.gpu
@pytest.mark.parametrize("solver,n,nu,steps", [("ns2d", (64, 64), 1e-3, 5),
                                                ("ns2d", (256, 128), 1e-4, 3),
                                                ("ns3d", (16, 16, 16), 1e-3, 3)])
def test_reference_simulation_on_gpu_tendency(solver, n, nu, steps):
    L = _lib()
    u0 = np.ascontiguousarray(ic.initial_state(solver, n, 21))
    dt = ic.cfl_dt(solver, n, u0)
    cpu = _run(L, solver, n, nu, dt, u0, steps)
    gpu = _run(L, solver + "_gpu", n, nu, dt, u0, steps)
    for v in range(u0.shape[0]):
        assert O.rel_l2(gpu[v], cpu[v]) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("solver,n", [("ns2d", (64, 64)), ("ns3d", (16, 16, 16))])
def test_reference_simulation_cfl_on_gpu(solver, n):
    """time_stepping.fixed_dt = 0: the reference's compute_dt asks the GPU
    solver's max_velocity_per_axis (skg_max_velocity) every step."""
    L = _lib()
    u0 = np.ascontiguousarray(ic.initial_state(solver, n, 8))
    cpu = _run(L, solver, n, 1e-3, 0.0, u0, 4)
    gpu = _run(L, solver + "_gpu", n, 1e-3, 0.0, u0, 4)
    for v in range(u0.shape[0]):
        assert O.rel_l2(gpu[v], cpu[v]) < 1e-10


GPUFFT = Path(__file__).resolve().parents[1] / "integration" / "_build" / "libskref_gpufft.so"


@pytest.mark.gpu
@pytest.mark.parametrize("solver,n,steps", [("ns2d", (64, 64), 4), ("ns2d", (24, 40), 3),
                                            ("ns3d", (16, 16, 16), 2), ("ns3d", (12, 8, 16), 2)])
def test_reference_core_on_gpu_fftw(ref_lib, solver, n, steps):
    """B1: the reference's own Simulation with every FftPlan transform on the
    GPU (integration/fftw_gpu.cpp in place of FFTW) vs the CPU reference."""
    if not GPUFFT.exists():
        pytest.skip("GPU FFTW shim not built (needs /root/reference at build time)")
    u0 = np.ascontiguousarray(ic.initial_state(solver, n, 4))
    dt = ic.cfl_dt(solver, n, u0)
    cpu = ref_lib.RefSimulation(solver, n, 1e-3, dt)
    gpu = ref_lib.RefSimulation(solver, n, 1e-3, dt, library=GPUFFT)
    for r in (cpu, gpu):
        r.set_state(u0)
        r.step(steps)
    a, b = gpu.get_state(), cpu.get_state()
    for v in range(u0.shape[0]):
        assert O.rel_l2(a[v], b[v]) < 1e-12
    assert abs(gpu.energy - cpu.energy) <= 1e-12 * cpu.energy
