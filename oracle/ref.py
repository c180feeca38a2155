"""ctypes binding of oracle/_ref/libskref.so -- the UNMODIFIED reference core.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU legs may import this module; it is the checker and the CPU
baseline, never the measured or shipped path.

The library is built by ``oracle/Makefile`` from /root/reference/proj/src
(compiled in place) + ``oracle/fft_shim.c`` (FFTW-API restatement) +
``oracle/sk_oracle.cpp`` (C driver).  On the GPU box the prebuilt .so is used.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_ref" / "libskref.so"
_lib = None

SOLVER_VARS = {"ns2d": 1, "ns3d": 3}


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def available() -> bool:
    return LIB_PATH.exists()


_libs = {}


def lib(path=None):
    """The compiled reference (default oracle/_ref/libskref.so); `path` loads
    another build of the same driver, e.g. the reference core linked against
    the GPU-backed FFTW API (integration/_build/libskref_gpufft.so)."""
    key = str(path or LIB_PATH)
    if key not in _libs:
        if not Path(key).exists():
            raise FileNotFoundError(f"{key} missing: run `make -C oracle`")
        L = C.CDLL(key)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.skref_last_error.restype = C.c_char_p
        L.skref_set_workers.argtypes = [C.c_int]
        L.skref_create.argtypes = [C.POINTER(C.c_void_p), C.c_char_p, C.c_int, ip,
                                   C.c_double, C.c_double, C.c_int, C.c_double]
        L.skref_destroy.argtypes = [C.c_void_p]
        L.skref_create_forced.argtypes = [C.POINTER(C.c_void_p), C.c_char_p, C.c_int, ip,
                                          C.c_double, C.c_double, C.c_int, C.c_double,
                                          C.c_double, C.c_double, C.c_double, C.c_long]
        L.skref_create_files.argtypes = [C.POINTER(C.c_void_p), C.c_char_p, C.c_int, ip,
                                         C.c_double, C.c_double, C.c_int, C.c_double,
                                         C.c_char_p, C.c_double]
        L.skref_output_dir.argtypes = [C.c_void_p, C.c_char_p, C.c_long]
        L.skref_restart.argtypes = [C.POINTER(C.c_void_p), C.c_char_p, C.c_double]
        L.skref_last_injection.argtypes = [C.c_void_p]
        L.skref_last_injection.restype = C.c_double
        for f in ("skref_spect_size", "skref_phys_size", "skref_iteration"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_long
        L.skref_nvars.argtypes = [C.c_void_p]
        for f in ("skref_energy", "skref_enstrophy", "skref_time"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_double
        L.skref_set_state.argtypes = [C.c_void_p, dp]
        L.skref_get_state.argtypes = [C.c_void_p, dp]
        L.skref_step.argtypes = [C.c_void_p, C.c_long, dp]
        L.skref_run.argtypes = [C.c_void_p, C.c_long, dp]
        L.skref_tendency.argtypes = [C.c_void_p, dp, dp]
        L.skref_grid.argtypes = [C.c_void_p, C.c_int, dp, C.POINTER(C.c_ubyte)]
        L.skref_last_divergence.argtypes = [C.c_void_p, C.POINTER(C.c_long), ip]
        L.skref_fft_forward.argtypes = [C.c_int, ip, dp, dp]
        L.skref_fft_inverse.argtypes = [C.c_int, ip, dp, dp]
        _libs[key] = L
    return _libs[key]


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().skref_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def set_workers(n: int) -> None:
    """set_fft_workers (proj/src/fft.cpp:51-54); capped by SPECTRALKIT_NUM_THREADS."""
    lib().skref_set_workers(int(n))


def fft_forward(u: np.ndarray) -> np.ndarray:
    """FftPlan::forward (proj/src/fft.cpp:92-98): r2c then *= 1/N."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    shape = (C.c_int * u.ndim)(*u.shape)
    out = np.empty(u.shape[:-1] + (u.shape[-1] // 2 + 1,), np.complex128)
    _check(lib().skref_fft_forward(u.ndim, shape, _dp(u), _dp(out.view(np.float64))))
    return out


def fft_inverse(uhat: np.ndarray, shape) -> np.ndarray:
    """FftPlan::inverse (proj/src/fft.cpp:100-106): unnormalised c2r, input kept."""
    uhat = np.ascontiguousarray(uhat, dtype=np.complex128)
    cs = (C.c_int * len(shape))(*shape)
    out = np.empty(tuple(shape), np.float64)
    _check(lib().skref_fft_inverse(len(shape), cs, _dp(uhat.view(np.float64)), _dp(out)))
    return out


class RefSimulation:
    """A reference ``Simulation`` (proj/src/simulation.cpp:297-346) with files
    and forcing off, fixed dt and an injected spectral state."""

    def __init__(self, solver: str, n, nu: float, dt: float, scheme: str = "RK4",
                 dealias_coef: float = 2.0 / 3.0, forcing=None, library=None, files=None,
                 _handle=None):
        """forcing: None, or (k_lo, k_hi, rate, seed) for forcing.enable = true.
        files: None, or (root_dir, period_save): output.enable_files = true
        (the OutputManager writes the run directory, output.cpp:105-300)."""
        self.solver = solver
        self.n = tuple(int(x) for x in n)
        self._L = lib(library)
        h = C.c_void_p()
        cn = (C.c_int * len(self.n))(*self.n)
        rk2 = 1 if scheme.upper() == "RK2" else 0
        if _handle is not None:
            h = _handle
        elif files is not None:
            root, period = files
            _check(self._L.skref_create_files(C.byref(h), solver.encode(), len(self.n), cn, float(nu),
                                            float(dt), rk2, float(dealias_coef),
                                            str(root).encode(), float(period)))
        elif forcing is None:
            _check(self._L.skref_create(C.byref(h), solver.encode(), len(self.n), cn, float(nu),
                                      float(dt), rk2, float(dealias_coef)))
        else:
            klo, khi, rate, seed = forcing
            _check(self._L.skref_create_forced(C.byref(h), solver.encode(), len(self.n), cn,
                                             float(nu), float(dt), rk2, float(dealias_coef),
                                             float(klo), float(khi), float(rate), int(seed)))
        self._h = h
        self.nvars = self._L.skref_nvars(h)
        self.spect_shape = self.n[:-1] + (self.n[-1] // 2 + 1,)

    @classmethod
    def restart(cls, run_dir, solver: str, n, time: float = -1.0, library=None):
        """load_state_phys_file(run_dir, time) (proj/src/simulation.cpp:705-732):
        a Simulation from run_dir/params.txt and the snapshot nearest `time`
        (time < 0: the latest), whose digest must match the params."""
        L = lib(library)
        h = C.c_void_p()
        _check(L.skref_restart(C.byref(h), str(run_dir).encode(), float(time)))
        return cls(solver, n, 0.0, 0.0, library=library, _handle=h)

    @property
    def output_dir(self) -> str:
        buf = C.create_string_buffer(4096)
        _check(self._L.skref_output_dir(self._h, buf, 4096))
        return buf.value.decode()

    def close(self):
        if self._h:
            self._L.skref_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_state(self, s: np.ndarray) -> None:
        s = np.ascontiguousarray(s, dtype=np.complex128).reshape((self.nvars,) + self.spect_shape)
        _check(self._L.skref_set_state(self._h, _dp(s.view(np.float64))))

    def get_state(self) -> np.ndarray:
        out = np.empty((self.nvars,) + self.spect_shape, np.complex128)
        _check(self._L.skref_get_state(self._h, _dp(out.view(np.float64))))
        return out

    def step(self, nsteps: int = 1) -> float:
        """step_once x nsteps (simulation.cpp:535-555); returns wall seconds."""
        sec = C.c_double(0.0)
        _check(self._L.skref_step(self._h, int(nsteps), C.byref(sec)))
        return sec.value

    def run(self, nsteps: int) -> float:
        """Simulation::run with n_iters = nsteps (simulation.cpp:565-590)."""
        sec = C.c_double(0.0)
        _check(self._L.skref_run(self._h, int(nsteps), C.byref(sec)))
        return sec.value

    def tendency(self, s: np.ndarray) -> np.ndarray:
        """Solver::tendency via Simulation::compute_tendency (simulation.cpp:478-480)."""
        s = np.ascontiguousarray(s, dtype=np.complex128).reshape((self.nvars,) + self.spect_shape)
        out = np.empty_like(s)
        _check(self._L.skref_tendency(self._h, _dp(s.view(np.float64)), _dp(out.view(np.float64))))
        return out

    def grid(self):
        """(k_axis list, dealias mask) from make_grid (proj/src/grid.cpp:20-110)."""
        ks = []
        mask = np.empty(self.spect_shape, np.uint8)
        for ax in range(len(self.n)):
            k = np.empty(self.spect_shape[ax], np.float64)
            _check(self._L.skref_grid(self._h, ax, _dp(k),
                                    mask.ctypes.data_as(C.POINTER(C.c_ubyte))))
            ks.append(k)
        return ks, mask

    def last_divergence(self):
        it = C.c_long(-1)
        var = C.c_int(-1)
        self._L.skref_last_divergence(self._h, C.byref(it), C.byref(var))
        return it.value, var.value

    @property
    def energy(self) -> float:
        return self._L.skref_energy(self._h)

    @property
    def enstrophy(self) -> float:
        return self._L.skref_enstrophy(self._h)

    @property
    def last_injection(self) -> float:
        return self._L.skref_last_injection(self._h)

    @property
    def t(self) -> float:
        return self._L.skref_time(self._h)

    @property
    def iteration(self) -> int:
        return self._L.skref_iteration(self._h)
