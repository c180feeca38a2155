"""Host mirror of the reference interface over the C ABI (include/skgpu.h).

Names and semantics follow spectralkit (paths relative to
/root/reference/proj):
  Simulation.step_once / run / compute_tendency / energy / enstrophy
      -> simulation.hpp:127-151 (fixed dt, forcing and files off)
  Simulation.state (spectral, reference layout)  -> state.hpp (StateSet)
  fft_forward / fft_inverse                       -> FftPlan::forward / inverse (fft.cpp:92-106)
  exceptions                                      -> errors.hpp (ConfigError, ShapeError,
                                                     DivergenceError(iteration, field))
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
_LIB_PATH = _PKG / "_lib" / "libskgpu.so"
_lib = None

SKG_OK, SKG_ECONFIG, SKG_ESHAPE, SKG_EDIVERGENCE, SKG_ECUDA, SKG_ENCCL, SKG_EUNSUPPORTED = range(7)
SKG_RK4, SKG_RK2 = 0, 1

KEYS_STATE_SPECT = {"ns2d": ["rot_fft"], "ns3d": ["vx_fft", "vy_fft", "vz_fft"]}
KEYS_STATE_PHYS = {"ns2d": ["rot"], "ns3d": ["vx", "vy", "vz"]}
KEYS_COMPUTABLE = {"ns2d": ["ux", "uy"], "ns3d": ["rotz"]}  # solvers.cpp:196, 359

EXPORTS = [
    "skg_version", "skg_last_error", "skg_create", "skg_destroy", "skg_set_stream",
    "skg_spect_size", "skg_phys_size", "skg_nvars", "skg_set_state", "skg_get_state",
    "skg_set_state_device", "skg_get_state_device", "skg_step", "skg_step_async", "skg_sync",
    "skg_iteration", "skg_time", "skg_tendency", "skg_fft_forward", "skg_fft_inverse",
    "skg_plan_forward", "skg_plan_inverse", "skg_get_grid", "skg_last_divergence",
    "skg_energy", "skg_pruned", "skg_launch_count", "skg_set_timing", "skg_kernel_stats",
    "skg_reset_stats", "skg_fp64_peak", "skg_nccl_unique_id", "skg_create_dist", "skg_create_pencil",
    "skg_run",
    "skg_set_cfl", "skg_last_dt", "skg_set_time", "skg_max_velocity", "skg_diagnostics",
    "skg_set_forcing", "skg_last_injection", "skg_sanitize_state", "skg_spectra",
    "skg_dist_p2p", "skg_dist_overlap", "skg_guard_violations", "skg_dist_ipc_handle", "skg_dist_open_peers", "skg_dft_r2c", "skg_dft_c2r",
]


class SkgError(RuntimeError):
    """Base class (spectralkit::Error)."""


class ConfigError(SkgError):
    pass


class ShapeError(SkgError):
    pass


class CudaError(SkgError):
    pass


class UnsupportedError(SkgError):
    pass


class DivergenceError(SkgError):
    """Non-finite state after a step (errors.hpp:44-51)."""

    def __init__(self, msg: str, iteration: int, field: str):
        super().__init__(msg)
        self.iteration = iteration
        self.field = field


def lib_path() -> Path:
    return _LIB_PATH


def load_library():
    """Load the sm_100a library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    # SKG_LIB_VARIANT=name loads _lib/variants/libskgpu_<name>.so (A/B builds
    # of the same sources with different tuning macros; tools/variants.sh)
    var = os.environ.get("SKG_LIB_VARIANT")
    path = _LIB_PATH.parent / "variants" / f"libskgpu_{var}.so" if var else _LIB_PATH
    if not path.exists():
        raise SkgError(f"{path} is missing: run `python -m paper_1807_01769_b200.build`")
    L = C.CDLL(str(path))
    vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
    L.skg_version.restype = C.c_char_p
    L.skg_last_error.restype = C.c_char_p
    L.skg_create.argtypes = [C.POINTER(vp), C.c_char_p, C.c_int, ip, dp, C.c_double, C.c_double,
                             C.c_int, C.c_int]
    L.skg_destroy.argtypes = [vp]
    L.skg_create_dist.argtypes = [C.POINTER(vp), C.c_char_p, C.c_int, ip, dp, C.c_double,
                                  C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p]
    L.skg_create_pencil.argtypes = [C.POINTER(vp), C.c_char_p, C.c_int, ip, dp, C.c_double,
                                    C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_char_p]
    L.skg_nccl_unique_id.argtypes = [C.c_char_p]
    L.skg_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.skg_set_stream.argtypes = [vp, vp]
    for f in ("skg_spect_size", "skg_phys_size", "skg_iteration", "skg_launch_count"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = C.c_long
    for f in ("skg_nvars", "skg_pruned"):
        getattr(L, f).argtypes = [vp]
    L.skg_time.argtypes = [vp]
    L.skg_time.restype = C.c_double
    for f in ("skg_set_state", "skg_get_state", "skg_set_state_device", "skg_get_state_device"):
        getattr(L, f).argtypes = [vp, C.c_void_p]
    L.skg_step.argtypes = [vp, C.c_double, C.c_long]
    L.skg_run.argtypes = [vp, C.c_double, C.c_long, C.c_void_p]
    L.skg_step_async.argtypes = [vp, C.c_double, C.c_long]
    L.skg_sync.argtypes = [vp]
    L.skg_tendency.argtypes = [vp, C.c_void_p, C.c_void_p]
    L.skg_fft_forward.argtypes = [vp, C.c_void_p, C.c_void_p]
    L.skg_fft_inverse.argtypes = [vp, C.c_void_p, C.c_void_p]
    L.skg_plan_forward.argtypes = [C.c_int, ip, C.c_void_p, C.c_void_p, C.c_int]
    L.skg_plan_inverse.argtypes = [C.c_int, ip, C.c_void_p, C.c_void_p, C.c_int]
    L.skg_get_grid.argtypes = [vp, C.c_int, C.c_void_p, C.c_void_p]
    L.skg_last_divergence.argtypes = [vp, C.POINTER(C.c_long), ip]
    L.skg_energy.argtypes = [vp, dp, dp]
    L.skg_set_timing.argtypes = [vp, C.c_int]
    L.skg_kernel_stats.argtypes = [vp, C.c_int, dp, C.POINTER(C.c_long), dp]
    L.skg_reset_stats.argtypes = [vp]
    L.skg_set_cfl.argtypes = [vp, C.c_double, C.c_double, C.c_double]
    L.skg_last_dt.argtypes = [vp]
    L.skg_last_dt.restype = C.c_double
    L.skg_set_time.argtypes = [vp, C.c_double]
    L.skg_max_velocity.argtypes = [vp, C.c_void_p, C.c_void_p]
    L.skg_diagnostics.argtypes = [vp, C.c_void_p]
    L.skg_set_forcing.argtypes = [vp, C.c_int, C.c_double, C.c_double, C.c_double, C.c_long]
    L.skg_last_injection.argtypes = [vp]
    L.skg_last_injection.restype = C.c_double
    L.skg_sanitize_state.argtypes = [vp]
    L.skg_dist_p2p.argtypes = [vp, C.c_int]
    L.skg_dist_overlap.argtypes = [vp, C.c_int]
    L.skg_guard_violations.argtypes = []
    L.skg_guard_violations.restype = C.c_long
    L.skg_dist_ipc_handle.argtypes = [vp, C.c_char_p]
    L.skg_dist_open_peers.argtypes = [vp, C.c_char_p]
    L.skg_spectra.argtypes = [vp, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.POINTER(C.c_int)]
    _lib = L
    return L


def _raise(rc: int, ctx=None, solver=None):
    L = load_library()
    msg = L.skg_last_error().decode()
    if rc == SKG_ECONFIG:
        raise ConfigError(msg)
    if rc == SKG_ESHAPE:
        raise ShapeError(msg)
    if rc == SKG_EDIVERGENCE:
        it = C.c_long(-1)
        var = C.c_int(-1)
        L.skg_last_divergence(ctx, C.byref(it), C.byref(var))
        keys = KEYS_STATE_SPECT.get(solver, ["?"])
        field = keys[var.value] if 0 <= var.value < len(keys) else "?"
        raise DivergenceError(msg, it.value, field)
    if rc == SKG_EUNSUPPORTED:
        raise UnsupportedError(msg)
    if rc == SKG_ECUDA:
        raise CudaError(msg)
    raise SkgError(f"[{rc}] {msg}")


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _check_shape(shape):
    shape = tuple(int(x) for x in shape)
    if not 1 <= len(shape) <= 3:
        raise ShapeError(f"transform rank must be 1..3, got {len(shape)}")
    for n in shape:
        if n < 4:
            raise ShapeError(f"extent {n} too small (min 4)")
        if n % 2:
            raise ShapeError(f"extent {n} is odd")
    return shape


def fp64_peak(device: int = 0) -> float:
    """Measured DFMA thread-instructions per second of `device` (skg_fp64_peak;
    2 flops each): the FP64 ceiling of bench.py's butterfly roofline."""
    out = C.c_double(0.0)
    rc = load_library().skg_fp64_peak(int(device), C.byref(out))
    if rc:
        _raise(rc)
    return out.value


def guard_violations() -> int:
    """Changed guard bytes around the library's device allocations
    (SKG_GUARD=1 debug mode, skg_guard_violations); 0 when the mode is off."""
    return int(load_library().skg_guard_violations())


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for skg_create_dist (rank 0 creates, the caller broadcasts)."""
    buf = C.create_string_buffer(128)
    rc = load_library().skg_nccl_unique_id(buf)
    if rc:
        _raise(rc)
    return buf.raw


def fft_forward(u: np.ndarray, device: int = 0) -> np.ndarray:
    """FftPlan::forward (fft.cpp:92-98) of a real field on the GPU."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    shape = _check_shape(u.shape)
    out = np.empty(shape[:-1] + (shape[-1] // 2 + 1,), np.complex128)
    cs = (C.c_int * len(shape))(*shape)
    rc = load_library().skg_plan_forward(len(shape), cs, _ptr(u), _ptr(out), device)
    if rc:
        _raise(rc)
    return out


def fft_inverse(uhat: np.ndarray, shape, device: int = 0) -> np.ndarray:
    """FftPlan::inverse (fft.cpp:100-106): unnormalised c2r, input intact."""
    shape = _check_shape(shape)
    uhat = np.ascontiguousarray(uhat, dtype=np.complex128)
    if uhat.shape != shape[:-1] + (shape[-1] // 2 + 1,):
        raise ShapeError(f"inverse: field has shape {uhat.shape}, plan expects "
                         f"{shape[:-1] + (shape[-1] // 2 + 1,)}")
    out = np.empty(shape, np.float64)
    cs = (C.c_int * len(shape))(*shape)
    rc = load_library().skg_plan_inverse(len(shape), cs, _ptr(uhat), _ptr(out), device)
    if rc:
        _raise(rc)
    return out


class Simulation:
    """Device-resident counterpart of spectralkit::Simulation for ns2d/ns3d
    with fixed dt and forcing/output off (the bench protocol, bench.cpp:51-85)."""

    def __init__(self, solver: str, n, nu: float = 0.0, dt: float = 0.0, scheme: str = "RK4",
                 L=None, dealias_coef: float = 2.0 / 3.0, device: int = 0, world: int = 1,
                 rank: int = 0, nccl_id: bytes | None = None, compact: bool = False,
                 pencil: tuple[int, int] | None = None):
        """world > 1: slab decomposition (ns2d and ns3d).  With nccl_id (from
        nccl_unique_id() on rank 0) this process runs partition `rank` over
        NCCL; without it all `world` partitions run here on one device.
        compact (ns3d, world 1): the kept-modes-only layout of the slab path
        on one GPU (dealiased states only; 1024^3 fits one B200).
        pencil = (py, pz) (ns3d): 2D process grid of py * pz ranks
        (skg_create_pencil; world is then py * pz, rank = r_y * pz + r_z)."""
        L_ = load_library()
        self.solver = solver
        self.n = tuple(int(x) for x in n)
        self.dims = len(self.n)
        self.nu = float(nu)
        self.dt = float(dt)
        self.scheme = scheme.upper()
        if self.scheme not in ("RK4", "RK2"):
            raise ConfigError(f"unknown time scheme '{scheme}' (use RK2 or RK4)")
        self.spect_shape = self.n[:-1] + (self.n[-1] // 2 + 1,)
        h = C.c_void_p()
        cn = (C.c_int * self.dims)(*self.n)
        cL = None if L is None else (C.c_double * self.dims)(*L)
        sch = SKG_RK2 if self.scheme == "RK2" else SKG_RK4
        if pencil is not None:
            py, pz = (int(x) for x in pencil)
            world = py * pz
            rc = L_.skg_create_pencil(C.byref(h), solver.encode(), self.dims, cn, cL,
                                      float(dealias_coef), self.nu, sch, int(device), int(rank),
                                      py, pz, nccl_id)
        elif world > 1 or (compact and solver == "ns3d"):
            rc = L_.skg_create_dist(C.byref(h), solver.encode(), self.dims, cn, cL,
                                    float(dealias_coef), self.nu, sch, int(device), int(rank),
                                    int(world), nccl_id)
        else:
            rc = L_.skg_create(C.byref(h), solver.encode(), self.dims, cn, cL, float(dealias_coef),
                               self.nu, sch, int(device))
        self.world = int(world)
        self.rank = int(rank)
        self.pencil = None if pencil is None else (py, pz)
        self._nccl = nccl_id
        if rc:
            _raise(rc)
        self._h = h
        self.nvars = L_.skg_nvars(h)
        self.keys_state_spect = KEYS_STATE_SPECT[solver]
        self.L = tuple(float(x) for x in (L if L is not None else [2 * np.pi] * self.dims))
        self._cfl = None          # (cfl_coef, dt_max) when the dt is adaptive
        self._t_end = None        # stopping rule of run() (Simulation::run)
        self._n_iters = None

    # --------------------------------------------- reference-style construction
    @classmethod
    def from_params(cls, params, device: int = 0, **kw):
        """From the reference's parameter leaves (create_default_params,
        simulation.cpp:73-125): a dict (or anything with .get) keyed by leaf
        path -- "solver", "nu_2", "oper.nx", "oper.Lx", "oper.dealias_coef",
        "time_stepping.scheme", "fixed_dt", "cfl_coef", "dt_max", "t_end",
        "n_iters".  fixed_dt = 0 selects the CFL dt.  Exactly one stopping
        rule, as the reference checks (simulation.cpp:246-251)."""
        g = params.get
        solver = g("solver")
        if solver not in KEYS_STATE_SPECT:
            raise ConfigError(f"unknown solver '{solver}' (registered: ns2d, ns3d)")
        dims = 2 if solver == "ns2d" else 3
        n = tuple(int(g(f"oper.{a}", 16)) for a in ("nx", "ny", "nz")[:dims])
        L = [float(g(f"oper.L{a}", 2 * np.pi)) for a in "xyz"[:dims]]
        t_end = float(g("time_stepping.t_end", 1.0))
        n_iters = int(g("time_stepping.n_iters", -1))
        if (t_end >= 0.0) == (n_iters >= 0):
            raise ConfigError("exactly one stopping rule: set time_stepping.t_end >= 0 "
                              "or time_stepping.n_iters >= 0, not both")
        fixed_dt = float(g("time_stepping.fixed_dt", 0.0))
        if fixed_dt < 0.0:
            raise ConfigError("time_stepping.fixed_dt must be >= 0")
        sim = cls(solver, n, float(g("nu_2", 0.0)), fixed_dt, str(g("time_stepping.scheme", "RK4")),
                  L=L, dealias_coef=float(g("oper.dealias_coef", 2.0 / 3.0)), device=device, **kw)
        if fixed_dt == 0.0:
            sim.set_cfl(float(g("time_stepping.cfl_coef", 0.5)), float(g("time_stepping.dt_max", 0.1)))
        if n_iters >= 0:
            sim.set_n_iters(n_iters)
        else:
            sim.set_t_end(t_end)
        if g("forcing.enable", False):
            sim.set_forcing(float(g("forcing.k_lo", 2.0)), float(g("forcing.k_hi", 4.0)),
                            float(g("forcing.rate", 1.0)), int(g("forcing.seed", 1234)))
        return sim

    @property
    def solver_name(self) -> str:
        return self.solver

    @property
    def shape(self):
        return list(self.n)

    @property
    def state_keys(self):
        return list(KEYS_STATE_PHYS[self.solver])

    @property
    def computable_keys(self):
        return list(KEYS_COMPUTABLE[self.solver])

    # ------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            load_library().skg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _call(self, fn, *args):
        rc = getattr(load_library(), fn)(self._h, *args)
        if rc:
            _raise(rc, self._h, self.solver)

    # ----------------------------------------------------------------- state
    def set_state(self, spect: np.ndarray) -> None:
        s = np.ascontiguousarray(spect, dtype=np.complex128)
        if s.size != self.nvars * int(np.prod(self.spect_shape)):
            raise ShapeError(f"state has {s.size} modes, expected "
                             f"{self.nvars} x {self.spect_shape}")
        self._call("skg_set_state", _ptr(s))

    def get_state(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.nvars,) + self.spect_shape, np.complex128)
        elif (out.dtype != np.complex128 or not out.flags.c_contiguous
              or out.size != self.nvars * int(np.prod(self.spect_shape))):
            raise ShapeError("get_state: out must be a contiguous complex128 array of the state size")
        self._call("skg_get_state", _ptr(out))
        return out

    def set_state_device(self, ptr: int) -> None:
        self._call("skg_set_state_device", C.c_void_p(ptr))

    def get_state_device(self, ptr: int) -> None:
        self._call("skg_get_state_device", C.c_void_p(ptr))

    def set_stream(self, stream_ptr) -> None:
        self._call("skg_set_stream", C.c_void_p(stream_ptr))

    # ---------------------------------------------------------------- stepping
    def step_once(self, dt: float | None = None) -> None:
        self.step(1, dt)

    def set_forcing(self, k_lo: float = 2.0, k_hi: float = 4.0, rate: float = 1.0, seed: int = 1234,
                    enable: bool = True) -> None:
        """forcing.* (simulation.cpp:112-117, 482-548): random band forcing
        injecting `rate`, refreshed before every step from the reference's
        own generator seeded with `seed`."""
        self._call("skg_set_forcing", C.c_int(1 if enable else 0), C.c_double(k_lo),
                   C.c_double(k_hi), C.c_double(rate), C.c_long(int(seed)))

    def spectra(self) -> dict:
        """Shell spectra as the reference's OutputManager records them
        (output.cpp:231-257): {"k", "E" (density), "T" (transfer), "D"}."""
        ns = C.c_int()
        self._call("skg_spectra", C.c_int(0), None, None, None, None, C.byref(ns))
        arr = {key: np.zeros(ns.value, np.float64) for key in ("k", "E", "T", "D")}
        self._call("skg_spectra", C.c_int(ns.value), _ptr(arr["k"]), _ptr(arr["E"]), _ptr(arr["T"]),
                   _ptr(arr["D"]), C.byref(ns))
        return arr

    # ------------------------------------------------------- snapshot files
    def save_fld(self, path, digest: str = "") -> None:
        """The reference's physical snapshot format (snapshot.cpp:65-100:
        "spectralkit-fld 1" header, time, shape, vars, digest, blank line,
        little-endian doubles per variable).  `digest` is the reference's
        params_digest when the file must pass its restart check."""
        keys = self.state_keys
        with open(path, "wb") as f:
            f.write(b"spectralkit-fld 1\n")
            f.write(f"time={self.t:.17g}\n".encode())
            f.write(("shape=" + "x".join(str(x) for x in self.n) + "\n").encode())
            f.write(("vars=" + ",".join(keys) + "\n").encode())
            f.write(f"digest={digest}\n\n".encode())
            for key in keys:
                f.write(np.ascontiguousarray(self.get_phys(key), dtype="<f8").tobytes())

    def load_fld(self, path, set_time: bool = True) -> dict:
        """Load a "spectralkit-fld 1" snapshot (snapshot.cpp:117-160) into the
        state (StateSet::load_phys per variable); returns its header."""
        with open(path, "rb") as f:
            if f.readline().rstrip(b"\n") != b"spectralkit-fld 1":
                raise ConfigError(f"'{path}': not a spectralkit-fld file")
            hdr = {}
            for key in ("time", "shape", "vars", "digest"):
                line = f.readline().decode().rstrip("\n")
                if not line.startswith(key + "="):
                    raise ConfigError(f"'{path}': expected header field '{key}', got '{line}'")
                hdr[key] = line[len(key) + 1:]
            if f.readline().strip():
                raise ConfigError(f"'{path}': header must end with a blank line")
            shape = tuple(int(x) for x in hdr["shape"].split("x"))
            if shape != self.n:
                raise ShapeError(f"snapshot shape {shape} does not match the grid {self.n}")
            size = int(np.prod(shape))
            for key in hdr["vars"].split(","):
                data = np.frombuffer(f.read(8 * size), dtype="<f8")
                if data.size != size:
                    raise ConfigError(f"'{path}': truncated payload for variable '{key}'")
                self.set_phys(key, data.reshape(shape))
        hdr["time"] = float(hdr["time"])
        if set_time:
            self.set_time(hdr["time"])
        return hdr

    def enable_p2p(self, all_gather=None) -> None:
        """Peer-memory exchange for the slab (ns2d and ns3d): producers store
        straight into the owners' receive buffers.  Single process: no argument.  One
        process per GPU: `all_gather(bytes) -> list[bytes]` in rank order
        (default: torch.distributed.all_gather_object)."""
        if self.world <= 1:
            raise UnsupportedError("peer exchange needs a slab-decomposed context")
        if getattr(self, "_nccl", None) is None:
            self._call("skg_dist_p2p", C.c_int(1))
            return
        mine = C.create_string_buffer(256)
        self._call("skg_dist_ipc_handle", mine)
        if all_gather is None:
            import torch.distributed as dist
            out = [None] * self.world
            dist.all_gather_object(out, mine.raw)
        else:
            out = all_gather(mine.raw)
        blob = b"".join(out)
        self._call("skg_dist_open_peers", C.create_string_buffer(blob, len(blob)))

    def set_overlap(self, on: bool) -> None:
        """ns3d slab, copy / NCCL exchange: all-to-all chunked per field on a
        second stream, overlapping the next field's pass (skg_dist_overlap)."""
        self._call("skg_dist_overlap", C.c_int(int(on)))

    def disable_p2p(self) -> None:
        """Back to the NCCL / device-copy exchange (skg_dist_p2p(0))."""
        self._call("skg_dist_p2p", C.c_int(0))

    def sanitize_state(self) -> None:
        """Solver::sanitize_state on the device (dealias, ns2d mean 0, ns3d
        Leray projection), as the reference applies to initial fields."""
        self._call("skg_sanitize_state")

    @property
    def last_injection(self) -> float:
        """Simulation::last_injection of the last step."""
        return load_library().skg_last_injection(self._h)

    def set_fixed_dt(self, dt: float) -> None:
        """Simulation::set_fixed_dt: a fixed dt (> 0) instead of the CFL dt."""
        if not dt > 0.0:
            raise ConfigError("fixed dt must be > 0")
        self.dt = float(dt)
        if self._cfl is not None:
            self._call("skg_set_cfl", C.c_double(0.0), C.c_double(0.1), C.c_double(-1.0))
            self._cfl = None

    def set_n_iters(self, n: int) -> None:
        """Simulation::set_n_iters: run() takes n steps (simulation.cpp:617-620)."""
        self._n_iters, self._t_end = int(n), None
        if self._cfl is not None:
            self._call("skg_set_cfl", C.c_double(self._cfl[0]), C.c_double(self._cfl[1]), C.c_double(-1.0))

    def set_t_end(self, t_end: float) -> None:
        """Simulation::set_t_end: run() stops at t_end, the last dt clamped."""
        self._t_end, self._n_iters = float(t_end), None
        if self._cfl is not None:
            self._call("skg_set_cfl", C.c_double(self._cfl[0]), C.c_double(self._cfl[1]),
                       C.c_double(self._t_end))

    def compute_dt(self) -> float:
        """Simulation::compute_dt (simulation.cpp:463-476) for the current state."""
        if self._cfl is None:
            dt = self.dt
        else:
            m = self.max_velocity(self.get_state())
            dt = self._cfl[1]
            for d in range(self.dims):
                dt = min(dt, self._cfl[0] * (self.L[d] / self.n[d]) / max(abs(m[d]), 1e-30))
        if self._t_end is not None and self._t_end >= 0.0:
            dt = min(dt, self._t_end - self.t)
        return dt

    def set_cfl(self, cfl_coef: float = 0.5, dt_max: float = 0.1, t_end: float | None = None) -> None:
        """Adaptive dt as the reference's time_stepping with fixed_dt = 0
        (compute_dt, simulation.cpp:463-476): per step
        dt = min(dt_max, cfl_coef * min_d dx_d / max|u_d|), clamped to t_end;
        computed on the device.  cfl_coef <= 0 returns to the fixed dt."""
        self._call("skg_set_cfl", C.c_double(cfl_coef), C.c_double(dt_max),
                   C.c_double(-1.0 if t_end is None else float(t_end)))
        self._cfl = (float(cfl_coef), float(dt_max)) if cfl_coef > 0 else None
        if t_end is not None:
            self._t_end, self._n_iters = float(t_end), None

    @property
    def last_dt(self) -> float:
        return load_library().skg_last_dt(self._h)

    def set_time(self, t: float) -> None:
        self._call("skg_set_time", C.c_double(t))

    def step(self, nsteps: int, dt: float | None = None) -> None:
        dt = self.dt if dt is None else float(dt)
        self._call("skg_step", C.c_double(dt), C.c_long(int(nsteps)))

    def step_async(self, nsteps: int, dt: float | None = None) -> None:
        dt = self.dt if dt is None else float(dt)
        self._call("skg_step_async", C.c_double(dt), C.c_long(int(nsteps)))

    def sync(self) -> None:
        self._call("skg_sync")

    def run(self, n_iters: int | None = None, dt: float | None = None):
        """Simulation::run (simulation.cpp:565-590).

        With n_iters: that many steps; returns the per-step means the
        reference's OutputManager records every step (output.cpp:204-214) --
        an (n_iters, 3) array of energy, enstrophy and dissipation rate.
        Without: the configured stopping rule (set_n_iters / set_t_end; t_end
        clamps the last dt like compute_dt and stops at t >= t_end - 1e-12);
        returns the RunSummary fields {"iterations", "t_final", "walltime"}
        plus "means" (the per-step series)."""
        if n_iters is not None:
            dt = self.dt if dt is None else float(dt)
            series = np.zeros((int(n_iters), 3), np.float64)
            self._call("skg_run", C.c_double(dt), C.c_long(int(n_iters)), _ptr(series))
            return series
        import time as _time
        t0 = _time.perf_counter()
        chunks = []
        if self._n_iters is not None:
            chunks.append(self.run(self._n_iters) if self._n_iters > 0 else np.zeros((0, 3)))
        elif self._t_end is not None:
            while self.t < self._t_end - 1e-12:
                if self._cfl is not None:   # the device clamps dt to t_end
                    chunks.append(self.run(1))
                    continue
                # fixed dt: the full steps, then one clamped step (t += dt in
                # double, as step_once accumulates it)
                k, t = 0, self.t
                while self._t_end - t >= self.dt and t < self._t_end - 1e-12:
                    t += self.dt
                    k += 1
                if k:
                    chunks.append(self.run(k))
                if self.t < self._t_end - 1e-12:
                    chunks.append(self.run(1, dt=self._t_end - self.t))
        else:
            raise ConfigError("run(): no stopping rule (set_n_iters or set_t_end)")
        means = np.concatenate(chunks) if chunks else np.zeros((0, 3))
        return {"iterations": len(means), "t_final": self.t,
                "walltime": _time.perf_counter() - t0, "means": means}

    def max_velocity(self, spect: np.ndarray) -> np.ndarray:
        """Solver::max_velocity_per_axis of `spect` (solvers.cpp:176-194, 341-357)."""
        s = np.ascontiguousarray(spect, dtype=np.complex128).reshape((self.nvars,) + self.spect_shape)
        out = np.zeros(self.dims, np.float64)
        self._call("skg_max_velocity", _ptr(s), _ptr(out))
        return out

    def compute_tendency(self, spect: np.ndarray) -> np.ndarray:
        s = np.ascontiguousarray(spect, dtype=np.complex128).reshape((self.nvars,) + self.spect_shape)
        out = np.empty_like(s)
        self._call("skg_tendency", _ptr(s), _ptr(out))
        return out

    # ----------------------------------------------------------- operators
    def fft_forward(self, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.shape != self.n:
            raise ShapeError(f"forward: field has shape {u.shape}, grid is {self.n}")
        out = np.empty(self.spect_shape, np.complex128)
        self._call("skg_fft_forward", _ptr(u), _ptr(out))
        return out

    def fft_inverse(self, uhat: np.ndarray) -> np.ndarray:
        uhat = np.ascontiguousarray(uhat, dtype=np.complex128)
        if uhat.shape != self.spect_shape:
            raise ShapeError(f"inverse: field has shape {uhat.shape}, grid is {self.spect_shape}")
        out = np.empty(self.n, np.float64)
        self._call("skg_fft_inverse", _ptr(uhat), _ptr(out))
        return out

    def grid(self):
        """(k_axis per axis, uint8 dealias mask) computed on the device."""
        ks = []
        mask = np.empty(self.spect_shape, np.uint8)
        for ax in range(self.dims):
            k = np.empty(self.spect_shape[ax], np.float64)
            self._call("skg_get_grid", C.c_int(ax), _ptr(k), _ptr(mask) if ax == 0 else None)
            ks.append(k)
        return ks, mask

    # -------------------------------------------------------------- queries
    @property
    def iteration(self) -> int:
        return load_library().skg_iteration(self._h)

    @property
    def t(self) -> float:
        return load_library().skg_time(self._h)

    @property
    def pruned(self) -> bool:
        return bool(load_library().skg_pruned(self._h))

    @property
    def launch_count(self) -> int:
        return load_library().skg_launch_count(self._h)

    KERNEL_CLASSES = ("x_inverse", "physical", "x_forward_rk", "y_inverse", "exchange", "y_forward")

    def set_timing(self, on: bool) -> None:
        self._call("skg_set_timing", C.c_int(1 if on else 0))

    def reset_stats(self) -> None:
        self._call("skg_reset_stats")

    def kernel_stats(self):
        """{class: (total_ms, launches, algorithmic_bytes)} since the last reset."""
        out = {}
        for i, name in enumerate(self.KERNEL_CLASSES):
            ms = C.c_double()
            nl = C.c_long()
            by = C.c_double()
            self._call("skg_kernel_stats", C.c_int(i), C.byref(ms), C.byref(nl), C.byref(by))
            out[name] = (ms.value, nl.value, by.value)
        return out

    def energy_enstrophy(self):
        e = C.c_double()
        z = C.c_double()
        self._call("skg_energy", C.byref(e), C.byref(z))
        return e.value, z.value

    def diagnostics(self):
        """(energy, enstrophy, dissipation rate) of the current state."""
        out = np.zeros(3, np.float64)
        self._call("skg_diagnostics", _ptr(out))
        return tuple(float(x) for x in out)

    def energy(self) -> float:
        return self.energy_enstrophy()[0]

    def enstrophy(self) -> float:
        return self.energy_enstrophy()[1]

    def dissipation_rate(self) -> float:
        """Simulation::dissipation_rate (simulation.cpp:608-615)."""
        return self.diagnostics()[2]

    # ---------------------------------------------------- physical fields
    def get_phys(self, key: str) -> np.ndarray:
        """Physical values of a state or computable field (bindings.cpp:123-129):
        ns2d "rot", "ux", "uy" (velocity_from_vorticity2d, grid.cpp:251-274);
        ns3d "vx", "vy", "vz", "rotz" (solvers.cpp:361-375).  Transforms on
        the GPU (FftPlan::inverse)."""
        s = self.get_state()
        if key in KEYS_STATE_PHYS[self.solver]:
            return self.fft_inverse(s[KEYS_STATE_PHYS[self.solver].index(key)])
        if key not in KEYS_COMPUTABLE[self.solver]:
            raise ConfigError(f"unknown state variable '{key}'")
        ks, _ = self.grid()
        if self.solver == "ns2d":
            kx, ky = ks[0][:, None], ks[1][None, :]
            ksq = kx * kx + ky * ky
            with np.errstate(divide="ignore", invalid="ignore"):
                psi = np.where(ksq == 0.0, 0.0, s[0] / np.where(ksq == 0.0, 1.0, ksq))
            f = 1j * ky * psi if key == "ux" else -1j * kx * psi
        else:
            kx, ky = ks[0][:, None, None], ks[1][None, :, None]
            f = 1j * kx * s[1] - 1j * ky * s[0]
        return self.fft_inverse(np.ascontiguousarray(f))

    def set_phys(self, key: str, values: np.ndarray) -> None:
        """StateSet::load_phys (state.cpp:59-69): one state variable from
        physical values (forward transform on the GPU); no sanitizing."""
        keys = KEYS_STATE_PHYS[self.solver]
        if key not in keys:
            raise ConfigError(f"unknown state variable '{key}'")
        v = np.ascontiguousarray(values, dtype=np.float64)
        if v.shape != self.n:
            raise ShapeError("array shape does not match the grid")
        s = self.get_state()
        s[keys.index(key)] = self.fft_forward(v)
        self.set_state(s)
