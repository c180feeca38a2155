#!/usr/bin/env python
"""bench.py -- RK4 step of the pseudo-spectral NS solver on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config ns2d_4096|ns2d_1024|ns3d_128|ns3d_512]

A "step" is one RK4 time step (Simulation::step_once, reference
proj/src/simulation.cpp:535-555) of the BASELINE config on synthetic seeded
input (paper_1807_01769_b200/ic.py), state resident in HBM.  Default workload:
BASELINE.json configs[3], ns3d 512^3, nu 2e-4, dt from CFL 0.5 on the IC --
the largest BASELINE config that fits one GPU in the reference layout and the
one the north-star target (>= 60% of the HBM roofline on 1 B200) names.

--gpus N: one process per GPU.  Under torchrun (WORLD_SIZE set) the ranks
come from the environment and must number N; without it, bench.py relaunches
itself through torch.distributed.run with N processes (127.0.0.1 rendezvous).

Our arm: W untimed steps, then K steps timed with CUDA events on the launch
stream (bracketed by barrier + synchronize, max over ranks), per-kernel-class
CUDA events inside the same region for the roofline, NVML clocks sampled
during it.  Every field array is larger than L2 (126 MB), so no L2 flush is
needed between steps.  `e2e` re-times the same metric through the public C
ABI with host buffers: per step skg_set_state (pinned H2D) + skg_step(1) +
skg_get_state (D2H).  `cpu_baseline` times the reference's own CPU step
(oracle/_ref: proj/src compiled unmodified + oracle/fft_shim.c) on a bounded
sample on this host.

--impl reference: the reference CPU implementation alone (rank 0), same
config/metric: one untimed warm-up step (the reference's own bench protocol,
proj/src/bench.cpp:79-82), then up to K step_once calls within a time budget.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pseudo-spectral NS RK4 ms/step & Gpts·steps/s; % of HBM/NVLink roofline"
UNIT = "Gpts*steps/s"

CONFIGS = {
    # name: solver, n, nu, dt (None = CFL 0.5 on the IC), BASELINE steps
    "ns2d_4096": ("ns2d", (4096, 4096), 1e-4, None, 20),
    "ns2d_1024": ("ns2d", (1024, 1024), 1e-4, 1e-3, 10),
    "ns3d_128": ("ns3d", (128, 128, 128), 1e-3, None, 10),
    "ns3d_512": ("ns3d", (512, 512, 512), 2e-4, None, 10),
    # one B200 in the compact (kept-modes) layout; IC generated at 128^3 and
    # spectrally embedded (all of its energy lies below |k| = 64)
    "ns3d_1024": ("ns3d", (1024, 1024, 1024), 1e-4, None, 5),
}
COARSE_IC = {"ns3d_1024": (128, 128, 128)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# 1-thread CPU row: a grid of the same solver whose single-threaded step takes
# seconds (the BASELINE configs' own single-thread steps take minutes at 512^3)
SINGLE_THREAD_CFG = {"ns2d": "ns2d_1024", "ns3d": "ns3d_128"}


def single_thread_row(solver):
    """The reference step on ONE host thread (the 1-thread
    row), on the small config of the same solver, as Gpts*steps/s."""
    from oracle import ref
    cfg = SINGLE_THREAD_CFG[solver]
    _, n, nu, dt, u0 = make_input(cfg)
    ref.set_workers(1)
    r = ref.RefSimulation(solver, n, nu, dt)
    r.set_state(u0)
    r.step(1)  # warm-up (plans)
    times = []
    while len(times) < 3 and sum(times) < 20.0:
        times.append(r.step(1))
    r.close()
    sec = sum(times) / len(times)
    return {"value": int(np.prod(n)) / sec / 1e9, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{len(times)} step_once of {cfg} on 1 thread after 1 warm-up ({sec:.3f} s/step)"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_ncu(cfg_name, key):
    """A per-launch counter of the dominant kernel (ncu), from the committed summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(cfg_name, {}).get(key)
    except Exception:
        return None


def load_traffic(cfg_name):
    """ncu dram bytes per launch of the dominant kernel."""
    return load_ncu(cfg_name, "dominant_dram_bytes_per_launch")


class ClockSampler:
    """NVML SM clock + throttle reasons, sampled from a thread during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples = []
        self.reasons = 0
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def make_input(cfg_name):
    from paper_1807_01769_b200 import ic
    solver, n, nu, dt, _ = CONFIGS[cfg_name]
    if cfg_name in COARSE_IC:
        small = COARSE_IC[cfg_name]
        v = ic.initial_state(solver, small, seed=1234)
        if dt is None:  # same max|u| (band-limited field), finer spacing
            dt = ic.cfl_dt(solver, small, v, cfl=0.5) * small[0] / n[0]
        return solver, n, nu, dt, ic.embed(v, n)
    u0 = ic.initial_state(solver, n, seed=1234)
    if dt is None:
        dt = ic.cfl_dt(solver, n, u0, cfl=0.5)
    return solver, n, nu, dt, u0


def cpu_reference_rate(solver, n, nu, dt, u0, steps, warmup, threads):
    """Reference CPU step (oracle/_ref) on this host; returns (s/step list, threads)."""
    from oracle import ref
    ref.set_workers(threads)
    r = ref.RefSimulation(solver, n, nu, dt)
    r.set_state(u0)
    t_warm = r.step(warmup) if warmup else 0.0
    # bounded sample (~10-30 s of CPU work): fewer timed steps when one step
    # is long (ns3d 512^3: ~30 s per step)
    times = []
    while len(times) < steps and sum(times) + (times[-1] if times else t_warm) <= 30.0:
        times.append(r.step(1))
    if not times:
        times.append(t_warm)  # the warm-up step itself is the sample
    # Simulation::run() per iteration: the step plus the per-step means
    # (E, Z, eps) and check_finite the reference writes every step
    # (simulation.cpp:565-590, output.cpp:204-214) -- one iteration
    t_run = r.run(1)
    r.close()
    return times, t_run


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if args.config in COARSE_IC:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"{args.config}: one reference step needs hundreds of GB of host memory "
                          "and minutes (bounded-sample rule); the ns3d_512 arm is the CPU reference"}))
        return 0
    solver, n, nu, dt, u0 = make_input(args.config)
    P = int(np.prod(n))
    threads = os.cpu_count() or 1
    from oracle import ref
    ref.set_workers(threads)
    r = ref.RefSimulation(solver, n, nu, dt)
    r.set_state(u0)
    # untimed warm-up steps (the reference's own bench protocol warms up
    # once, proj/src/bench.cpp:79-82); then up to K steps within a time budget so
    # the run stays within a few minutes (each step is a full step_once).
    # W >= 3 warm-up steps (bench rule), at most 3: each is a full step_once
    nwarm = max(1, min(args.warmup, 3))
    for _ in range(nwarm):
        t_warm = r.step(1)
    budget = args.ref_budget_s
    times = []
    while len(times) < args.steps and (sum(times) + (times[-1] if times else t_warm)) <= budget:
        times.append(r.step(1))
    if not times:
        times.append(r.step(1))
    r.close()
    sec = sum(times) / len(times)
    value = P / sec / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": len(times),
        "requested_steps": args.steps, "warmup": nwarm, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded spectral Gaussian IC, BASELINE recipe)", "impl": "reference",
        "config": {"workload": f"{args.config} RK4 step (step_once), nu={nu}, dt={dt:.6g}",
                   "solver": solver, "n": list(n), "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{len(times)} step_once calls of {args.config} after "
                                   f"{nwarm} warm-up (budget {budget:.0f} s); reference proj/src compiled "
                                   f"unmodified, FFT = oracle/fft_shim.c (batched Stockham, not FFTW)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_our_arm(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1807_01769_b200 import api

    solver, n, nu, dt, u0 = make_input(args.config)
    P = int(np.prod(n))
    S = u0.size  # complex modes over all variables
    slab = ws > 1
    p2p_used = False
    grid = None
    if args.decomp == "pencil":
        if solver != "ns3d":
            raise SystemExit("bench.py: --decomp pencil is an ns3d decomposition")
        if args.grid:
            grid = tuple(int(x) for x in args.grid.lower().split("x"))
        else:  # the paper's process grids: 2x2 at 4 ranks, 2x4 at 8
            grid = {1: (2, 2), 2: (1, 2), 4: (2, 2), 8: (2, 4), 16: (4, 4)}.get(ws, (1, ws))
    if slab:
        # slab decomposition over the ranks (strong scaling of
        # one grid), transposes as NCCL all-to-all inside libskgpu
        obj = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        if grid is not None:  # BASELINE configs[4]: py x pz pencils, two transposes per 3D FFT
            if grid[0] * grid[1] != ws:
                raise SystemExit(f"bench.py: --grid {grid[0]}x{grid[1]} needs {grid[0] * grid[1]} ranks")
            sim = api.Simulation(solver, n, nu, dt, device=local, rank=rank, nccl_id=obj[0], pencil=grid)
        else:
            sim = api.Simulation(solver, n, nu, dt, device=local, world=ws, rank=rank, nccl_id=obj[0])
        if not args.no_p2p:
            # fused exchange: the pass epilogues store into the owners'
            # receive buffers (CUDA IPC over NVLink); every rank must agree,
            # else all fall back to the NCCL all-to-all
            import torch
            ok, why = 1, ""
            try:
                sim.enable_p2p()
            except Exception as exc:  # e.g. CUDA IPC not permitted on this host
                ok, why = 0, str(exc)
            flag = torch.tensor([ok], device="cuda", dtype=torch.int32)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            p2p_used = bool(flag.item())
            if not p2p_used:
                if ok:
                    sim.disable_p2p()
                if rank == 0:
                    print(f"peer exchange unavailable ({why or 'another rank failed'}); "
                          "NCCL all-to-all", file=sys.stderr)
    elif grid is not None:
        # one GPU: all py x pz parts in this process, device copies as the
        # exchanges (the decomposition's compute and layout cost, no NVLink)
        sim = api.Simulation(solver, n, nu, dt, device=local, pencil=grid)
    else:
        compact = args.layout == "compact" or (args.layout == "auto" and args.config in COARSE_IC)
        sim = api.Simulation(solver, n, nu, dt, device=local, compact=compact)
    # a dedicated (non-default) stream: the library launches on it and the
    # CUDA events below are recorded on the same stream
    stream = torch.cuda.Stream(device=local)
    assert stream.cuda_stream != 0
    sim.set_stream(stream.cuda_stream)
    sim.set_state(u0)
    pruned = sim.pruned

    def barrier():
        if dist is not None:
            dist.barrier()

    nparts = grid[0] * grid[1] if (grid and not slab) else 1
    # ---- warm-up (also captures the per-step CUDA graph)
    sim.step(args.warmup)
    l0 = sim.launch_count
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        start.record(stream)
        sim.step_async(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    sim.sync()
    launches = sim.launch_count - l0
    ms = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- instrumented repeat: CUDA events around every launch (no graph),
    # for the per-kernel durations of the roofline
    k_inst = max(1, min(args.steps, args.instrumented_steps))
    sim.reset_stats()
    sim.set_timing(True)
    s2 = torch.cuda.Event(enable_timing=True)
    e2 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s2.record(stream)
    sim.step_async(k_inst)
    e2.record(stream)
    torch.cuda.synchronize()
    sim.sync()
    stats = sim.kernel_stats()
    sim.set_timing(False)
    inst_ms_step = s2.elapsed_time(e2) / k_inst
    ms_step = ms / args.steps
    units = P if slab else ws * P  # grid points advanced per step by the whole job
    value = units * args.steps / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel class
    peak, peak_src = load_peaks()
    dom = max((k for k in stats if k != "exchange"), key=lambda k: stats[k][0])
    dms, dn, dbytes = stats[dom]
    achieved = (dbytes / dn) / ((dms / dn) / 1e3) / 1e9 if dn else 0.0
    kernels = {k: {"ms_total": v[0], "launches": v[1],
                   "avg_us": (v[0] / v[1] * 1e3) if v[1] else None,
                   "GBps": (v[2] / (v[0] / 1e3) / 1e9) if v[0] else None,
                   "share": v[0] / sum(x[0] for x in stats.values())} for k, v in stats.items()
               if v[1]}
    step_bytes = sum(v[2] for k, v in stats.items() if k != "exchange") / k_inst
    # SURVEY.md 8(d) "fused minimal-pass" model of BASELINE's roofline:
    # 55 F (ns2d) / 181 F (ns3d) HBM bytes per RK4 step, F = 16 * modes per field
    F = 16.0 * (S // (1 if solver == "ns2d" else 3))
    fmp_bytes = (55.0 if solver == "ns2d" else 181.0) * F
    fmp = {"bytes_per_step": fmp_bytes,
           "t_roof_ms_at_8TBps": fmp_bytes / 8e12 * 1e3,
           "frac_of_8TBps": (fmp_bytes / 8e12 * 1e3) / ms_step,
           "frac_of_measured_peak": (fmp_bytes / (peak * 1e9) * 1e3) / ms_step,
           "note": "BASELINE target: >= 0.60 on 1 B200 (SURVEY 8(d) model, unpruned bytes)"}
    traffic = load_traffic(args.config)
    # FP64 roofline of the same kernel: its ncu FP64 instruction count per
    # launch over its average launch time, against the measured DFMA rate
    fp64 = None
    try:
        peak_inst = api.fp64_peak(local)
        inst = load_ncu(args.config, "dominant_fp64_inst_per_launch")
        avg_s = (dms / dn) / 1e3 if dn else None
        fp64 = {"bound": "fp64", "kernel": dom, "peak_inst_per_s": peak_inst,
                "peak_tflops": 2.0 * peak_inst / 1e12,
                "peak_source": "measured (skg_fp64_peak: DFMA-only kernel on every SM)",
                "inst_per_launch": inst,
                "inst_source": "ncu DADD+DMUL+DFMA thread instructions (profiles/ncu_summary.json)",
                "achieved_inst_per_s": (inst / avg_s) if (inst and avg_s) else None,
                "frac": (inst / avg_s / peak_inst) if (inst and avg_s) else None}
    except Exception as exc:
        fp64 = {"unavailable": str(exc)}

    # ---- e2e through the C ABI with host buffers
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if S * 16 <= (8 << 30):
        host_in = torch.empty(u0.shape, dtype=torch.complex128, pin_memory=True).numpy()
        host_in[...] = u0
        host_out = torch.empty(u0.shape, dtype=torch.complex128, pin_memory=True).numpy()
    else:  # 1024^3: 25.8 GB states, pageable (pinning two more copies per rank is not affordable)
        e2e_steps = 1
        host_in = u0
        host_out = np.empty_like(u0)
    sim.set_stream(None)  # C-ABI default stream of the context
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sim.set_state(host_in)
        sim.step(1)
        sim.get_state(out=host_out)
    t_e2e = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e_value = units * e2e_steps / t_e2e / 1e9

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if ws == 1 and rank == 0 and not args.no_cpu_baseline and args.config in COARSE_IC:
        cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
               "sample": "not run: one reference step at this size needs hundreds of GB of host "
                         "memory and minutes; see the ns3d_512 line"}
    elif ws == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            times, t_run = cpu_reference_rate(solver, n, nu, dt, u0, args.cpu_steps, 1, threads)
            sec = sum(times) / len(times)
            cpu = {"value": P / sec / 1e9, "unit": UNIT, "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(),
                   "sample": f"{len(times)} step_once of {args.config} after 1 warm-up "
                             f"({sec:.2f} s/step); reference proj/src compiled unmodified, "
                             f"FFT = oracle/fft_shim.c (batched Stockham; FFTW absent), {threads} threads",
                   "run_s_per_iter": t_run,
                   "run_note": "Simulation::run() per iteration (step + per-step E/Z/eps means + "
                               "check_finite, simulation.cpp:565-590), one iteration"}
            try:
                cpu["single_thread"] = single_thread_row(solver)
            except Exception as exc:
                cpu["single_thread"] = {"value": None, "sample": f"unavailable: {exc}"}
        except Exception as exc:  # the oracle .so may be missing on a foreign box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if slab else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded spectral Gaussian IC, BASELINE recipe)",
            "config": {
                "workload": f"{args.config}: {solver} {'x'.join(map(str, n))} RK4 step, "
                            f"nu={nu}, dt={dt:.6g} (CFL 0.5)",
                "solver": solver, "n": list(n), "global_batch": 1 if slab else ws,
                "parallelism": (
                    (f"pencil {grid[0]}x{grid[1]}" if grid else f"slab{ws}") +
                    f" ({'peer-memory exchange over NVLink' if p2p_used else 'NCCL all-to-all'})"
                    if slab else
                    f"pencil {grid[0]}x{grid[1]}, all parts on one GPU (device copies as the exchanges)"
                    if grid else "single-gpu"),
                "l2": "every field array > 126 MB L2; no flush needed",
                "dealiased_fast_path": pruned,
            },
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "algorithmic_bytes_per_launch": dbytes / dn if dn else None,
                         "step_algorithmic_GB": step_bytes / 1e9,
                         "step_frac": (step_bytes / (ms_step / 1e3) / 1e9) / peak},
            "fmp_roofline": fmp,
            "fp64_roofline": fp64,
            # one GPU with all pencil parts: the exchange class sums over the parts
            "all_to_all": ({"bytes_per_step_per_gpu": stats["exchange"][2] / k_inst / nparts,
                            "ms_per_step": stats["exchange"][0] / k_inst,
                            "t_roof_ms_at_900GBps": stats["exchange"][2] / k_inst / nparts / 900e9 * 1e3}
                           if slab or grid else None),
            "kernels": kernels,
            "instrumented": {"steps": k_inst, "ms_per_step": inst_ms_step,
                             "note": "per-kernel CUDA events (no graph); roofline.achieved uses these"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": S * 16,
                    "d2h_bytes_per_step": S * 16, "steps": e2e_steps,
                    "path": "skg_set_state(host) + skg_step(1) + skg_get_state(host)"},
            "gpu_launches": launches,
            "clocks": sampler.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="ns3d_512")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    ap.add_argument("--instrumented-steps", type=int, default=20)
    ap.add_argument("--no-p2p", action="store_true",
                    help="slab under torchrun: NCCL all-to-all copies instead of the peer-memory "
                         "exchange (CUDA IPC stores from the pass epilogues, the default)")
    ap.add_argument("--decomp", choices=["slab", "pencil"], default="slab",
                    help="multi-GPU decomposition of ns3d: slab (one all-to-all per 3D FFT, the "
                         "default: fewer NVLink bytes up to 8 GPUs) or the py x pz pencils BASELINE "
                         "configs[4] names (two all-to-alls per 3D FFT)")
    ap.add_argument("--grid", default="", help="pencil process grid PYxPZ (default 2x2 / 2x4 at 4 / 8 ranks)")
    ap.add_argument("--layout", choices=["auto", "full", "compact"], default="auto",
                    help="ns3d one-GPU layout (auto: compact where the full layout does not fit)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: relaunch through torchrun (127.0.0.1 rendezvous)
        import socket
        import subprocess
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
        return subprocess.call(cmd)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
