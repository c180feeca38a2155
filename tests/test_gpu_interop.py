"""Output-format interoperability with the reference's own snapshot and
records path:

* a snapshot the REFERENCE's OutputManager wrote (output.cpp:259-266,
  snapshot.cpp:65-100) loads on the GPU and continues in step with the
  reference;
* a snapshot the GPU wrote (Simulation.save_fld) restarts the REFERENCE
  through its own load_state_phys_file (simulation.cpp:705-732: digest check
  against params.txt, snapshot_filename lookup by time) and continues in step
  with the GPU;
* the device shell spectra (skg_spectra) equal the records the reference's
  OutputManager writes with files enabled: spectra.ndrec E(k) density and
  spect_energy_budg.ndrec T(k), D(k) (output.cpp:223-257).
"""
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import spectral_np as O
from paper_1807_01769_b200 import api, ic

pytestmark = pytest.mark.gpu
PARITY = 1e-10

CASES = [("ns2d", (64, 64), 1e-3, 21), ("ns3d", (32, 32, 32), 1e-3, 22)]


def read_ndrec(path):
    """Records of a .ndrec stream (records.hpp: one `key=value` record per
    line; lists as [a,b,...]; doubles printed with 17 digits)."""
    out = []
    for line in Path(path).read_text().splitlines():
        if not line.strip():
            continue
        rec = {}
        for key, val in re.findall(r"(\w+)=(\[[^\]]*\]|\S+)", line):
            if val.startswith("["):
                body = val[1:-1]
                rec[key] = np.array([float(x) for x in body.split(",")] if body else [], np.float64)
            else:
                try:
                    rec[key] = float(val)
                except ValueError:
                    rec[key] = val.strip('"')
        out.append(rec)
    return out


def fld_header(path):
    with open(path, "rb") as f:
        assert f.readline().rstrip(b"\n") == b"spectralkit-fld 1"
        return dict(f.readline().decode().rstrip("\n").split("=", 1) for _ in range(4))


def snapshot_filename(t):
    return f"state_phys_t{t:.6f}.fld"  # snapshot.hpp:25-26


def reference_run(ref_lib, tmp_path, solver, n, nu, seed, steps):
    u0 = ic.initial_state(solver, n, seed)
    dt = ic.cfl_dt(solver, n, u0)
    r = ref_lib.RefSimulation(solver, n, nu, dt, files=(tmp_path, 2 * dt))
    r.set_state(u0)
    r.run(steps)
    return r, u0, dt, Path(r.output_dir)


@pytest.mark.parametrize("solver,n,nu,seed", CASES, ids=[c[0] for c in CASES])
def test_reference_snapshot_continues_on_gpu(ref_lib, tmp_path, solver, n, nu, seed):
    r, _, dt, run_dir = reference_run(ref_lib, tmp_path, solver, n, nu, seed, 4)
    snaps = sorted((run_dir / "snapshots").glob("*.fld"), key=lambda p: float(fld_header(p)["time"]))
    assert len(snaps) >= 2
    g = api.Simulation(solver, n, nu, dt)
    hdr = g.load_fld(snaps[-1])
    assert hdr["time"] == r.t and g.t == r.t
    # physical snapshot -> spectral state on the device (FftPlan::forward)
    assert max(O.rel_l2(a, b) for a, b in zip(g.get_state(), r.get_state())) < 1e-13
    r.step(5)
    g.step(5)
    assert max(O.rel_l2(a, b) for a, b in zip(g.get_state(), r.get_state())) < PARITY
    assert abs(g.t - r.t) < 1e-15 * r.t
    r.close()
    g.close()


@pytest.mark.parametrize("solver,n,nu,seed", CASES, ids=[c[0] for c in CASES])
def test_gpu_snapshot_restarts_reference(ref_lib, tmp_path, solver, n, nu, seed):
    # the reference's run directory (params.txt, its own t = 0 snapshot)
    r, u0, dt, run_dir = reference_run(ref_lib, tmp_path, solver, n, nu, seed, 1)
    r.close()
    digest = fld_header(run_dir / "snapshots" / snapshot_filename(0.0))["digest"]
    g = api.Simulation(solver, n, nu, dt)
    g.set_state(u0)
    g.step(3)
    path = run_dir / "snapshots" / snapshot_filename(g.t)
    g.save_fld(path, digest=digest)
    # load_state_phys_file: params.txt + the snapshot nearest t, digest checked
    rr = ref_lib.RefSimulation.restart(run_dir, solver, n, time=g.t)
    assert rr.t == g.t
    assert max(O.rel_l2(a, b) for a, b in zip(rr.get_state(), g.get_state())) < 1e-13
    rr.step(4)
    g.step(4)
    assert max(O.rel_l2(a, b) for a, b in zip(g.get_state(), rr.get_state())) < PARITY
    rr.close()
    g.close()


def test_gpu_snapshot_with_wrong_digest_is_rejected(ref_lib, tmp_path):
    """The reference's restart refuses a snapshot of a different run setup
    (simulation.cpp:719-723); a GPU-written file carries the digest it is given."""
    solver, n, nu, seed = CASES[0]
    r, u0, dt, run_dir = reference_run(ref_lib, tmp_path, solver, n, nu, seed, 1)
    r.close()
    g = api.Simulation(solver, n, nu, dt)
    g.set_state(u0)
    g.step(2)
    g.save_fld(run_dir / "snapshots" / snapshot_filename(g.t), digest="0123456789abcdef")
    with pytest.raises(ref_lib.RefError, match="digest"):
        ref_lib.RefSimulation.restart(run_dir, solver, n, time=g.t)
    g.close()


@pytest.mark.parametrize("solver,n,nu,seed", CASES, ids=[c[0] for c in CASES])
def test_spectra_match_output_manager_records(ref_lib, tmp_path, solver, n, nu, seed):
    r, _, dt, run_dir = reference_run(ref_lib, tmp_path, solver, n, nu, seed, 4)
    t_end = r.t
    spectra = [x for x in read_ndrec(run_dir / "spectra.ndrec") if x["t"] == t_end]
    budget = [x for x in read_ndrec(run_dir / "spect_energy_budg.ndrec") if x["t"] == t_end]
    assert len(spectra) == 1 and len(budget) == 1
    g = api.Simulation(solver, n, nu, dt)
    g.set_state(r.get_state())
    sp = g.spectra()
    assert np.array_equal(sp["k"], spectra[0]["k"])
    for key, rec in (("E", spectra[0]), ("T", budget[0]), ("D", budget[0])):
        ref_v = rec[key]
        assert sp[key].shape == ref_v.shape
        assert np.abs(sp[key] - ref_v).max() <= 1e-11 * np.abs(ref_v).max(), key
    r.close()
    g.close()
