"""Summarise ncu reports/launch lists into profiles/ (committed evidence).

    python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches_r01.csv \
        --report gpurun_out/prof_r01_ns2d.ncu-rep --config ns2d_4096

Writes profiles/<tag>_<config>_launches.csv (per-kernel share of the step from
the serialized cold-cache launch list), profiles/<tag>_<config>_ncu.md (key
counters of the full capture) and merges the dominant kernel's DRAM bytes per
launch into profiles/ncu_summary.json (read by bench.py as roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
]


# setup / measurement kernels of a bench run that are not part of the RK step
NOT_STEP = ("fp64_probe", "count_masked", "transpose_c", "grid_dump")


def short(name: str) -> str:
    m = re.search(r"(k\w+?)<([^>]*)>", name)
    return f"{m.group(1)}<{m.group(2)}>" if m else name.split("(")[0][-40:]


def launches(path: Path, out: Path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    i_n, i_v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = short(r[i_n])
        if any(x in k for x in NOT_STEP):
            continue
        agg.setdefault(k, []).append(float(r[i_v].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    with open(out, "w") as f:
        f.write("kernel,launches,avg_us,total_us,share\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k},{len(v)},{sum(v)/len(v)/1e3:.2f},{sum(v)/1e3:.1f},{sum(v)/tot:.3f}\n")
    return agg


def report(rep: Path, out: Path):
    if rep.suffix == ".csv":  # `ncu -i … --page raw --csv` captured on the GPU box
        txt = rep.read_text()
    else:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    # drop ncu's ==PROF== / ==WARNING== banner lines of --log-file captures
    rows = [r for r in csv.reader(l for l in txt.splitlines() if not l.startswith("=="))]
    if "Metric Name" in rows[0]:  # `ncu --metrics ... --csv` launch-per-metric rows: pivot
        h = rows[0]
        i_id, i_k, i_m, i_u, i_v = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name",
                                                          "Metric Unit", "Metric Value"))
        launch = collections.OrderedDict()
        unit = {}
        for r in rows[1:]:
            if len(r) <= i_v:
                continue
            launch.setdefault(r[i_id], {"Kernel Name": r[i_k]})[r[i_m]] = r[i_v]
            unit[r[i_m]] = r[i_u]
        names = ["Kernel Name"] + sorted(unit)
        rows = [names, [""] + [unit[n] for n in names[1:]]] + [
            [d.get(n, "") for n in names] for d in launch.values()]
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    kern = []
    fp64_ops = [f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
                for op in ("dadd", "dmul", "dfma")]
    for r in rows[2:]:
        d = {"kernel": short(r[idx["Kernel Name"]])}
        if all(m in idx for m in fp64_ops) and "sm__cycles_elapsed.avg" in idx:
            # FP64 thread-instructions of the launch (DADD + DMUL + DFMA)
            cyc = float(r[idx["sm__cycles_elapsed.avg"]].replace(",", ""))
            d["fp64_inst"] = cyc * sum(float(r[idx[m]].replace(",", "")) for m in fp64_ops)
        for m, lab in METRICS:
            if m in idx:
                d[lab] = (r[idx[m]], units[idx[m]])
        kern.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {rep.name}\n\n")
        labs = [lab for _, lab in METRICS]
        f.write("| kernel | " + " | ".join(labs) + " |\n|" + "---|" * (len(labs) + 1) + "\n")
        for d in kern:
            f.write(f"| {d['kernel']} | " + " | ".join(
                f"{d[l][0]} {d[l][1]}" if l in d else "" for l in labs) + " |\n")
    return kern


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--report", help=".ncu-rep, or its raw page as CSV")
    ap.add_argument("--dominant", help="kernel name prefix of the roofline kernel")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    if a.launches:
        launches(Path(a.launches), PROF / f"{a.tag}_{a.config}_launches.csv")
    if a.report:
        kern = report(Path(a.report), PROF / f"{a.tag}_{a.config}_ncu.md")
        summ = PROF / "ncu_summary.json"
        d = json.loads(summ.read_text()) if summ.exists() else {}
        per = {}
        for k in kern:
            if "DRAM read" in k and "DRAM write" in k:
                per.setdefault(k["kernel"], []).append(to_bytes(*k["DRAM read"]) + to_bytes(*k["DRAM write"]))
        fp = {}
        for k in kern:
            if "fp64_inst" in k:
                fp.setdefault(k["kernel"], []).append(k["fp64_inst"])
        entry = {"tag": a.tag, "kernels_dram_bytes_per_launch":
                 {k: sum(v) / len(v) for k, v in per.items()},
                 "kernels_fp64_inst_per_launch": {k: sum(v) / len(v) for k, v in fp.items()}}
        if a.dominant:
            for k, v in per.items():
                if k.startswith(a.dominant):
                    entry["dominant"] = k
                    entry["dominant_dram_bytes_per_launch"] = sum(v) / len(v)
                    if k in fp:
                        entry["dominant_fp64_inst_per_launch"] = sum(fp[k]) / len(fp[k])
        d[a.config] = entry
        summ.write_text(json.dumps(d, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
