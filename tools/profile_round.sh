#!/bin/bash
# Round profile evidence: per config, a plain run, then the ncu launch list
# (gpu__time_duration of every launch) and one --set full capture of the
# stage kernels.  Outputs into gpurun_out/ (summarised by tools/ncu_summary.py).
tag=${1:-r02}
run() {  # cfg kernel_regex count
  cfg=$1; kre=$2; cnt=$3
  cmd="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --instrumented-steps 1"
  $cmd > gpurun_out/plain_${tag}_$cfg.log 2>&1 || { echo "plain run failed: $cfg"; return 1; }
  ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 60 --csv \
      --log-file gpurun_out/launches_${tag}_$cfg.csv $cmd > /dev/null 2>&1
  echo "launches $cfg rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 8 -c $cnt \
      -o gpurun_out/prof_${tag}_$cfg $cmd > gpurun_out/ncu_${tag}_$cfg.log 2>&1
  echo "full $cfg rc=$?"
}
run ns2d_4096 'k3b_phys|k4b_xfwd' 2
run ns3d_512 'k1_3d|k2s_3d|k3_3d|k2f_3d|k4_3d' 5
# keep what comes back under gpurun's 64 MiB: raw counter pages as CSV, the
# reports themselves only if small
for r in gpurun_out/prof_${tag}_*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}_details.csv" 2>/dev/null
  sz=$(stat -c %s "$r"); echo "$r $sz bytes"
  [ "$sz" -gt 20000000 ] && rm -f "$r"
done
ls -la gpurun_out/ | head -30
