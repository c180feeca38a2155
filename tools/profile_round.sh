#!/bin/bash
# Round profile evidence: per config, a plain run, then the ncu launch list
# (gpu__time_duration of every launch) and one --set full capture of the
# stage kernels (1024^3: DRAM bytes, duration and FP64 counts only -- a full
# capture replays each kernel ~40 times over ~140 GB of device state).
# Outputs into gpurun_out/ (summarised by tools/ncu_summary.py).
# usage: tools/profile_round.sh tag [config ...]
tag=${1:-r06}; shift
cfgs=${@:-ns2d_1024 ns2d_4096 ns3d_128 ns3d_512 ns3d_1024}
FP64="smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed,sm__cycles_elapsed.avg"
run() {  # cfg kernel_regex count
  cfg=$1; kre=$2; cnt=$3
  cmd="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --instrumented-steps 1"
  $cmd > gpurun_out/plain_${tag}_$cfg.log 2>&1 || { echo "plain run failed: $cfg"; return 1; }
  ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 60 --csv \
      --log-file gpurun_out/launches_${tag}_$cfg.csv $cmd > /dev/null 2>&1
  echo "launches $cfg rc=$?"
  if [ "$cfg" = ns3d_1024 ]; then
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,$FP64 \
        --clock-control none -k regex:"$kre" -s 8 -c $cnt --csv \
        --log-file gpurun_out/prof_${tag}_${cfg}_metrics.csv $cmd > gpurun_out/ncu_${tag}_$cfg.log 2>&1
    echo "metrics $cfg rc=$?"
  else
    ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 8 -c $cnt \
        -o gpurun_out/prof_${tag}_$cfg $cmd > gpurun_out/ncu_${tag}_$cfg.log 2>&1
    echo "full $cfg rc=$?"
  fi
}
for cfg in $cfgs; do
  case $cfg in
    ns2d_*) run $cfg 'k3b_phys|k4b_xfwd|k4p_xfwd' 2 ;;
    ns3d_*) run $cfg 'k1_3d|k2s_3d|k3_3d|k2f_3d|k4_3d' 5 ;;
  esac
done
# keep what comes back under gpurun's 64 MiB: raw counter pages as CSV, the
# reports themselves only if small
for r in gpurun_out/prof_${tag}_*.ncu-rep; do
  [ -e "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  sz=$(stat -c %s "$r"); echo "$r $sz bytes"
  [ "$sz" -gt 8000000 ] && rm -f "$r"
done
ls -la gpurun_out/ | head -40
