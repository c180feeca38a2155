tag=r05; cfg=ns3d_512
cmd="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --instrumented-steps 1"
$cmd > gpurun_out/plain_${tag}_$cfg.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 80 --csv --log-file gpurun_out/launches_${tag}_$cfg.csv $cmd > /dev/null 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k1_3d|k2s_3d|k3_3d|k2f_3d|k4_3d" -s 10 -c 8 -o gpurun_out/prof_${tag}_$cfg $cmd > gpurun_out/ncu_${tag}_$cfg.log 2>&1; echo full rc=$?
ncu -i gpurun_out/prof_${tag}_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_${cfg}_raw.csv 2>/dev/null
rm -f gpurun_out/prof_${tag}_$cfg.ncu-rep
