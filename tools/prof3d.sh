#!/bin/bash
# ns3d 512^3: plain run, then launch list + one full capture of each stage kernel
cmd="python bench.py --config ns3d_512 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --instrumented-steps 1"
$cmd > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k[1234]f?_3d' -s 20 -c 5 \
    -o gpurun_out/prof_r02_ns3d512 $cmd > gpurun_out/ncu3.log 2>&1
echo rc=$?
