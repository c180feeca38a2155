#!/bin/bash
# one kernel, full set with source correlation; SASS source page + raw page as CSV
cfg=$1; kre=$2; tag=$3; skip=${4:-8}
cmd="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --instrumented-steps 1"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
    -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/src_$tag.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
rm -f gpurun_out/prof_$tag.ncu-rep
echo done
