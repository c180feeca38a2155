#!/bin/bash
# usage: prof_k.sh config kernel_regex tag [skip] — plain run, then one full ncu capture
cfg=$1; kre=$2; tag=$3; skip=${4:-20}
cmd="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --instrumented-steps 1"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
    -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
echo rc=$?
