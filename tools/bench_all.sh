#!/bin/bash
# Full GPU test suite, then every bench config (and the reference arm of the default one).
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for cfg in ns2d_4096 ns2d_1024 ns3d_128 ns3d_512 ns3d_1024; do
  extra=""
  [ "$cfg" = "ns3d_1024" ] && extra="--steps 5 --warmup 3"
  timeout 900 python bench.py --config $cfg $extra > gpurun_out/bench_$cfg.log 2>&1
  echo "$cfg rc=$?"; tail -1 gpurun_out/bench_$cfg.log | cut -c1-300
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_ns2d_4096.log 2>&1
echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_ns2d_4096.log | cut -c1-400
