# checkpoint: bench lines (default ns3d_512 + ns2d configs) and r07 profiles of the changed kernels
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench7_512.log 2>&1; echo rc=$? >> gpurun_out/bench7_512.log
for c in ns2d_1024 ns2d_4096 ns3d_128; do
timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench7_$c.log 2>&1; echo rc=$? >> gpurun_out/bench7_$c.log
done
timeout 2400 bash tools/profile_round.sh r07 ns3d_512 ns2d_1024 ns3d_128 > gpurun_out/prof7.log 2>&1
