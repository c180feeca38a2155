# round-2 final numbers: every bench config on the committed kernels, the reference arm, r13 profiles of 1024^3 and 128^3
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench13_default.log 2>&1; echo rc=$? >> gpurun_out/bench13_default.log
for c in ns2d_1024 ns2d_4096 ns3d_128; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench13_$c.log 2>&1; echo rc=$? >> gpurun_out/bench13_$c.log
done
timeout 900 python bench.py --config ns3d_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench13_ns3d_1024.log 2>&1; echo rc=$? >> gpurun_out/bench13_ns3d_1024.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench13_ref.log 2>&1; echo rc=$? >> gpurun_out/bench13_ref.log
timeout 2000 bash tools/profile_round.sh r13 ns3d_1024 ns3d_128 > gpurun_out/prof13.log 2>&1
