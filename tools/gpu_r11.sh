mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pencil.py tests/test_gpu_dist.py -x -q -m gpu --durations=5 > gpurun_out/pytest11.log 2>&1; echo rc=$? >> gpurun_out/pytest11.log
for g in 2x4; do
timeout 600 python bench.py --config ns3d_512 --decomp pencil --grid $g --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench11_pencil_$g.log 2>&1; echo rc=$? >> gpurun_out/bench11_pencil_$g.log
done
timeout 600 python bench.py --config ns3d_512 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/bench11_512.log 2>&1; echo rc=$? >> gpurun_out/bench11_512.log
timeout 600 python bench.py --config ns3d_128 --steps 200 --warmup 3 --no-cpu-baseline > gpurun_out/bench11_128.log 2>&1; echo rc=$? >> gpurun_out/bench11_128.log
