# chain kernel validation + A/B timing, dist/interop tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_interop.py tests/test_gpu_dist.py tests/test_gpu_ns3d.py -x -q --durations=15 > gpurun_out/pytest3.log 2>&1; echo rc=$? >> gpurun_out/pytest3.log
for v in 1 0; do
  SKG_CHAIN=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3_chain$v.log 2>&1
  SKG_CHAIN=$v timeout 600 python bench.py --config ns3d_128 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench3_128_chain$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "configs3" > gpurun_out/pytest3_full.log 2>&1; echo rc=$? >> gpurun_out/pytest3_full.log
