mkdir -p gpurun_out
timeout 900 python bench.py --config ns3d_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench12_1024.log 2>&1; echo rc=$? >> gpurun_out/bench12_1024.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "1024 or round_trip" --durations=5 > gpurun_out/pytest12.log 2>&1; echo rc=$? >> gpurun_out/pytest12.log
timeout 600 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_guard.py -x -q -m gpu > gpurun_out/pytest12b.log 2>&1; echo rc=$? >> gpurun_out/pytest12b.log
