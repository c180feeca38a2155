# New dist / interop tests, then compute-sanitizer over tools/sanitize_case.py.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_interop.py tests/test_gpu_dist.py -x -q --durations=15 > gpurun_out/pytest2.log 2>&1; echo rc=$? >> gpurun_out/pytest2.log
timeout 1500 bash tools/sanitize.sh
