free -g | head -2; nproc
python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config ns3d_1024 --steps 3 --warmup 3 --e2e-steps 1 --instrumented-steps 3 > gpurun_out/b1024.log 2>&1; echo rc=$?; tail -c 3000 gpurun_out/b1024.log
