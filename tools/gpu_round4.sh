# chain variants A/B at 512^3 + chain test
mkdir -p gpurun_out
SKG_CHAIN=0 STEPS=50 bash tools/var_sweep.sh ns3d_512 1 base > gpurun_out/sweep4.log 2>&1
STEPS=50 bash tools/var_sweep.sh ns3d_512 1 c1 c2 c3 c4 c5 >> gpurun_out/sweep4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_guard.py -x -q > gpurun_out/pytest4.log 2>&1; echo rc=$? >> gpurun_out/pytest4.log
