# last check of the committed tree: smoke, core parity tests, default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke25.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke25.log
timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_ns3d.py tests/test_gpu_integration.py tests/test_gpu_interop.py tests/test_gpu_api_mirror.py -x -q -m gpu > gpurun_out/pytest25.log 2>&1; echo rc=$? >> gpurun_out/pytest25.log
timeout 900 python bench.py > gpurun_out/bench25_default.log 2>&1; echo rc=$? >> gpurun_out/bench25_default.log
