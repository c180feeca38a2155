mkdir -p gpurun_out
out=gpurun_out/ab_p8.log; : > $out
for v in base p8r80 p8r128 p8r80m512 base p8r80; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d 256 512 1024 2048 >> $out 2>&1
done
SKG_LIB_VARIANT=p8r80 timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_dist.py tests/test_gpu_api_mirror.py tests/test_gpu_cfl.py tests/test_gpu_forcing.py -x -q > gpurun_out/ab_p8_pytest.log 2>&1; echo "p8r80 rc=$?" >> gpurun_out/ab_p8_pytest.log
timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_fft*.py tests/test_gpu_cfl.py -x -q >> gpurun_out/ab_p8_pytest.log 2>&1; echo "base rc=$?" >> gpurun_out/ab_p8_pytest.log
