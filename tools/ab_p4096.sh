mkdir -p gpurun_out
out=gpurun_out/ab_p4096.log; : > $out
for v in base p4096 base p4096; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d 4096 >> $out 2>&1
done
timeout 300 python tools/time_steps.py ns3d 512 >> $out 2>&1
timeout 1200 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_fullsize.py tests/test_gpu_cfl.py tests/test_gpu_guard.py -x -q > gpurun_out/ab_p4096_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_p4096_pytest.log
