# A/B: ns3d z-pass groups, ns2d small-grid staging
mkdir -p gpurun_out
out=gpurun_out/ab_mix.log; : > $out
for v in base zg2 zg1; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 256 512 >> $out 2>&1
done
for v in base xstg base xstg; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d 256 512 1024 2048 4096 >> $out 2>&1
done
SKG_LIB_VARIANT=xstg timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_dist.py tests/test_gpu_api_mirror.py -x -q > gpurun_out/ab_mix_pytest.log 2>&1; echo "xstg rc=$?" >> gpurun_out/ab_mix_pytest.log
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_cfl.py tests/test_gpu_guard.py -x -q >> gpurun_out/ab_mix_pytest.log 2>&1; echo "base rc=$?" >> gpurun_out/ab_mix_pytest.log
