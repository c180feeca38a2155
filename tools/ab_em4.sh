mkdir -p gpurun_out
out=gpurun_out/ab_em4.log; : > $out
for v in base em4x em4xy em4x128 em4xy128 base; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d 256 512 1024 2048 >> $out 2>&1
done
for v in em4xy em4x; do
SKG_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_dist.py tests/test_gpu_api_mirror.py tests/test_gpu_cfl.py -x -q > gpurun_out/ab_em4_pytest_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/ab_em4_pytest_$v.log
done
