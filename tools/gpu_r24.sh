# ns2d fused x-forward: hoisted receive/send addresses (variant hoist2) vs per-element index arithmetic
mkdir -p gpurun_out
out=gpurun_out/ab_r24.log; : > $out
for rep in 1 2 3; do
for v in base hoist2; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d 512 1024 2048 4096 >> $out 2>&1
done; done
SKG_LIB_VARIANT=hoist2 timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_dist.py tests/test_gpu_cfl.py tests/test_gpu_forcing.py -x -q -m gpu > gpurun_out/pytest24.log 2>&1; echo rc=$? >> gpurun_out/pytest24.log
