mkdir -p gpurun_out
out=gpurun_out/ab_ybulk.log; : > $out
for v in base ybulk base ybulk; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 128 256 512 >> $out 2>&1
done
SKG_LIB_VARIANT=ybulk timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_dist.py -x -q > gpurun_out/ab_ybulk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_ybulk_pytest.log
