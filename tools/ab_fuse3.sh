mkdir -p gpurun_out
out=gpurun_out/ab_fuse3.log; : > $out
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_ns2d.py tests/test_gpu_cfl.py tests/test_gpu_forcing.py tests/test_gpu_api_mirror.py tests/test_gpu_dist.py -x -q > gpurun_out/ab_fuse3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_fuse3_pytest.log
for v in base nofuse3 base nofuse3; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 64 128 256 512 >> $out 2>&1
done
timeout 300 python tools/time_steps.py ns2d 256 512 1024 >> $out 2>&1
