# A/B of ns2d small-grid variants: parity subset + ms/step at 256..2048 (+4096)
mkdir -p gpurun_out
out=gpurun_out/ab_small.log; : > $out
for v in ${VARIANTS:-base pair512 pair1024 pair2048 pair1024y16}; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d ${SIZES:-256 512 1024 2048} >> $out 2>&1
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns2d ${SIZES:-256 512 1024 2048} >> $out 2>&1
done
for v in ${TESTV:-pair2048}; do
  SKG_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_ns2d.py tests/test_gpu_dist.py tests/test_gpu_cfl.py -x -q -k "ns2d or slab or cfl" >> gpurun_out/ab_small_pytest.log 2>&1; echo "$v rc=$?" >> gpurun_out/ab_small_pytest.log
done
