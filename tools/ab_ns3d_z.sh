# A/B of ns3d z-pass variants: ms/step at 128/256/512 + parity subset on the first variant
mkdir -p gpurun_out
out=gpurun_out/ab_z.log; : > $out
for v in ${VARIANTS:-base zsG3 zsG3r zG3 zsG4}; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d ${SIZES:-128 256 512} >> $out 2>&1
done
for v in ${TESTV:-zsG3}; do
  SKG_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_dist.py -x -q >> gpurun_out/ab_z_pytest.log 2>&1; echo "$v rc=$?" >> gpurun_out/ab_z_pytest.log
done
