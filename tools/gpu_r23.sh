# modified tests (scratch slots forced on/off, guard zones with slots on); streaming-store variant at 128^3 / 64^3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_guard.py -x -q -m gpu > gpurun_out/pytest23.log 2>&1; echo rc=$? >> gpurun_out/pytest23.log
out=gpurun_out/ab_r23.log; : > $out
for rep in 1 2 3; do
for v in base stcs; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 64 128 256 >> $out 2>&1
done; done
