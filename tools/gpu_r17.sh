# A/B of the hoisted-address changes per kernel (variants built by tools/build_variant.sh)
mkdir -p gpurun_out
out=gpurun_out/ab_r17.log; : > $out
for rep in 1 2; do
for v in base yfld0; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  SKG_LIB_VARIANT=$var timeout 600 python bench.py --config ns3d_512 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --instrumented-steps 3 > gpurun_out/bench17_$v.log 2>&1
  python - >> $out <<PY
import json
l=[x for x in open("gpurun_out/bench17_$v.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("$v", "ms/step", round(d["ms_per_step"],3), {k:round(x["avg_us"]) for k,x in d["kernels"].items()})
else:
    print("$v", open("gpurun_out/bench17_$v.log").read()[-600:])
PY
done; done
timeout 300 python tools/time_steps.py ns3d 64 128 256 512 >> $out 2>&1
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_pencil.py tests/test_gpu_dist.py -x -q -m gpu > gpurun_out/pytest17.log 2>&1; echo rc=$? >> gpurun_out/pytest17.log
