# z pass with 16 elements per thread at 128^3 and 1024^3 (A/B against the 8-element lines)
mkdir -p gpurun_out
out=gpurun_out/ab_ze.log; : > $out
for v in base z128e16g16 z128e16g28 base z128e16g16 z128e16g28; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 300 python tools/time_steps.py ns3d 128 >> $out 2>&1
done
for v in base z1024e16g2 z1024e16g4; do
  var=$([ "$v" = base ] && echo "" || echo $v)
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$var timeout 900 python bench.py --config ns3d_1024 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --instrumented-steps 2 > gpurun_out/ab_ze_1024_$v.log 2>&1
  python - >> $out <<PY
import json
l=[x for x in open("gpurun_out/ab_ze_1024_$v.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("ms/step", d["ms_per_step"], {k:round(x["avg_us"]) for k,x in d["kernels"].items()})
else:
    print(open("gpurun_out/ab_ze_1024_$v.log").read()[-800:])
PY
done
