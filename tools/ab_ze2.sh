mkdir -p gpurun_out
out=gpurun_out/ab_ze3.log; : > $out
for v in ct1024all ct1024x ct1024y; do
  echo "== $v" >> $out
  SKG_LIB_VARIANT=$v timeout 900 python bench.py --config ns3d_1024 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --instrumented-steps 2 > gpurun_out/ab_ze_1024_$v.log 2>&1
  python - >> $out <<PY
import json
l=[x for x in open("gpurun_out/ab_ze_1024_$v.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("ms/step", d["ms_per_step"], {k:round(x["avg_us"]) for k,x in d["kernels"].items()})
else:
    print(open("gpurun_out/ab_ze_1024_$v.log").read()[-800:])
PY
done
