# staged z pass: first bulk copy issued before the divergence-flag check (A/B against r22: z pass 2130-2158 us)
mkdir -p gpurun_out
out=gpurun_out/ab_r28.log; : > $out
for rep in 1 2; do
  timeout 600 python bench.py --config ns3d_512 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --instrumented-steps 3 > gpurun_out/bench28_$rep.log 2>&1
  python - >> $out <<PY
import json
l=[x for x in open("gpurun_out/bench28_$rep.log") if x.startswith("{")]
d=json.loads(l[-1]); print("new", "ms/step", round(d["ms_per_step"],3), {k:round(x["avg_us"]) for k,x in d["kernels"].items()})
PY
  timeout 300 python tools/time_steps.py ns3d 256 512 >> $out 2>&1
done
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_cfl.py tests/test_gpu_pencil.py tests/test_gpu_dist.py -x -q -m gpu > gpurun_out/pytest28.log 2>&1; echo rc=$? >> gpurun_out/pytest28.log
