# strided passes: hoisted address arithmetic (base pointer + stride per thread); A/B vs r14 numbers
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_guard.py tests/test_gpu_pencil.py tests/test_gpu_dist.py tests/test_gpu_cfl.py -x -q -m gpu > gpurun_out/pytest15.log 2>&1; echo rc=$? >> gpurun_out/pytest15.log
out=gpurun_out/ab_r15.log; : > $out
for rep in 1 2; do
  timeout 300 python tools/time_steps.py ns3d 64 128 256 512 >> $out 2>&1
done
timeout 600 python bench.py --config ns3d_512 --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench15_512.log 2>&1
timeout 600 python bench.py --config ns3d_128 --steps 200 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench15_128.log 2>&1
timeout 900 python bench.py --config ns3d_1024 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --instrumented-steps 2 > gpurun_out/bench15_1024.log 2>&1
python - >> $out <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench15_*.log")):
    l=[x for x in open(f) if x.startswith("{")]
    if l:
        d=json.loads(l[-1]); print(f, "ms/step", round(d["ms_per_step"],3), {k:round(x["avg_us"]) for k,x in d["kernels"].items()})
    else:
        print(f, open(f).read()[-600:])
PY
