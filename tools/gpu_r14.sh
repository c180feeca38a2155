# x-forward scratch slots (k4_3d): correctness, then A/B against the in-place write-back (SKG_NO_XSCR=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ns3d.py tests/test_gpu_guard.py tests/test_gpu_pencil.py tests/test_gpu_dist.py tests/test_gpu_cfl.py tests/test_gpu_forcing.py -x -q -m gpu > gpurun_out/pytest14.log 2>&1; echo rc=$? >> gpurun_out/pytest14.log
out=gpurun_out/ab_xscr.log; : > $out
for rep in 1 2; do
for v in 1 0; do
  echo "== SKG_NO_XSCR=$v" >> $out
  if [ $v = 1 ]; then export SKG_NO_XSCR=1; else unset SKG_NO_XSCR; fi
  timeout 300 python tools/time_steps.py ns3d 64 128 256 512 >> $out 2>&1
done; done
for v in 1 0; do
  if [ $v = 1 ]; then export SKG_NO_XSCR=1; else unset SKG_NO_XSCR; fi
  timeout 600 python bench.py --config ns3d_512 --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench14_512_noxscr$v.log 2>&1
  timeout 900 python bench.py --config ns3d_1024 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --instrumented-steps 2 > gpurun_out/bench14_1024_noxscr$v.log 2>&1
done
unset SKG_NO_XSCR
python - >> $out <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench14_*.log")):
    l=[x for x in open(f) if x.startswith("{")]
    if l:
        d=json.loads(l[-1]); print(f, "ms/step", round(d["ms_per_step"],3), {k:round(x["avg_us"]) for k,x in d["kernels"].items()})
    else:
        print(f, open(f).read()[-600:])
PY
