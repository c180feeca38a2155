#!/bin/bash
# usage: opt_sweep.sh config opts...
cfg=$1; shift
extra=${EXTRA:-}
for o in "$@"; do
  SKG_OPT=$o timeout 300 python bench.py --config $cfg --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 2 $extra > gpurun_out/sw_${cfg}_$o.log 2>&1
  python - "$o" gpurun_out/sw_${cfg}_$o.log <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print("opt",sys.argv[1],"ms/step %.4f"%d["ms_per_step"], " ".join(f"{k}={v['avg_us']:.1f}" for k,v in d["kernels"].items()))
except Exception as e:
    print("opt",sys.argv[1],"FAILED",open(sys.argv[2]).read()[-800:])
PY
done
