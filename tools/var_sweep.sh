#!/bin/bash
# usage: var_sweep.sh config rounds variants...   (A/B of _lib/variants/libskgpu_<v>.so)
cfg=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
for v in "$@"; do
  SKG_LIB_VARIANT=$([ "$v" = base ] && echo "" || echo $v) timeout 300 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/var_${cfg}_$v.log 2>&1
  python - "$v" gpurun_out/var_${cfg}_$v.log <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print("var",sys.argv[1],"ms/step %.4f"%d["ms_per_step"], " ".join(f"{k}={v['avg_us']:.1f}" for k,v in d["kernels"].items()))
except Exception as e:
    print("var",sys.argv[1],"FAILED",open(sys.argv[2]).read()[-800:])
PY
done; done
