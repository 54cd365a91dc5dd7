#!/bin/bash
# A/B a GIFT_* env switch on bench.py: tools/ab_bench.sh VAR "v1 v2" "c3 c2" [steps]
var=$1; vals=$2; cfgs=$3; steps=${4:-10}
mkdir -p gpurun_out
for c in $cfgs; do for v in $vals; do for rep in 1 2; do
  env $var=$v timeout 600 python bench.py --config $c --steps $steps --no-cpu-baseline > gpurun_out/ab_${var}_${v}_${c}_${rep}.log 2>&1
  python - "$c" "$v" "$rep" "gpurun_out/ab_${var}_${v}_${c}_${rep}.log" <<'PY'
import json, sys
c, v, rep, f = sys.argv[1:]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ks = {k: x.get("mean_launch_ms") for k, x in d["kernels"].items()}
    print(c, v, rep, round(d["ms_per_step"], 3), ks)
except Exception as e:
    print(c, v, rep, "FAILED", open(f).read()[-400:])
PY
done; done; done
