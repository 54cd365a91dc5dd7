#!/bin/bash
# A/B library variants (tools/build_variants.sh) on bench.py:
#   tools/ab_libs.sh "base d43 s43" "c3 c4" [steps] [extra env assignments...]
libs=$1; cfgs=$2; steps=${3:-10}; shift 3 2>/dev/null
mkdir -p gpurun_out
for c in $cfgs; do for v in $libs; do
  log=gpurun_out/ab_${v}_${c}$(echo "$@" | tr ' =' '_-').log
  env GIFT_LIB=_variants/lib_$v.so "$@" timeout 600 python bench.py --config $c --steps $steps --no-cpu-baseline --no-factored > $log 2>&1
  python - "$c" "$v" "$log" "$*" <<'PY'
import json, sys
c, v, f, extra = sys.argv[1:]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ks = {k: x.get("mean_launch_ms") for k, x in d["kernels"].items()}
    print(c, v, extra, round(d["ms_per_step"], 3), ks, "e2e", round(d["e2e"]["ms_per_step"], 3))
except Exception as e:
    print(c, v, extra, "FAILED", open(f).read()[-400:])
PY
done; done
