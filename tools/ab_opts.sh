#!/bin/bash
# A/B kernel options on bench.py (product library):
#   tools/ab_opts.sh "c3 c4" 10 "balance=0" "balance=1" "tile_rows=7424,col_bits=12"
# (an option set is a comma-separated list of name=value)
cfgs=$1; steps=$2; shift 2
mkdir -p gpurun_out
for c in $cfgs; do for set in "$@"; do
  args=""; for kv in ${set//,/ }; do args="$args --option $kv"; done
  log=gpurun_out/abo_${c}_$(echo "$set" | tr ',=' '_-').log
  timeout 600 python bench.py --config $c --steps $steps --no-cpu-baseline --no-oneshot --no-factored ${AB_EXTRA:-} $args > $log 2>&1
  python - "$c" "$set" "$log" <<'PY'
import json, sys
c, v, f = sys.argv[1:]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ks = {k: x.get("mean_launch_ms") for k, x in d["kernels"].items()}
    t = d["config"].get("tiled", {})
    sh = {k: (x["tile_rows"], x["block_cols"], x["slots"]) for k, x in t.items()}
    print(c, v, round(d["ms_per_step"], 3), ks, "e2e", round(d["e2e"]["ms_per_step"], 3), sh)
except Exception as e:
    print(c, v, "FAILED", open(f).read()[-400:])
PY
done; done
