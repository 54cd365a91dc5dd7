#!/bin/bash
# double-buffered staging A/B (+ c4 tile rows)
for spec in "c3 1 0" "c3 0 0" "c2 1 0" "c2 0 0" "c4 1 0" "c4 0 0" "c4 1 4096" "c4 0 4096"; do
  set -- $spec
  c=$1; db=$2; tr=$3
  env GIFT_BMT_DB=$db GIFT_BMT_TILE_ROWS=$tr timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/db_${c}_${db}_${tr}.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/db_${c}_${db}_${tr}.log').read().strip().splitlines()[-1])
print('$c db=$db tr=$tr', round(d['ms_per_step'],3), {k:v.get('mean_launch_ms') for k,v in d['kernels'].items()})
" || tail -3 gpurun_out/db_${c}_${db}_${tr}.log
done
