#!/bin/bash
# e2e A/B of the in-place pinned host path: tools/ab_e2e.sh "c3 c2"
for c in ${1:-c3}; do for v in 1 0; do
  GIFT_ZERO_COPY=$v timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/e2e_${c}_${v}.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/e2e_${c}_${v}.log').read().strip().splitlines()[-1])
print('$c', 'zero_copy=$v', 'device ms', round(d['ms_per_step'],3), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'e2e', '%.3e'%d['e2e']['value'], 'h2d', d['e2e']['h2d_bytes_per_step'])
" || tail -5 gpurun_out/e2e_${c}_${v}.log
done; done
