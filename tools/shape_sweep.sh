#!/bin/bash
# Per-hop time of the config-4 depth sweep (F=2 passes only) for BMT tile shapes
# "rows:colbits" (tools/depth_sweep.py; env GIFT_BMT_TILE_ROWS / GIFT_BMT_COL_BITS).
#   bash tools/shape_sweep.sh "4096:13 8192:13 8192:12" [config]
shapes=$1; c=${2:-c4}
mkdir -p gpurun_out
for sh in $shapes; do
  r=${sh%%:*}; cb=${sh#*:}
  GIFT_BMT_TILE_ROWS=$r GIFT_BMT_COL_BITS=$cb timeout 600 python tools/depth_sweep.py --config $c --depths 4 8 16 \
    > gpurun_out/shape_${c}_${r}_${cb}.jsonl 2>&1
  echo "$c rows=$r colbits=$cb: $(tail -1 gpurun_out/shape_${c}_${r}_${cb}.jsonl | cut -c1-200)"
done
