#!/bin/bash
# Full ncu captures of the BMT hop launches (one F=4, one F=2 pass) on c3 and c4.
# Usage (on the GPU box): bash tools/ncu_hop.sh TAG
set -u
tag=${1:-hop}
mkdir -p gpurun_out
for c in c3 c4; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hop_bmt -s 2 -c 2 \
    -o gpurun_out/${tag}_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_$c.log 2>&1
  echo "ncu $c exit $?"
done
