#!/bin/bash
# Full ncu captures of the BMT hop launches (F=4 and F=2 passes) on c3 and c4;
# exports the raw metrics and the SASS source page as CSV on the box (the
# .ncu-rep files are too large to bring back together).
# Usage (on the GPU box): bash tools/ncu_hop.sh TAG [configs]
set -u
tag=${1:-hop}; cfgs=${2:-"c3 c4"}
mkdir -p gpurun_out
for c in $cfgs; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hop_bmt -s 4 -c 4 \
    -o /tmp/${tag}_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_$c.log 2>&1
  echo "ncu $c exit $?"
  ncu -i /tmp/${tag}_$c.ncu-rep --page raw --csv > gpurun_out/${tag}_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_${c}_sass.csv 2>/dev/null
  gzip -f gpurun_out/${tag}_${c}_sass.csv
done
ls -la gpurun_out/
