set -u
mkdir -p gpurun_out
# where the tiled hop starts to beat the row kernel / graph replay / fused kernel: c1 at several scales
for sc in 1.0 0.5 0.25 0.12; do
  echo "== c1 x$sc"
  AB_EXTRA="--scale $sc" bash tools/ab_opts.sh "c1" 20 "balance=1" "tiled_min_rows=10000"
done > gpurun_out/ab_c1_tiled.txt 2>&1
# c2 scaled to mid sizes (long rows)
for sc in 0.2 0.1 0.05; do
  echo "== c2 x$sc"
  AB_EXTRA="--scale $sc" bash tools/ab_opts.sh "c2" 20 "balance=1" "tiled_min_rows=10000"
done >> gpurun_out/ab_c1_tiled.txt 2>&1
cut -c1-300 gpurun_out/ab_c1_tiled.txt
