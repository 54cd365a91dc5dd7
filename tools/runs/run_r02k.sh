set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/ab_opts.sh "c3" 20 "balance=0" "balance=1" "tile_rows=7424,col_bits=12" "tile_rows=5952,col_bits=12" "tile_rows=4960,col_bits=12" "tile_rows=3712,col_bits=12" "balance=0" "balance=1" > gpurun_out/ab_balance.txt 2>&1
bash tools/ab_opts.sh "c2 c4" 20 "balance=0" "balance=1" >> gpurun_out/ab_balance.txt 2>&1
cat gpurun_out/ab_balance.txt | cut -c1-400
