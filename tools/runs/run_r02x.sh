set -u
mkdir -p gpurun_out
# c2 runs exactly one wave of 148 tiles: are two or three waves of smaller tiles better balanced?
bash tools/ab_opts.sh "c2" 20 "balance=1" "tile_rows=3744,col_bits=12" "tile_rows=2496,col_bits=12" "tile_rows=3744,col_bits=14" "tile_rows=2496,col_bits=14" > gpurun_out/ab_c2_waves.txt 2>&1
cut -c1-300 gpurun_out/ab_c2_waves.txt
