set -u
mkdir -p gpurun_out
bash tools/ab_opts.sh "c4" 10 "balance=1" "tile_rows=5664,col_bits=13" "tile_rows=4864,col_bits=13" "tile_rows=3392,col_bits=13" "tile_rows=2912,col_bits=13" "tile_rows=7552,col_bits=12" > gpurun_out/ab_shapes_final.txt 2>&1
bash tools/ab_opts.sh "c3" 10 "balance=1" "tile_rows=4960,col_bits=13" "tile_rows=3712,col_bits=13" "tile_rows=7424,col_bits=11" >> gpurun_out/ab_shapes_final.txt 2>&1
cut -c1-330 gpurun_out/ab_shapes_final.txt
