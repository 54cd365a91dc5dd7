set -u
mkdir -p gpurun_out
AB_EXTRA="--scale 1.0" bash tools/ab_opts.sh "c1" 20 "tiled_min_rows=10000" "tiled_min_rows=10000,tile_rows=1440,col_bits=13" "tiled_min_rows=10000,tile_rows=1440,col_bits=14" "tiled_min_rows=10000,tile_rows=1024,col_bits=13" > gpurun_out/ab_small_tiles.txt 2>&1
AB_EXTRA="--scale 0.2" bash tools/ab_opts.sh "c2" 20 "tiled_min_rows=10000" "tiled_min_rows=10000,tile_rows=1504,col_bits=12" "tiled_min_rows=10000,tile_rows=1504,col_bits=14" >> gpurun_out/ab_small_tiles.txt 2>&1
AB_EXTRA="--scale 0.5" bash tools/ab_opts.sh "c1" 20 "balance=1" "tiled_min_rows=10000,tile_rows=1024,col_bits=13" "tiled_min_rows=10000,tile_rows=1024,col_bits=14" >> gpurun_out/ab_small_tiles.txt 2>&1
cut -c1-300 gpurun_out/ab_small_tiles.txt
