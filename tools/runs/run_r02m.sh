set -u
mkdir -p gpurun_out
bash tools/ab_opts.sh "c4" 20 "balance=1" "tile_rows=2048,col_bits=12,barrier_free=2" "tile_rows=2560,col_bits=12,barrier_free=2" "tile_rows=2880,col_bits=12,barrier_free=2" "tile_rows=2048,col_bits=12,barrier_free=1" "tile_rows=4000,col_bits=12" > gpurun_out/ab_nb_c4.txt 2>&1
cut -c1-400 gpurun_out/ab_nb_c4.txt
bash tools/ab_opts.sh "c3" 20 "tile_rows=2048,col_bits=12,barrier_free=2" "tile_rows=2496,col_bits=12,barrier_free=2" >> gpurun_out/ab_nb_c4.txt 2>&1
tail -2 gpurun_out/ab_nb_c4.txt | cut -c1-400
