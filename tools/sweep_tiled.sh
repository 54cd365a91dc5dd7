# tiled vs row kernel on c3 / c2 (bench kernels block)
for cfg in c3 c2; do
for T in 0 1; do for G in 8 16; do
  if [ $T = 0 ] && [ $G = 8 ]; then continue; fi
  GIFT_HOP_TILED=$T GIFT_TILE_G=$G timeout 300 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/st_${cfg}_${T}_${G}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/st_${cfg}_${T}_${G}.log').read().strip().splitlines()[-1]); print('$cfg tiled=$T G=$G', round(d['ms_per_step'],3), {k:(v.get('mean_launch_ms'), v.get('frac')) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/st_${cfg}_${T}_${G}.log
done; done; done
