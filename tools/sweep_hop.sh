for cfg in c3 c1; do
for G in 8 16 32; do for U in 1 2; do
  if [ $cfg = c3 ] && [ $G = 8 ]; then continue; fi
  GIFT_HOP_G=$G GIFT_HOP_U=$U timeout 300 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/sw_${cfg}_${G}_${U}.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_${cfg}_${G}_${U}.log').read().strip().splitlines()[-1]); k=d['kernels']; print('$cfg G=$G U=$U', round(d['ms_per_step'],3), {n:(v.get('mean_launch_ms'), v.get('frac')) for n,v in k.items()})"
done; done; done
