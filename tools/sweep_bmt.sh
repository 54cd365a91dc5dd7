# BMT vs row kernel on c3 / c2 (bench kernels block)
for cfg in c3 c2; do
for B in 0 1; do
  GIFT_BMT=$B timeout 300 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/sb_${cfg}_${B}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sb_${cfg}_${B}.log').read().strip().splitlines()[-1]); print('$cfg bmt=$B', round(d['ms_per_step'],3), {k:(v.get('mean_launch_ms'), v.get('frac')) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/sb_${cfg}_${B}.log
done; done
