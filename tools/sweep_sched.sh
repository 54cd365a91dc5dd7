# BMT conflict-aware schedule on/off (c3, c2)
for cfg in c3 c2; do
for S in 0 1; do
  GIFT_BMT_SCHEDULE=$S timeout 300 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/ss_${cfg}_${S}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ss_${cfg}_${S}.log').read().strip().splitlines()[-1]); print('$cfg sched=$S', round(d['ms_per_step'],3), d['config']['graph_build_s'], {k:(v.get('mean_launch_ms'), v.get('frac')) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/ss_${cfg}_${S}.log
done; done
