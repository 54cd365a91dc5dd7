set -u
mkdir -p gpurun_out
for o in "" "--option tiled_min_rows=100000" "--option tiled_min_rows=100000 --option tiled_min_mean=16"; do
  timeout 300 python bench.py --config c1 --steps 50 --no-cpu-baseline --no-oneshot $o > gpurun_out/c1.log 2>&1
  echo "c1 [$o] $?"; tail -1 gpurun_out/c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k:v['mean_launch_ms'] for k,v in d['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],3))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bank_fused -c 20 --csv python bench.py --config c0 --steps 10 --no-cpu-baseline --no-oneshot > gpurun_out/ncu_c0.csv 2>&1; echo "ncu c0 $?"
grep k_bank_fused gpurun_out/ncu_c0.csv | tail -5 | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv python bench.py --config c1 --steps 3 --no-cpu-baseline --no-oneshot > gpurun_out/ncu_c1.csv 2>&1; echo "ncu c1 $?"
python tools/ncu_summary.py launches gpurun_out/ncu_c1.csv 2>/dev/null | sort -k2 -n -r | head -8
