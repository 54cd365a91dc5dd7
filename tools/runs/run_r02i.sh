set -u
mkdir -p gpurun_out
for o in "" "--option row_lanes=8" "--option row_lanes=16" "--option row_lanes=32"; do
  timeout 300 python bench.py --config c0 --steps 100 --no-cpu-baseline --no-oneshot $o > gpurun_out/c0.log 2>&1
  echo "c0 [$o] $?"; tail -1 gpurun_out/c0.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],3))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bank_fused -c 10 --csv python bench.py --config c0 --steps 10 --no-cpu-baseline --no-oneshot > gpurun_out/ncu_c0.csv 2>&1; echo "ncu c0 $?"
grep k_bank_fused gpurun_out/ncu_c0.csv | tail -3 | cut -c60-250
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "cuda_graph or c0_matches or signal_widths or many_sigma" 2>&1 | tail -2
