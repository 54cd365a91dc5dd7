set -u
# Round-2 GPU check: full GPU tests, smoke, one-shot profile, c3 bench (with
# the one-shot and reference legs), c4 bench, c3 launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_all.log | tail -15
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 600 python tools/oneshot_profile.py --config c3 > gpurun_out/oneshot_c3.jsonl 2>&1; echo "oneshot exit $?"; cat gpurun_out/oneshot_c3.jsonl | tail -4
timeout 1200 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log | cut -c1-600
timeout 900 python bench.py --config c4 --steps 10 --no-cpu-baseline --no-oneshot > gpurun_out/bench_c4.log 2>&1
echo "bench c4 exit $?"; tail -1 gpurun_out/bench_c4.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-oneshot > gpurun_out/ncu_l.log 2>&1
echo "ncu launches exit $?"
