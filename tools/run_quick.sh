set -u
# Quick GPU check: full GPU tests, smoke, c3/c4 bench lines, c3 launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -x > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; tail -15 gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log | cut -c1-900
for c in c4; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/bench_$c.log | cut -c1-900
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
echo "ncu launches exit $?"
