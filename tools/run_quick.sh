set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log | cut -c1-600
for c in c4; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/bench_$c.log | cut -c1-600
done
