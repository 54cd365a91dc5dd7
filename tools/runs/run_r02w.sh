set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -x > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; tail -4 gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke $?"
for c in c1 c0 c3; do
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --no-oneshot > gpurun_out/r02_bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/r02_bench_$c.log | cut -c1-200
done
