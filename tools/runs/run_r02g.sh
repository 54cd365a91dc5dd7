set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_all.log | tail -5
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke $?"
timeout 1500 python bench.py > gpurun_out/r02_bench_c3_d4.log 2>&1; echo "bench c3 $?"; tail -1 gpurun_out/r02_bench_c3_d4.log | cut -c1-300
timeout 900 python bench.py --config c4 --steps 20 --no-cpu-baseline --no-oneshot > gpurun_out/r02_bench_c4_d4.log 2>&1; echo "bench c4 $?"; tail -1 gpurun_out/r02_bench_c4_d4.log | cut -c1-300
