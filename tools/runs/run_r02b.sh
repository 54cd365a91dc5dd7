set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_all.log | tail -15
for c in c0 c1; do timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --no-oneshot > gpurun_out/bench_$c.log 2>&1; echo "bench $c $?"; tail -1 gpurun_out/bench_$c.log | cut -c1-300; done
/usr/bin/time -v timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log | cut -c1-700; grep -E "Elapsed|Maximum resident" gpurun_out/bench_ref.err
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
