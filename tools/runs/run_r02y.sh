set -u
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02_bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r02_bench_c3.log | cut -c1-200
for c in c2 c4 c1 c0; do
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --no-oneshot > gpurun_out/r02_bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/r02_bench_$c.log | cut -c1-160
done
