#!/bin/bash
# One GPU call that refreshes the round's evidence: full GPU tests, smoke,
# both bench arms, c2/c4 lines, the ncu launch list and a full capture of the
# hop kernels.  Outputs land in gpurun_out/ (copy what is judged to profiles/).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log
for c in c2 c4; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/bench_$c.log | cut -c1-400
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hop -s 16 -c 8 \
  -o gpurun_out/prof_final_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
echo "ncu full exit $?"
