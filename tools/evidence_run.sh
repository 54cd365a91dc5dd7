#!/bin/bash
# One GPU call that refreshes the round's evidence: full GPU tests, smoke, ncu
# captures of the hop kernels (raw + SASS CSV, DRAM traffic json, launch list),
# then both bench arms (the bench reads the fresh traffic json), c2/c4 lines
# and the config-4 depth sweep.  Outputs land in gpurun_out/ (copy what is
# judged to profiles/).   Usage: bash tools/evidence_run.sh [tag]
set -u
tag=${1:-ev}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
for c in c3 c4; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hop -s 8 -c 8 \
    -o /tmp/${tag}_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_$c.log 2>&1
  echo "ncu full $c exit $?"
  ncu -i /tmp/${tag}_$c.ncu-rep --page raw --csv > gpurun_out/${tag}_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_$c.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${tag}_${c}_sass.csv.gz
  python tools/ncu_traffic.py /tmp/${tag}_$c.ncu-rep \
    "ncu --set full --clock-control none -k regex:k_hop -s 8 -c 8, bench.py --config $c (tools/evidence_run.sh)" \
    > gpurun_out/r01_traffic_$c.json && cp gpurun_out/r01_traffic_$c.json profiles/
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
echo "ncu launches exit $?"
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
for c in c2 c4; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/bench_$c.log | cut -c1-300
done
timeout 1500 python tools/full_parity.py c0 c1 c2 c3 c4 > gpurun_out/full_parity.jsonl 2>gpurun_out/full_parity.err
echo "full parity exit $?"; cut -c1-160 gpurun_out/full_parity.jsonl
timeout 900 python tools/depth_sweep.py --config c4 > gpurun_out/depth_sweep_c4.jsonl 2>gpurun_out/depth_sweep_c4.err
echo "depth sweep exit $?"; tail -2 gpurun_out/depth_sweep_c4.jsonl | cut -c1-300
ls -la gpurun_out | head -40
