#!/bin/bash
# Round-2 evidence in one GPU call: full GPU tests, smoke, ncu captures of the
# hop kernels (c3, c4), the c3 launch list, all bench lines (c3 default with
# the one-shot / reference legs, reference arm, c0-c2, c4), full-size parity
# of the five configs, the c4 depth sweep and the one-shot profile.
# Outputs in gpurun_out/ (copy what is judged to profiles/).
set -u
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_all.log 2>&1
  echo "pytest exit $?"; grep -E "passed|failed" gpurun_out/pytest_all.log | tail -3
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
fi
for c in c3 c4; do
  timeout 1500 ncu --set full --clock-control none --import-source on -f -k regex:k_hop -s 8 -c 8 \
    -o /tmp/r02_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-oneshot --no-factored > gpurun_out/r02_ncu_$c.log 2>&1
  echo "ncu full $c exit $?"
  # (the reports stay in /tmp: gpurun_out/ must stay under 64 MiB)
  ncu -i /tmp/r02_$c.ncu-rep --page raw --csv > /tmp/r02_${c}_raw.csv 2>/dev/null
  python tools/ncu_stalls.py /tmp/r02_${c}_raw.csv > gpurun_out/r02_hop_kernels_$c.txt 2>&1
  ncu -i /tmp/r02_$c.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/r02_${c}_sass.csv.gz
  gzip -c /tmp/r02_${c}_raw.csv > gpurun_out/r02_${c}_raw.csv.gz
  python tools/ncu_traffic.py /tmp/r02_$c.ncu-rep \
    "ncu --set full --clock-control none -k regex:k_hop -s 8 -c 8, bench.py --config $c (tools/evidence_r02.sh)" \
    > gpurun_out/r02_traffic_$c.json
done
# the factored clique model's two hop kernels (bench.py "factored" leg)
timeout 1200 ncu --set full --clock-control none --import-source on -f -k regex:k_fact -s 8 -c 4 -o /tmp/fact_c3 \
  python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-oneshot > gpurun_out/ncu_fact.log 2>&1
echo "ncu factored exit $?"
ncu -i /tmp/fact_c3.ncu-rep --page raw --csv > /tmp/fact_c3_raw.csv 2>/dev/null
python tools/ncu_stalls.py /tmp/fact_c3_raw.csv > gpurun_out/r02_fact_kernels_c3.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-oneshot --no-factored > gpurun_out/ncu_l.log 2>&1
echo "ncu launches exit $?"
cp gpurun_out/r02_traffic_c3.json gpurun_out/r02_traffic_c4.json profiles/ 2>/dev/null
timeout 1500 python bench.py > gpurun_out/r02_bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r02_bench_c3.log | cut -c1-300
timeout 1500 python bench.py --impl reference > gpurun_out/r02_bench_reference.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/r02_bench_reference.log | cut -c1-300
for c in c0 c1 c2 c4; do
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --no-oneshot > gpurun_out/r02_bench_$c.log 2>&1
  echo "bench $c exit $?"; tail -1 gpurun_out/r02_bench_$c.log | cut -c1-200
done
timeout 2400 python tools/full_parity.py c0 c1 c2 c3 c4 > gpurun_out/r02_full_parity.jsonl 2> gpurun_out/full_parity.err
echo "full parity exit $?"; cut -c1-200 gpurun_out/r02_full_parity.jsonl
timeout 900 python tools/depth_sweep.py --config c4 > gpurun_out/r02_depth_sweep_c4.jsonl 2> gpurun_out/depth_sweep.err
echo "depth sweep exit $?"; tail -2 gpurun_out/r02_depth_sweep_c4.jsonl | cut -c1-300
timeout 600 python tools/oneshot_profile.py --config c3 > gpurun_out/r02_oneshot_c3.jsonl 2>&1; echo "oneshot exit $?"
ls -la gpurun_out | head -50
