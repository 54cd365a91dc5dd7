set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "factored or high_fanout" > gpurun_out/pytest_fact.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_fact.log
timeout 1200 ncu --set full --clock-control none --import-source on -f -k regex:k_fact -s 8 -c 4 -o /tmp/fact_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-oneshot > gpurun_out/ncu_fact.log 2>&1
echo "ncu $?"
ncu -i /tmp/fact_c3.ncu-rep --page raw --csv > /tmp/fact_c3_raw.csv 2>/dev/null
python tools/ncu_stalls.py /tmp/fact_c3_raw.csv > gpurun_out/r02_fact_kernels_c3.txt 2>&1
cat gpurun_out/r02_fact_kernels_c3.txt | head -80
ncu -i /tmp/fact_c3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/r02_fact_c3_sass.csv.gz
