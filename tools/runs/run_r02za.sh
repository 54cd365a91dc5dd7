set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "small_graph or golden or c0 or full_size or fused or factored" > gpurun_out/pytest_prep.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_prep.log
bash tools/ab_opts.sh "c3 c4 c2 c1" 20 "balance=1" > gpurun_out/ab_prep4.txt 2>&1; cut -c1-230 gpurun_out/ab_prep4.txt
