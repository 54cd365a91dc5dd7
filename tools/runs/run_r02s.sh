set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "optimal_schedule or bmt_hop" > gpurun_out/pytest_sched.log 2>&1; echo "pytest $?"; tail -4 gpurun_out/pytest_sched.log
bash tools/ab_opts.sh "c3 c4 c2" 20 "schedule=1" "schedule=2" "schedule=1" > gpurun_out/ab_sched2.txt 2>&1; cut -c1-330 gpurun_out/ab_sched2.txt
