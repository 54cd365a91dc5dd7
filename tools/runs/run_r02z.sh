set -u
mkdir -p gpurun_out
# launcher + sharded bench code path end to end with two ranks SHARING the one GPU (gloo control group,
# peer exchange over real CUDA IPC between the two processes): a smoke test of bench.py --gpus N, not a measurement
GIFT_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config c2 --steps 3 --warmup 3 > gpurun_out/bench_gpus2_shared.log 2>&1
echo "shared-gpu bench exit $?"; tail -3 gpurun_out/bench_gpus2_shared.log | cut -c1-700
GIFT_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --exchange nccl > gpurun_out/bench_gpus2_shared_a2a.log 2>&1
echo "shared-gpu bench (all_to_all) exit $?"; tail -3 gpurun_out/bench_gpus2_shared_a2a.log | cut -c1-400
