set -u
mkdir -p gpurun_out
bash tools/ab_libs.sh "base t768d5 t768d6 d4" "c3 c4" 20 > gpurun_out/ab_threads.txt 2>&1; cat gpurun_out/ab_threads.txt | cut -c1-250
for i in 1 2; do timeout 300 python tools/oneshot_profile.py --config c3 --repeat 1 > gpurun_out/oneshot_a$i.jsonl 2>&1; cat gpurun_out/oneshot_a$i.jsonl; done
timeout 300 python tools/oneshot_profile.py --config c3 --repeat 1 --warm-small > gpurun_out/oneshot_w.jsonl 2>&1; cat gpurun_out/oneshot_w.jsonl
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/oneshot_profile.py --config c3 --repeat 1 > gpurun_out/oneshot_e.jsonl 2>&1; cat gpurun_out/oneshot_e.jsonl
./tools/ubench_atoms > gpurun_out/ubench.txt 2>&1; cat gpurun_out/ubench.txt
