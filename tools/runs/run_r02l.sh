set -u
mkdir -p gpurun_out
for v in pre0 pre1; do echo "== $v"; GIFT_LIB=_variants/lib_$v.so timeout 300 python tools/ab_hash.py; done > gpurun_out/ab_hash_pre.txt 2>&1; cat gpurun_out/ab_hash_pre.txt
bash tools/ab_libs.sh "pre0 pre1" "c3 c4 c2" 20 > gpurun_out/ab_pre.txt 2>&1; cut -c1-220 gpurun_out/ab_pre.txt
bash tools/ab_libs.sh "pre1 pre0" "c4" 20 >> gpurun_out/ab_pre.txt 2>&1; tail -2 gpurun_out/ab_pre.txt | cut -c1-220
timeout 1500 python -m pytest tests/test_peer_ipc.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "peer or sharded or bmt_hop or tiled_policy or high_fanout" > gpurun_out/pytest_sel.log 2>&1; echo "pytest $?"; tail -15 gpurun_out/pytest_sel.log
