set -u
mkdir -p gpurun_out
for v in base nobulk; do echo "== $v"; GIFT_LIB=_variants/lib_$v.so timeout 300 python tools/ab_hash.py; done > gpurun_out/ab_hash_bulk.txt 2>&1; cat gpurun_out/ab_hash_bulk.txt
bash tools/ab_libs.sh "base nobulk" "c3 c4 c2" 20 > gpurun_out/ab_bulk.txt 2>&1; cat gpurun_out/ab_bulk.txt | cut -c1-220
bash tools/ab_libs.sh "nobulk base" "c3" 20 >> gpurun_out/ab_bulk.txt 2>&1; tail -2 gpurun_out/ab_bulk.txt | cut -c1-220
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bmt_hop or full_size or sharded or high_fanout or tiled_policy" > gpurun_out/pytest_sel.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_sel.log
