set -u
mkdir -p gpurun_out
for v in epf0 epf1; do echo "== $v"; GIFT_LIB=_variants/lib_$v.so timeout 300 python tools/ab_hash.py c3 0.05 c4 0.02; done > gpurun_out/ab_hash_epf.txt 2>&1; cat gpurun_out/ab_hash_epf.txt
bash tools/ab_libs.sh "epf0 epf1 epf0 epf1" "c4 c3" 20 > gpurun_out/ab_epf.txt 2>&1; cut -c1-200 gpurun_out/ab_epf.txt
