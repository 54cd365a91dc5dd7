set -u
mkdir -p gpurun_out
for v in meta0 meta1 meta2; do echo "== $v"; GIFT_LIB=_variants/lib_$v.so timeout 300 python tools/ab_hash.py; done > gpurun_out/ab_hash_meta.txt 2>&1; cat gpurun_out/ab_hash_meta.txt
bash tools/ab_libs.sh "meta0 meta1 meta2" "c4 c3 c2" 20 > gpurun_out/ab_meta.txt 2>&1; cut -c1-200 gpurun_out/ab_meta.txt
bash tools/ab_libs.sh "meta2 meta1 meta0" "c4" 20 >> gpurun_out/ab_meta.txt 2>&1; tail -3 gpurun_out/ab_meta.txt | cut -c1-200
