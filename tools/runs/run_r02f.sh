set -u
mkdir -p gpurun_out
for v in base d4 st std4; do echo "== $v"; GIFT_LIB=_variants/lib_$v.so timeout 300 python tools/ab_hash.py; done > gpurun_out/ab_hash.txt 2>&1; cat gpurun_out/ab_hash.txt
bash tools/ab_libs.sh "base d4 st std4" "c3 c4" 20 > gpurun_out/ab_stream.txt 2>&1; cat gpurun_out/ab_stream.txt | cut -c1-250
bash tools/ab_libs.sh "base st" "c2" 20 >> gpurun_out/ab_stream.txt 2>&1; tail -2 gpurun_out/ab_stream.txt | cut -c1-250
