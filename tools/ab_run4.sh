set -u
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider -k "bmt or sharded or deterministic or pinned" > gpurun_out/pytest_bmt.log 2>&1
echo "bmt tests exit $?"; tail -3 gpurun_out/pytest_bmt.log; grep -E "^FAILED|assert" gpurun_out/pytest_bmt.log | head
tools/ab_libs.sh "main" "c4" 10
tools/ab_libs.sh "main" "c4" 10 GIFT_BMT_CHUNK=0
tools/ab_libs.sh "main" "c3" 10
tools/ab_libs.sh "main" "c3" 10 GIFT_BMT_TILE_ROWS=1024 GIFT_BMT_COL_BITS=11
tools/ab_libs.sh "main" "c2" 10
tools/ab_libs.sh "main" "c2" 10 GIFT_BMT_TILE_ROWS=1024 GIFT_BMT_COL_BITS=11
