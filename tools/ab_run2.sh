set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "bmt or sharded or deterministic or pinned" > gpurun_out/pytest_bmt.log 2>&1
echo "bmt tests exit $?"; tail -3 gpurun_out/pytest_bmt.log
tools/ab_libs.sh "main n43 n64 d53" "c3 c4" 10
tools/ab_libs.sh "main" "c3 c4" 10 GIFT_BMT_NB=0
