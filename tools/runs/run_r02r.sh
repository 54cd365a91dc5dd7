set -u
mkdir -p gpurun_out
timeout 300 python tools/sanitize_smoke.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain $?"; tail -2 gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|sanitize smoke ok|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log | tail -3
done
