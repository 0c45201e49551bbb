# usage: bash tools/sanitize.sh TOOL  -> gpurun_out/sanitize_TOOL.log
tool=$1
timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
  python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$tool.log
