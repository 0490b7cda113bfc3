# one compute-sanitizer tool per gpurun call: bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck
tool=$1
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 3 --print-limit 50 python tools/sanitize_case.py \
  > gpurun_out/sanitize_$tool.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$tool.log
tail -12 gpurun_out/sanitize_$tool.log
