#!/bin/bash
# compute-sanitizer over a small training run; ONE tool per gpurun call (the
# profiling guide: several tools in one call left B200 GPUs unusable).
#   gpurun --timeout 1800 -- 'bash scripts/sanitize.sh memcheck'   (then racecheck, synccheck)
# Log: gpurun_out/sanitize_<tool>.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tool=${1:-memcheck}
export DGNN_LAYER_STREAMS=1
extra=""
[ "$tool" = memcheck ] && extra="--leak-check no"
python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$tool" $extra --print-limit 50 \
  python scripts/sanitize_run.py > "gpurun_out/sanitize_$tool.log" 2>&1
echo "exit $?" >> "gpurun_out/sanitize_$tool.log"
