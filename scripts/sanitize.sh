#!/bin/bash
# compute-sanitizer over a small training run (memcheck, racecheck, synccheck,
# initcheck); logs to gpurun_out/sanitize_<tool>.log. Run on the GPU box:
#   gpurun --timeout 3000 -- 'bash scripts/sanitize.sh'
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export DGNN_LAYER_STREAMS=1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
