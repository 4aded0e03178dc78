#!/bin/bash
# compute-sanitizer over scripts/sanitize_workload.py, ONE tool per call (the
# profiling guide: several tools in one call have left B200 GPUs unusable).
# usage (under gpurun): bash scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck
tool=${1:-memcheck}
mkdir -p gpurun_out
python scripts/sanitize_workload.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 compute-sanitizer --tool "$tool" --error-exitcode 9 --print-limit 50 \
  python scripts/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
echo "SANITIZER_EXIT $?" >> gpurun_out/sanitize_$tool.log
tail -5 gpurun_out/sanitize_$tool.log
