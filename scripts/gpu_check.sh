#!/bin/bash
# GPU iteration helper: parity tests then a bench line.
# usage (under gpurun): bash scripts/gpu_check.sh TAG [pytest-args...]
# env: BENCH_ARGS (default "--no-cpu"), NO_TESTS=1 skips pytest
tag=$1; shift
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --durations=25 "$@" > gpurun_out/pytest_$tag.log 2>&1
  echo PYTEST_EXIT $? >> gpurun_out/pytest_$tag.log
fi
timeout 1200 python bench.py ${BENCH_ARGS:---no-cpu} > gpurun_out/bench_$tag.log 2>&1
echo BENCH_EXIT $? >> gpurun_out/bench_$tag.log
tail -c 300 gpurun_out/pytest_$tag.log 2>/dev/null
tail -c 200 gpurun_out/bench_$tag.log
