#!/bin/bash
# GPU iteration helper: parity tests then a bench line (no CPU leg).
# usage (under gpurun): bash scripts/gpu_check.sh TAG [pytest-args...]
tag=$1; shift
python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_$tag.log 2>&1
echo PYTEST_EXIT $? >> gpurun_out/pytest_$tag.log
python bench.py --no-cpu > gpurun_out/bench_$tag.log 2>&1
echo BENCH_EXIT $? >> gpurun_out/bench_$tag.log
