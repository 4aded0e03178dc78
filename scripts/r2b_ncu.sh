#!/bin/bash
# Round-2 (second half) ncu evidence: the bench launch list, the marching
# uniform stage kernels, and the adaptive re-grid's launch list (config 3).
# Every profiled command first exits 0 without ncu.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-configs --uniform-steps 4 --solver-steps 16"
$B > gpurun_out/r2b_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_bench.csv $B > gpurun_out/r2b_ncu_bench.log 2>&1
python scripts/prof_uniform.py 1 > gpurun_out/r2b_plain_uni.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_uni_march" -s 2 -c 2 -o gpurun_out/r2b_uni python scripts/prof_uniform.py 1 > gpurun_out/r2b_ncu_uni.log 2>&1
python scripts/prof_adapt.py c3 4 > gpurun_out/r2b_plain_adapt.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_adapt_launches.csv python scripts/prof_adapt.py c3 4 > gpurun_out/r2b_ncu_adapt.log 2>&1
ls -la gpurun_out/r2b_*
