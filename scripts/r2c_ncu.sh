#!/bin/bash
# Round-2 (end) ncu evidence: the bench launch list, the MRA encode, the DG2
# stage kernels and the adaptive re-grid's warm launch list.  Every profiled
# command first exits 0 without ncu.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-configs --uniform-steps 4 --solver-steps 16"
$B > gpurun_out/r2c_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches_bench.csv $B > gpurun_out/r2c_ncu_bench.log 2>&1
python scripts/prof_mra.py > gpurun_out/r2c_plain_mra.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_encode_tiles|k_grade_count_quad|k_topdown_quad" -s 20 -c 4 -o gpurun_out/r2c_mra python scripts/prof_mra.py > gpurun_out/r2c_ncu_mra.log 2>&1
python scripts/prof_solver.py dg2 1 4 5 > gpurun_out/r2c_plain_dg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stage|k_seg" -s 12 -c 3 -o gpurun_out/r2c_dg2 python scripts/prof_solver.py dg2 1 4 5 > gpurun_out/r2c_ncu_dg2.log 2>&1
python scripts/prof_adapt.py c3 4 > gpurun_out/r2c_plain_adapt.log 2>&1 && \
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2c_adapt_warm.csv python scripts/prof_adapt.py c3 4 > gpurun_out/r2c_ncu_adapt.log 2>&1
ls -la gpurun_out/r2c_*
