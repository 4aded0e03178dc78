#!/bin/bash
# Round-2 ncu evidence (one gpurun call): the bench workload's launch list,
# then one full capture each of the top kernels.  Every profiled command
# first exits 0 without ncu.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-configs --uniform-steps 0 --solver-steps 16"
$B > gpurun_out/r2_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv $B > gpurun_out/r2_ncu_bench.log 2>&1
python scripts/prof_solver.py dg2 1 4 5 > gpurun_out/r2_plain_dg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stage|k_seg" -s 12 -c 3 -o gpurun_out/r2_dg2 python scripts/prof_solver.py dg2 1 4 5 > gpurun_out/r2_ncu_dg2.log 2>&1
python scripts/prof_solver.py acc 1 4 5 > gpurun_out/r2_plain_acc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_acc" -s 10 -c 2 -o gpurun_out/r2_acc python scripts/prof_solver.py acc 1 4 5 > gpurun_out/r2_ncu_acc.log 2>&1
python scripts/prof_solver.py fv1 1 4 5 > gpurun_out/r2_plain_fv1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stage|k_seg|k_head" -s 12 -c 3 -o gpurun_out/r2_fv1 python scripts/prof_solver.py fv1 1 4 5 > gpurun_out/r2_ncu_fv1.log 2>&1
python scripts/prof_mra.py > gpurun_out/r2_plain_mra.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_encode_tiles|k_sig_from_dmx|k_grade|k_topdown" -s 20 -c 6 -o gpurun_out/r2_mra python scripts/prof_mra.py > gpurun_out/r2_ncu_mra.log 2>&1
ls -la gpurun_out/r2_*
