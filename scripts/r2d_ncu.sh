#!/bin/bash
# Round-2 final ncu evidence on the committed code: the bench launch list, one
# --set full capture per dominant kernel (DG2 stage / segment, ACC faces /
# leaves, MRA encode, uniform marching kernel).  Every profiled command first
# exits 0 without ncu.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-configs --uniform-steps 4 --solver-steps 16"
$B > gpurun_out/r2d_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_bench.csv $B > gpurun_out/r2d_ncu_bench.log 2>&1
python scripts/prof_solver.py dg2 1 4 5 > gpurun_out/r2d_plain_dg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stage|k_seg" -s 12 -c 4 -o gpurun_out/r2d_dg2 python scripts/prof_solver.py dg2 1 4 5 > gpurun_out/r2d_ncu_dg2.log 2>&1
python scripts/prof_solver.py acc 1 4 5 > gpurun_out/r2d_plain_acc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_acc_faces|k_acc_leaves" -s 8 -c 2 -o gpurun_out/r2d_acc python scripts/prof_solver.py acc 1 4 5 > gpurun_out/r2d_ncu_acc.log 2>&1
python scripts/prof_mra.py > gpurun_out/r2d_plain_mra.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_encode_tiles|k_grade|k_topdown" -s 20 -c 4 -o gpurun_out/r2d_mra python scripts/prof_mra.py > gpurun_out/r2d_ncu_mra.log 2>&1
python scripts/prof_solver.py uni 1 2 3 > gpurun_out/r2d_plain_uni.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_uni_march" -s 6 -c 2 -o gpurun_out/r2d_uni python scripts/prof_solver.py uni 1 2 3 > gpurun_out/r2d_ncu_uni.log 2>&1
for r in dg2 acc mra uni; do
  python scripts/ncu_summary.py gpurun_out/r2d_$r.ncu-rep > gpurun_out/r2d_${r}_summary.txt 2>&1
  ncu -i gpurun_out/r2d_$r.ncu-rep --page details --csv > gpurun_out/r2d_${r}_details.csv 2>/dev/null
done
ls -la gpurun_out/r2d_*
