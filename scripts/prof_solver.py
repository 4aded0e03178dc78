"""Deterministic config-4 workload for ncu and A/B runs, any static solver:
MRA, sim, W warm-up steps, then fm_sim_profile over N steps.

usage: python scripts/prof_solver.py SOLVER [scale] [steps] [warmup]
       SOLVER in dg2 | fv1 | acc | uni (the uniform-raster DG2)
"""
import dataclasses
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

solver = sys.argv[1] if len(sys.argv) > 1 else "dg2"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
warm = int(sys.argv[4]) if len(sys.argv) > 4 else 5
lib = api.lib()
if solver == "uni":
    sc = S.config4(scale, uniform=True)
    s = lib.sim(sc, None)
else:
    sc = S.config4(scale)
    sc = dataclasses.replace(sc, solver=solver, courant={"dg2": 0.33, "fv1": 0.5, "acc": 0.7}[solver])
    g = lib.grid(sc.dem, sc.L, sc.eps)
    s = lib.sim(sc, g)
s.run(warm, gauge_interval=10.0)
prof = s.profile(steps)
print("solver", solver, "cells", s.num_cells, "segments", s.num_segments)
for k, (ms, n) in prof.items():
    print(f"{k:18s} {ms / n:.4f} ms/launch x{n}")
