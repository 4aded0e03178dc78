"""Small deterministic workload for ncu: config-4 MRA + a few DG2 steps.

usage: python scripts/prof_run.py [scale] [steps]
"""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
lib = api.lib()
sc = S.config4(scale)
g = lib.grid(sc.dem, sc.L, sc.eps)
s = lib.sim(sc, g)
prof = s.profile(steps)
print("leaves", s.num_cells, "segments", s.num_segments, "mra", g.timing())
for k, (ms, n) in prof.items():
    print(f"{k:18s} {ms / n:.3f} ms/launch x{n}")
