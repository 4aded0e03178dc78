"""Config-4 static MRA, built twice (the second build is the steady state);
for ncu launch lists of the MRA kernels."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

lib = api.lib()
sc = S.config4(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
for rep in range(3):
    g = lib.grid(sc.dem, sc.L, sc.eps)
    print(rep, "mra kernels ms, bytes:", g.timing(), "leaves", g.num_leaves, flush=True)
    del g
