"""MRA of config 4 with a given library build (A/B of allocation modes)."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200.abi import Backend  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

be = Backend(os.path.abspath(sys.argv[1]), "fm_")
be.call("init", 0)
sc = S.config4(1)
for rep in range(3):
    g = be.grid(sc.dem, sc.L, sc.eps)
    print(os.path.basename(sys.argv[1]), rep, "mra kernels ms:", round(g.timing()[0], 3), flush=True)
    del g
