"""Config-4 uniform raster DG2: a few steps for ncu (kernel k_uni_march)."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

lib = api.lib()
sc = S.config4(int(sys.argv[1]) if len(sys.argv) > 1 else 1, uniform=True)
s = lib.sim(sc, None)
s.run(3, gauge_interval=10.0)
print("uniform ok", s.num_cells, flush=True)
