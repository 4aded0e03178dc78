"""Config-3 adaptive MWDG2 (2048^2, L = 11): a few re-gridded steps, for ncu."""
import os
import sys
import time

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

if os.environ.get("FM_ADAPT_LIB"):  # A/B a variant build
    from paper_2107_02750_b200.abi import Backend  # noqa: E402
    lib = Backend(os.environ["FM_ADAPT_LIB"], "fm_")
    lib.call("init", 0)
else:
    lib = api.lib()
sc = S.config3(1) if (len(sys.argv) < 2 or sys.argv[1] == "c3") else S.config2(1)
s = lib.sim(sc, None)
s.run(3, gauge_interval=10.0)
t = time.perf_counter()
ck, r = s.run(int(sys.argv[2]) if len(sys.argv) > 2 else 5, gauge_interval=10.0)
print("steps", r.steps, "ms/step", 1000 * (time.perf_counter() - t) / max(r.steps, 1),
      "device ms/step", s.last_run_ms() / max(r.steps, 1), "leaves", s.num_cells)
