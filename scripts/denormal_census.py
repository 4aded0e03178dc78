"""Census of subnormal values in the config-4 state after warm-up (what sends
fp64 divisions down their slow path)."""
import os
import sys

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

lib = api.lib()
sc = S.config4(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
g = lib.grid(sc.dem, sc.L, sc.eps)
s = lib.sim(sc, g)
for steps in (5, 16, 32):
    s.run(steps if steps == 5 else steps - 5, gauge_interval=10.0) if steps == 5 else None
names = ["h0", "h1x", "h1y", "qx0", "qx1x", "qx1y", "qy0", "qy1x", "qy1y"]
for k in (5, 20, 40):
    s2 = lib.sim(sc, g)
    s2.run(k, gauge_interval=10.0)
    lv, i, j, u, z = s2.download()
    tiny = np.finfo(np.float64).tiny
    sub = (u != 0) & (np.abs(u) < tiny)
    small = (u != 0) & (np.abs(u) < 2.0 ** -969)
    zero = u == 0
    print(f"after {k} steps: n={len(u)}")
    print("  subnormal frac :", " ".join(f"{n}={sub[:, q].mean():.4f}" for q, n in enumerate(names)))
    print("  < 2^-969 frac  :", " ".join(f"{n}={small[:, q].mean():.4f}" for q, n in enumerate(names)))
    print("  zero frac      :", " ".join(f"{n}={zero[:, q].mean():.4f}" for q, n in enumerate(names)))
    h = u[:, 0]
    print("  h quantiles    :", np.quantile(h, [0, 0.01, 0.1, 0.5, 0.9, 1.0]))
    print("  wet (h>1e-6)   :", (h > 1e-6).mean())
