"""Wall-clock of repeated state downloads of the config-4 sim into pinned and
pageable host buffers (the e2e leg's last phase)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

lib = api.lib()
sc = S.config4(1)
g = lib.grid(sc.dem, sc.L, sc.eps)
s = lib.sim(sc, g)
s.run(5, gauge_interval=10.0)
n = s.num_cells
for mode in ("pinned", "pinned-fresh", "pageable"):
    ts = []
    for rep in range(4):
        if mode == "pageable":
            out = None
        elif mode == "pinned-fresh" or rep == 0:
            shapes = [((n,), torch.int32)] * 3 + [((n, 9), torch.float64), ((n, 3), torch.float64)]
            pin = [torch.empty(sh, dtype=dt, pin_memory=True) for sh, dt in shapes]
            out = [t.numpy() for t in pin]
        t = time.perf_counter()
        s.download(out=out)
        ts.append(round(1000 * (time.perf_counter() - t), 2))
    print(mode, "ms:", ts, flush=True)
