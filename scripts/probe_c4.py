"""Probe: how config 4 behaves on the GPU (step time, dt, blow-up horizon)."""
import os
import sys
import time

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402
from paper_2107_02750_b200.abi import BlowUpError  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
gi = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
lib = api.lib()
t = time.time()
sc = S.config4(scale)
print("gen", round(time.time() - t, 2), flush=True)
g = lib.grid(sc.dem, sc.L, sc.eps)
print("mra ms", g.timing(), "leaves", g.num_leaves, flush=True)
t = time.time()
s = lib.sim(sc, g)
print("create s", round(time.time() - t, 2), "segments", s.num_segments, flush=True)
ck = None
tot = 0
for k in range(40):
    try:
        if ck is None:
            ck, r = s.run(10, gauge_interval=gi)
        else:
            ck, r = s.run(10, clock=ck)
    except BlowUpError as e:
        print("BLOWUP at step", tot, "t", e.t, flush=True)
        break
    tot += r.steps
    u = s.download()[3] if k % 5 == 4 else None
    print(tot, f"now={ck.now:.6g} dtmin={r.dt_min:.3g} dtmax={r.dt_max:.3g} ms/step={s.last_run_ms() / r.steps:.3f}",
          "" if u is None else f"max|u|={np.abs(u).max(axis=0)[[0, 3, 6]]}", flush=True)
