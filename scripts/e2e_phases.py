"""Wall-clock breakdown of the bench's e2e leg (public API from host buffers)."""
import os
import sys
import time

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402
from paper_2107_02750_b200.abi import c_clock  # noqa: E402

lib = api.lib()
sc = S.config4(1)
for rep in range(2):
    T = {}
    t = time.perf_counter()
    g = lib.grid(sc.dem, sc.L, sc.eps)
    lib.call("synchronize") if lib.has("synchronize") else None
    T["grid"] = time.perf_counter() - t
    t = time.perf_counter()
    s = lib.sim(sc, g)
    T["sim_create"] = time.perf_counter() - t
    t = time.perf_counter()
    ck, r = s.run(5, gauge_interval=10.0)
    T["warmup5"] = time.perf_counter() - t
    t = time.perf_counter()
    s.snapshot()
    T["snapshot"] = time.perf_counter() - t
    ck0 = (ck.end_time, ck.output_interval, ck.gauge_interval, ck.now, ck.next_output, ck.next_gauge)
    t = time.perf_counter()
    done = 0
    while done < 200:
        s.restore()
        _, r = s.run(16, clock=c_clock(*ck0))
        done += 16
    T["run200"] = time.perf_counter() - t
    t = time.perf_counter()
    out = s.download()
    T["download"] = time.perf_counter() - t
    print(rep, {k: round(v * 1000, 1) for k, v in T.items()}, "ms; mra kernels", g.timing())
    del s, g
