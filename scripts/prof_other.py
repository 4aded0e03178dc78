"""Per-kernel timing of the other BASELINE workloads: config-4 uniform-raster
DG2 (8192^2 cells), config-1 ACC and config-2 FV1 (1024^2, L = 10)."""
import os
import sys
import time

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

lib = api.lib()
which = sys.argv[1:] or ["uni", "acc", "fv1"]
static = [w for w in which if w in ("uni", "acc", "fv1")]
for w in static:
    if w == "uni":
        sc = S.config4(1, uniform=True)
        g = None
    elif w == "acc":
        sc = S.config1(1)
        g = lib.grid(sc.dem, sc.L, sc.eps)
    else:
        sc = S.config2(1, adaptive=False)
        g = lib.grid(sc.dem, sc.L, sc.eps)
    s = lib.sim(sc, g)
    s.run(20, gauge_interval=10.0)
    prof = s.profile(10)
    s.run(50, gauge_interval=10.0)
    ms = s.last_run_ms() / 50
    n = s.num_cells
    print(w, "cells", n, "segments", s.num_segments, f"run {ms:.4f} ms/step",
          f"{n / ms / 1e3 / 1e6:.1f} M cell-updates/s")
    for k, (t, c) in prof.items():
        print(f"   {k:16s} {t / c:.4f} ms/launch")
    del s, g


def adaptive(scale=1, steps=20):
    """Config 3 (MWDG2, re-gridded every step) and config 2 (HWFV1)."""
    for name, sc in (("c3_mwdg2", S.config3(scale)), ("c2_hwfv1", S.config2(scale))):
        t0 = time.perf_counter()
        s = lib.sim(sc, None)
        t1 = time.perf_counter()
        s.run(3, gauge_interval=10.0)
        t2 = time.perf_counter()
        ck, r = s.run(steps, gauge_interval=10.0)
        t3 = time.perf_counter()
        t, cnt = s.element_log()
        print(name, f"create {1e3 * (t1 - t0):.1f} ms, {r.steps} steps in {1e3 * (t3 - t2):.1f} ms "
              f"({1e3 * (t3 - t2) / max(r.steps, 1):.2f} ms/step incl. adapt), leaves {cnt[-1] if len(cnt) else '?'}",
              flush=True)
        del s


if "adapt" in which:
    adaptive()
