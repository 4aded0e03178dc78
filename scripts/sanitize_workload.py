"""Small workload touching every kernel family, for compute-sanitizer
(scripts/sanitize.sh): static MRA (MW + HW), static DG2 / FV1 / ACC steps
(graph and host-API paths), adaptive HWFV1 / MWDG2 re-grids, the uniform
raster solvers, rasters, gauges and the reference-order download."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

small = "--small" in sys.argv  # C0 / C1 only (the -m gpu sanitizer test)
lib = api.lib()
static = ((S.config0(8), 6), (S.config1(16), 10))
if not small:
    static += ((S.config2(16, adaptive=False), 10),)
for sc, steps in static:
    g = lib.grid(sc.dem, sc.L, sc.eps)
    lib.grid(sc.dem, sc.L, sc.eps, kind=1)
    s = lib.sim(sc, g)
    s.run(steps, gauge_interval=10.0)
    s.step(s.compute_dt() if np.isfinite(s.compute_dt()) else 1.0)
    s.apply_inflows(0.0, 1.0)
    s.raster(0)
    s.sample_gauges([10.0], [10.0])
    s.download()
    s.volume()
    s.finite_state()
def guard_line():
    import ctypes as C
    if os.environ.get("FM_GUARD") == "1":
        c, o = C.c_int64(0), C.c_int64(0)
        lib.call("debug_guard_report", C.byref(c), C.byref(o))
        print(f"FM_GUARD checked={c.value} overruns={o.value}")


if small:
    guard_line()
    print("sanitize workload ok (small)")
    sys.exit(0)
for sc, steps in ((S.config2(16), 4), (S.config3(32), 3)):
    s = lib.sim(sc, None)
    s.run(steps, gauge_interval=10.0)
    s.download()
sc = S.config4(64, uniform=True)
for solver in ("dg2", "fv1", "acc"):
    sc.solver = solver
    s = lib.sim(sc, None)
    s.run(3, gauge_interval=10.0)
    s.download()
guard_line()
print("sanitize workload ok")
