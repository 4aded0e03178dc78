import sys, time, numpy as np
import os; sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import api
gpu = api.lib()
orc = Backend(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "oracle/liboracle.so"), "orc_")
def cmp_grid(sc, kind=0):
    g = gpu.grid(sc.dem, sc.L, sc.eps, True, kind); o = orc.grid(sc.dem, sc.L, sc.eps, True, kind)
    a = g.leaves(); b = o.leaves()
    same = g.num_leaves == o.num_leaves and all(np.array_equal(x, y) for x, y in zip(a, b))
    ms, by = g.timing()
    print("GRID", sc.name, kind, g.num_leaves, o.num_leaves, "EXACT" if same else "DIFF", f"{ms:.3f}ms", flush=True)
    if not same and g.num_leaves == o.num_leaves:
        for n, (x, y) in enumerate(zip(a, b)):
            bad = np.nonzero(x != y)[0]
            print("  field", n, len(bad), bad[:5])
    return g, o
for k, scale in [(0, 1), (1, 1), (3, 1), (4, 8)]:
    sc = S.CONFIGS[k](scale)
    cmp_grid(sc)
cmp_grid(S.config1(2), kind=1)
for name, sc, n in [("c0", S.config0(1), 50), ("c1", S.config1(2), 200), ("c2fv1", S.config2(2, adaptive=False), 100), ("c4nu", S.config4(16), 30)]:
    go = gpu.grid(sc.dem, sc.L, sc.eps); oo = orc.grid(sc.dem, sc.L, sc.eps)
    sg = gpu.sim(sc, go); so = orc.sim(sc, oo)
    t = time.time(); cg, rg = sg.run(n, gauge_interval=10.0); tg = time.time() - t
    t = time.time(); co, ro = so.run(n, gauge_interval=10.0); to = time.time() - t
    a = sg.download(); b = so.download()
    u1, u2 = a[3], b[3]
    d = np.abs(u1 - u2); tol = np.maximum(1e-9 * np.abs(u2), 1e-10)
    print("SIM", name, sg.num_cells, so.num_cells, rg.steps, ro.steps, cg.now, co.now, "maxdiff", d.max(), "viol", int((d > tol).sum()), "exact", int((d == 0).sum()), "/", d.size, f"gpu {tg:.3f}s ({sg.last_run_ms():.2f} ms dev) cpu {to:.3f}s", flush=True)
