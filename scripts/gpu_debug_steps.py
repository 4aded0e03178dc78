import os, sys, numpy as np
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import api
gpu = api.lib(); orc = Backend(os.path.join(ROOT, "oracle/liboracle.so"), "orc_")
def lockstep(name, sc, nsteps, use_run=False):
    go = gpu.grid(sc.dem, sc.L, sc.eps); oo = orc.grid(sc.dem, sc.L, sc.eps)
    sg = gpu.sim(sc, go); so = orc.sim(sc, oo)
    a = sg.download(); b = so.download()
    print(name, "init u equal:", np.array_equal(a[3], b[3]), "z equal:", np.array_equal(a[4], b[4]), flush=True)
    t = 0.0
    for k in range(nsteps):
        dg, do = sg.compute_dt(), so.compute_dt()
        dt = min(do, 10.0 - (t % 10.0)) if do == do else 10.0
        if dt <= 0 or dt == float("inf"): dt = 10.0
        sg.step(dt); so.step(dt)
        ag = sg.apply_inflows(t, dt); ao = so.apply_inflows(t, dt)
        t += dt
        a = sg.download(); b = so.download()
        ua, ub = a[3], b[3]
        d = np.abs(ua - ub)
        if k < 3 or (d > 0).any():
            bad = np.argwhere(d > 0)
            print(f" step {k} dt_gpu={dg!r} dt_orc={do!r} added {ag!r} {ao!r} ndiff={len(bad)} maxd={d.max():.3e}", flush=True)
            for r, c in bad[:6]:
                print(f"   leaf l={a[0][r]} i={a[1][r]} j={a[2][r]} coef {c}: gpu {ua[r,c]!r} orc {ub[r,c]!r} (u0 h {ub[r,0]!r})")
            if (d > 0).any():
                return
lockstep("c0", S.config0(1), 30)
lockstep("c4nu_s16", S.config4(16), 10)
lockstep("c0_s4", S.config0(4), 30)
