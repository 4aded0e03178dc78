"""Where the reference DG2/adaptive runs stop tolerating a libm perturbation: the
unmodified reference (native glibc) against the oracle with the portable cube
root, step by step, for every golden sim case; prints the first step that
leaves isclose_flow.  Used to pick the golden horizons in make_golden.py."""
import os, sys, numpy as np
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import Backend, isclose_flow, c_clock
ref = Backend(os.path.join(sys.path[1], 'oracle/_ref/libfmref.so'), 'ref_')
orc = Backend(os.path.join(sys.path[1], 'oracle/liboracle.so'), 'orc_')
ref.fn["set_threads"](8)
import make_golden as MG
for name,(sc,steps) in MG.SIMS.items():
    res=[]
    for be,libm in ((ref,0),(orc,1)):
        g = None
        if sc.grid_mode == "nonuniform" and sc.solver not in ("mwdg2", "hwfv1"):
            g = be.grid(sc.dem, sc.L, sc.eps)
        res.append(be.sim(sc, g, libm=libm) if be is orc else be.sim(sc,g))
    a,b=res
    cka=c_clock(1e12,0.0,10.0,0.0,1,1); ckb=c_clock(1e12,0.0,10.0,0.0,1,1)
    first=None
    maxn=max(steps,200)
    for k in range(1,maxn+1):
        cka,_=a.run(1,clock=cka); ckb,_=b.run(1,clock=ckb)
        ua=a.download(); ub=b.download()
        if not all(np.array_equal(x,y) for x,y in zip(ua[:3],ub[:3])):
            first=(k,'grid'); break
        ok=isclose_flow(ub[3],ua[3])
        if not ok.all():
            first=(k,int((~ok).sum())); break
    print(name, sc.solver, a.num_cells, 'golden steps',steps,'first fail',first, flush=True)
