import sys, dataclasses, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
orc = Backend('/root/repo/oracle/liboracle.so', 'orc_')
for uni in (False, True):
    sc = dataclasses.replace(S.config4(8, uniform=uni), solver="fv1", courant=0.5)
    def go(be):
        g = None if uni else be.grid(sc.dem, sc.L, sc.eps)
        s = be.sim(sc, g, libm=1)
        s.run(5, gauge_interval=10.0)
        ck, r = s.run(16, gauge_interval=10.0)
        return s.download()[3], ck.now
    uo, to = go(orc)
    out = []
    for lib in sys.argv[1:]:
        be = Backend(lib, "fm_"); be.call("init", 0)
        u, t = go(be)
        out.append((lib.split('/')[-1], int((u != uo).sum()), t == to))
    print("uniform" if uni else "nonuniform", out, flush=True)
