import sys, dataclasses, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
orc = Backend('/root/repo/oracle/liboracle.so', 'orc_')
for scale, steps in ((16, 30), (8, 20), (4, 21)):
    sc = dataclasses.replace(S.config4(scale), solver="fv1", courant=0.5)
    o = orc.sim(sc, orc.grid(sc.dem, sc.L, sc.eps), libm=1)
    o.run(steps, gauge_interval=10.0)
    uo = o.download()[3]
    res = []
    for lib in sys.argv[1:]:
        be = Backend(lib, "fm_"); be.call("init", 0)
        s = be.sim(sc, be.grid(sc.dem, sc.L, sc.eps), libm=1)
        s.run(steps, gauge_interval=10.0)
        u = s.download()[3]
        res.append((lib.split('/')[-1], int((u != uo).sum()), float(np.nanmax(np.abs(u - uo)))))
    print(scale, res, flush=True)
