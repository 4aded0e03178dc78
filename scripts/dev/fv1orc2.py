import sys, dataclasses, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
orc = Backend('/root/repo/oracle/liboracle.so', 'orc_')
sc = dataclasses.replace(S.config4(4), solver="fv1", courant=0.5)
for libm, gi in ((1, 1e9), (0, 10.0), (0, 1e9)):
    res = []
    us = []
    for lib in sys.argv[1:]:
        be = Backend(lib, "fm_"); be.call("init", 0)
        s = be.sim(sc, be.grid(sc.dem, sc.L, sc.eps), libm=libm)
        ck, r = s.run(21, gauge_interval=gi)
        us.append(s.download()[3]); res.append((r.steps, ck.now))
    if libm == 1:
        o = orc.sim(sc, orc.grid(sc.dem, sc.L, sc.eps), libm=1)
        ck, r = o.run(21, gauge_interval=gi); uo = o.download()[3]
        print("orc", r.steps, ck.now, [int((u != uo).sum()) for u in us])
    print(libm, gi, res, int((us[0] != us[1]).sum()), np.isnan(us[0]).sum(), np.isnan(us[1]).sum(), flush=True)
