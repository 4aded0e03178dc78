import sys, hashlib, dataclasses, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
def h(u): return hashlib.sha1(u.tobytes()).hexdigest()[:12]
for lib in sys.argv[1:]:
    be = Backend(lib, "fm_"); be.call("init", 0)
    sc = dataclasses.replace(S.config4(4), solver="fv1", courant=0.5)
    g = be.grid(sc.dem, sc.L, sc.eps)
    out = []
    for mode in ("A", "B", "C"):
        s = be.sim(sc, g)
        s.run(5, gauge_interval=1e9)
        if mode == "A":
            s.snapshot(); s.profile(16); s.restore()
        if mode == "C":
            s.snapshot(); s.restore()
        s.run(16, gauge_interval=1e9)
        out.append(h(s.download()[3]))
    print(lib.split('/')[-1], out)
