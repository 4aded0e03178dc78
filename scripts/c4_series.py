import os, sys
import numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2107_02750_b200 import api
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import c_clock
lib = api.lib()
sc = S.config4(1)
g = lib.grid(sc.dem, sc.L, sc.eps)
s = lib.sim(sc, g)
ck = c_clock(1e12, 0.0, 10.0, 0.0, 1, 1)
for k in range(60):
    t0 = ck.now
    _, r = s.run(1, clock=ck)
    u = s.download()[3]
    a = np.abs(u)
    print(k + 1, f"t={ck.now:.6g} dt={ck.now - t0:.3e} max|h0|={a[:,0].max():.3e} max|q0|={max(a[:,3].max(), a[:,6].max()):.3e} max|slope|={a[:,[1,2,4,5,7,8]].max():.3e} n>1e6={(a>1e6).any(1).sum()}", flush=True)
