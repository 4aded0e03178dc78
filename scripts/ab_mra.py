"""A/B of static-MRA library variants on config 4: min kernel time over
repetitions and a hash of the leaf set and every level's details.

usage: python scripts/ab_mra.py LIB.so [LIB2.so ...]
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
be = Backend(LIB, "fm_")
be.call("init", 0)
sc = S.config4(1)
dem_d = torch.from_numpy(np.ascontiguousarray(sc.dem.values)).cuda()
torch.cuda.synchronize()
ts = []
for rep in range(6):
    g = be.grid(sc.dem, sc.L, sc.eps, device_ptr=dem_d.data_ptr())
    ts.append(g.timing()[0])
    if rep < 5:
        del g
h = hashlib.sha1()
for a in g.leaves():
    h.update(a.tobytes())
for l in range(sc.L):
    h.update(g.dhat(l).tobytes())
print(json.dumps({"min_ms": min(ts), "ms": ts, "hash": h.hexdigest()[:12]}))
"""


def main():
    hashes = set()
    for lib in sys.argv[1:]:
        code = CHILD.replace("ROOT", repr(ROOT)).replace("LIB", repr(os.path.abspath(lib)))
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if out.returncode:
            print(os.path.basename(lib), "FAILED", out.stderr[-1500:])
            continue
        d = json.loads(out.stdout.strip().splitlines()[-1])
        hashes.add(d["hash"])
        print(f"{os.path.basename(lib):24s} min {d['min_ms']:.3f} ms  {[round(t, 2) for t in d['ms']]}  {d['hash']}")
    print("identical grids and details across variants:", len(hashes) == 1)


if __name__ == "__main__":
    main()
