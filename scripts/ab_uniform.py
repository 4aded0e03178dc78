"""A/B of library variants on the config-4 uniform raster (k_uni_march)."""
import json
import os
import subprocess
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, ROOT)
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
be = Backend(LIB, "fm_")
be.call("init", 0)
s = be.sim(S.config4(1, uniform=True), None)
s.run(3, gauge_interval=1e9)
s.snapshot()
prof = s.profile(4)
s.restore()
s.run(8, gauge_interval=1e9)
u = s.download()[3]
print(json.dumps({"ms": s.last_run_ms() / 8, "k": {k: v[0] / v[1] for k, v in prof.items()},
                  "hash": hashlib.sha1(u.tobytes()).hexdigest()[:12]}))
"""
for lib in sys.argv[1:]:
    code = CHILD.replace("ROOT", repr(ROOT)).replace("LIB", repr(os.path.abspath(lib)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    if out.returncode:
        print(os.path.basename(lib), "FAILED", out.stderr[-1500:])
        continue
    d = json.loads(out.stdout.strip().splitlines()[-1])
    print(f"{os.path.basename(lib):24s} {d['ms']:.3f} ms/step", " ".join(f"{k}={v:.3f}" for k, v in d["k"].items()), d["hash"])
