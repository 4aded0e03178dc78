"""A/B timing of library variants on the bench workload (config 4 static DG2).

usage: python scripts/ab_profile.py [--scale S] [--steps N] LIB.so [LIB2.so ...]

Each library runs in its own process: MRA, sim, warm-up, then fm_sim_profile
(CUDA events per kernel family) and a timed fm_sim_run, printing one line per
variant.  Also checks that every variant ends in the same state bits.
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r"""
import hashlib, json, sys, time
sys.path.insert(0, ROOT)
from paper_2107_02750_b200.abi import Backend
from paper_2107_02750_b200 import scenarios as S
be = Backend(LIB, "fm_")
be.call("init", 0)
import dataclasses
sc = S.config4(SCALE)
if SOLVER != "dg2":
    sc = dataclasses.replace(sc, solver=SOLVER, courant={"fv1": 0.5, "acc": 0.7}[SOLVER])
g = be.grid(sc.dem, sc.L, sc.eps)
s = be.sim(sc, g)
s.run(5, gauge_interval=1e9)
s.snapshot()
prof = s.profile(STEPS)
s.restore()
ck, r = s.run(STEPS, gauge_interval=1e9)
ms = s.last_run_ms()
u = s.download()[3]
print(json.dumps({"run_ms_per_step": ms / STEPS,
                  "kernels": {k: v[0] / v[1] for k, v in prof.items()},
                  "hash": hashlib.sha1(u.tobytes()).hexdigest()[:12]}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--solver", default="dg2", choices=["dg2", "fv1", "acc"])
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    hashes = set()
    for lib in a.libs:
        code = (CHILD.replace("ROOT", repr(ROOT)).replace("LIB", repr(os.path.abspath(lib)))
                .replace("SCALE", str(a.scale)).replace("STEPS", str(a.steps))
                .replace("SOLVER", repr(a.solver)))
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if out.returncode:
            print(os.path.basename(lib), "FAILED", out.stderr[-2000:])
            continue
        d = json.loads(out.stdout.strip().splitlines()[-1])
        hashes.add(d["hash"])
        ks = " ".join(f"{k}={v:.3f}" for k, v in d["kernels"].items())
        print(f"{os.path.basename(lib):28s} run {d['run_ms_per_step']:.3f} ms/step | {ks} | {d['hash']}")
    print("identical final state across variants:", len(hashes) == 1)


if __name__ == "__main__":
    main()
