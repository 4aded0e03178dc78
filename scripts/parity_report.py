"""Parity report: every BASELINE config at full size, the GPU (native libm, the
production path) against the unmodified reference (oracle/_ref) on the same
seeded inputs, over the stated step counts where the reference can run them
in reasonable time (or until the reference's own DG2 divergence).

For each config it records
  * the static grid (or the adaptive grid after the run): bit-identical?
  * the near-threshold census of the static detail tree (|d - eps| <= 1e-12 eps);
  * the flow state after the run: max |d| / (|ref| + tiny), and how many
    coefficients violate the north-star tolerance (1e-9 rel or 1e-10 abs);
  * for the adaptive solvers, the per-adapt element counts.

usage: python scripts/parity_report.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402
from paper_2107_02750_b200.abi import Backend, BlowUpError, isclose_flow  # noqa: E402

REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfmref.so")

# name, factory, static grid?, steps (the BASELINE count, or a stated cap)
CASES = [
    # DG2: the reference itself diverges (no slope limiter) and
    # amplifies libm ulp differences chaotically, so the DG2 horizons are short
    # ones before the divergence, plus one run to the blow-up
    ("c0_static_dg2_to_blowup", lambda: S.config0(1), True, 1000),
    ("c0_static_dg2_10", lambda: S.config0(1), True, 10),
    ("c0_static_dg2_20", lambda: S.config0(1), True, 20),
    ("c0_static_dg2_40", lambda: S.config0(1), True, 40),
    ("c0_static_dg2_60", lambda: S.config0(1), True, 60),
    ("c1_static_acc", lambda: S.config1(1), True, 2000),
    ("c2_static_fv1", lambda: S.config2(1, adaptive=False), True, 2000),
    ("c2_adaptive_hwfv1", lambda: S.config2(1), False, 200),
    ("c3_adaptive_mwdg2", lambda: S.config3(1), False, 10),
    ("c4_static_dg2", lambda: S.config4(1), True, 5),
    ("c4_uniform_dg2", lambda: S.config4(1, uniform=True), False, 5),
]


def run(be, sc, static, steps):
    t0 = time.perf_counter()
    g = be.grid(sc.dem, sc.L, sc.eps) if (static and sc.grid_mode == "nonuniform") else None
    s = be.sim(sc, g)
    info = {}
    try:
        ck, r = s.run(steps, gauge_interval=10.0)
        info["steps"] = int(r.steps)
        info["t"] = ck.now
        info["blew_up"] = False
    except BlowUpError as e:
        info["steps"] = int(e.result.steps)
        info["t"] = e.t
        info["blew_up"] = True
    info["seconds"] = time.perf_counter() - t0
    lv, i, j, u, z = s.download()
    elog = s.element_log()[1] if sc.solver in ("mwdg2", "hwfv1") else None
    near = None
    if g is not None and hasattr(g, "near_threshold"):
        try:
            near = g.near_threshold(1e-12)
        except Exception:
            near = None
    return info, (lv, i, j, u, z), elog, near


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity_report.json")
    gpu = api.lib()
    ref = Backend(REF_SO, "ref_")
    ref.fn["set_threads"](os.cpu_count() or 1)
    report = {}
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    for name, mk, static, steps in CASES:
        if only and name not in only:
            continue
        sc = mk()
        gi, ga, ge, gnear = run(gpu, sc, static, steps)
        ri, ra, re_, _ = run(ref, sc, static, steps)
        same_grid = all(np.array_equal(a, b) for a, b in zip(ga[:3], ra[:3]))
        d = {"steps_gpu": gi["steps"], "steps_ref": ri["steps"], "t_gpu": gi["t"], "t_ref": ri["t"],
             "blew_up_gpu": gi["blew_up"], "blew_up_ref": ri["blew_up"], "grid_identical": same_grid,
             "leaves": int(len(ga[0])), "gpu_s": round(gi["seconds"], 3), "ref_s": round(ri["seconds"], 3),
             "near_threshold_nodes": gnear}
        if same_grid and not (gi["blew_up"] or ri["blew_up"]):
            u, v = ga[3], ra[3]
            fin = np.isfinite(u) & np.isfinite(v)
            ok = isclose_flow(u, v)
            with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
                rel = np.abs(u - v) / (np.abs(v) + 1e-300)
            d["flow_within_tolerance"] = bool(ok.all())
            d["violations"] = int((~ok).sum())
            d["coefficients"] = int(u.size)
            d["max_abs_diff"] = float(np.max(np.abs(u - v)[fin])) if fin.any() else None
            d["max_rel_diff_where_abs_gt_1e-10"] = float(np.max(rel[fin & (np.abs(u - v) > 1e-10)])) \
                if (fin & (np.abs(u - v) > 1e-10)).any() else 0.0
            d["bit_identical_fraction"] = float(np.mean(u == v))
        if ge is not None:
            d["element_counts_identical"] = bool(np.array_equal(ge, re_))
            d["element_counts_first_diff"] = None if np.array_equal(ge, re_) else int(
                np.argmax(ge[:min(len(ge), len(re_))] != re_[:min(len(ge), len(re_))]))
        report[name] = d
        print(name, json.dumps(d), flush=True)
    with open(out_path, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
