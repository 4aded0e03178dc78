"""Lockstep parity (SURVEY Appendix A rule 3(ii)): the GPU with the native libm
(the production path) against the unmodified reference (oracle/_ref), re-seeded
from the reference every K steps so the ulp-level libm drift that DG2
amplifies chaotically cannot cascade over the horizon.

Each window: both start from the reference's state and clock, both run K
steps, then
  * the grids (level, i, j) must be identical (adaptive runs regrid each step),
  * the flow state is compared against the north-star tolerance
    (1e-9 rel or 1e-10 abs, `isclose_flow`),
and the GPU is re-seeded with the reference state (fm_sim_upload).  The
free-running comparison is scripts/parity_report.py.

usage: python scripts/parity_lockstep.py [out.json] [case,case,...] [K]
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
from paper_2107_02750_b200.abi import Backend, BlowUpError, c_clock, isclose_flow  # noqa: E402

REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfmref.so")

# name, factory, static grid?, total steps, window K
CASES = [
    ("c0_static_dg2", lambda: S.config0(1), True, 400, 5),
    ("c4_static_dg2", lambda: S.config4(1), True, 200, 5),
    ("c3_adaptive_mwdg2", lambda: S.config3(1), False, 200, 5),
    ("c2_adaptive_hwfv1", lambda: S.config2(1), False, 2000, 50),
]


def copy_clock(c):
    return c_clock(c.end_time, c.output_interval, c.gauge_interval, c.now, c.next_output, c.next_gauge)


def make(be, sc, static):
    g = be.grid(sc.dem, sc.L, sc.eps) if (static and sc.grid_mode == "nonuniform") else None
    return be.sim(sc, g)


def window(s, ck, k):
    try:
        _, r = s.run(k, clock=ck)
        return int(r.steps), False
    except BlowUpError as e:
        return int(e.result.steps), True


def run_case(gpu, ref, name, mk, static, total, k):
    sc = mk()
    sg, sr = make(gpu, sc, static), make(ref, sc, static)
    ckg = c_clock(1e12, 0.0, 10.0, 0.0, 1, 1)
    ckr = copy_clock(ckg)
    out = {"window": k, "windows": 0, "steps": 0, "grid_mismatch_windows": 0, "violating_windows": 0,
           "violations": 0, "max_abs_diff": 0.0, "max_rel_diff_where_abs_gt_1e-10": 0.0,
           "bit_identical_fraction_min": 1.0, "blew_up": False}
    t0 = time.perf_counter()
    while out["steps"] < total:
        t_prev = ckr.now
        ng, bg = window(sg, ckg, k)
        nr, br = window(sr, ckr, k)
        if bg or br:
            out["blew_up"] = True
            out["blew_up_gpu"], out["blew_up_ref"] = bg, br
            out["blow_up_same_window"] = bool(bg and br and ng == nr)
            break
        if ng != nr or ng == 0:
            out["step_count_mismatch"] = [ng, nr]
            break
        out["windows"] += 1
        out["steps"] += ng
        a = sg.download()
        b = sr.download()
        if not all(np.array_equal(x, y) for x, y in zip(a[:3], b[:3])):
            out["grid_mismatch_windows"] += 1
            out["first_grid_mismatch_step"] = out.get("first_grid_mismatch_step", out["steps"])
            break
        u, v = a[3], b[3]
        ok = isclose_flow(u, v)
        nv = int((~ok).sum())
        out["violations"] += nv
        out["violating_windows"] += int(nv > 0)
        if nv:
            # where it happens: how large the reference state is, and the
            # window's mean dt (the DG2 divergence shows as |u| >> 1, dt -> 0)
            fv = np.isfinite(v)
            out.setdefault("violating", []).append(
                {"step": out["steps"], "violations": nv,
                 "max_abs_ref_state": float(np.abs(v[fv]).max()) if fv.any() else None,
                 "mean_dt": (ckr.now - t_prev) / ng})
        d = np.abs(u - v)
        fin = np.isfinite(d)
        if fin.any():
            out["max_abs_diff"] = max(out["max_abs_diff"], float(d[fin].max()))
            m = fin & (d > 1e-10)
            if m.any():
                with np.errstate(over="ignore"):
                    rel = float((d[m] / (np.abs(v[m]) + 1e-300)).max())
                out["max_rel_diff_where_abs_gt_1e-10"] = max(out["max_rel_diff_where_abs_gt_1e-10"], rel)
        out["bit_identical_fraction_min"] = min(out["bit_identical_fraction_min"], float(np.mean(u == v)))
        # re-seed: state and clock from the reference
        sg.upload(v)
        ckg = copy_clock(ckr)
    out["t_end"] = ckr.now
    out["leaves_end"] = int(len(sr.download()[0]))
    out["seconds"] = round(time.perf_counter() - t0, 1)
    out["within_tolerance"] = out["violations"] == 0 and out["grid_mismatch_windows"] == 0
    return out


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity_lockstep.json")
    only = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] != "all" else None
    gpu = api.lib()
    ref = Backend(REF_SO, "ref_")
    ref.fn["set_threads"](os.cpu_count() or 1)
    report = {}
    kk = int(sys.argv[3]) if len(sys.argv) > 3 else None
    for name, mk, static, total, k in CASES:
        if only and name not in only:
            continue
        k = kk or k
        report[name] = run_case(gpu, ref, name, mk, static, total, k)
        print(name, json.dumps(report[name]), flush=True)
        with open(out_path, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
