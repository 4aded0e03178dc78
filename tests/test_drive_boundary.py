"""The drop-in boundary proved with the reference's OWN batch driver.

oracle/_ref/run_drive (built by `make -C oracle ref`, oracle/run_drive.cpp)
compiles the reference's run.cpp and instantiates its drive<Sim>
(run.cpp:35-141) with fm_gpu::UniformSim / NonUniformSim / AdaptiveSim
(include/fm_gpu.hpp).  Both arms read the same scenario files (the reference's
config / ASCII raster / hydrograph formats, scenarios.emit_config) and write
through the reference's own writers, so the outputs are compared file by file:

* stats.txt: step count, leaf_count and per-level leaf counts identical;
  dt range, volumes and inflow volume within the flow tolerance;
* gauge_k.csv, depth/qx/qy_NNNN.asc: within 1e-9 rel / 1e-10 abs;
* elements.csv (config 2's required output) and grid_NNNN.nug dumps: identical
  leaf counts / leaf sets (times within the tolerance).

The horizons end inside the reference's stable window for DG2
(tests/golden horizons, scripts/golden_horizons.py).
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2107_02750_b200 import scenarios as S

EXE = os.path.join(ROOT, "oracle", "_ref", "run_drive")

# name: (scenario, end_time, output_interval, gauge_interval, gauges)
CASES = {
    "c0_static_dg2": (lambda: S.config0(4), 4.0, 2.0, 1.0, [(500.0, 1300.0), (1800.0, 1200.0)]),
    "c1_static_acc": (lambda: S.config1(8), 600.0, 200.0, 50.0, [(300.0, 2600.0), (2000.0, 2500.0)]),
    "c2_static_fv1": (lambda: S.config2(8, adaptive=False), 600.0, 300.0, 50.0, [(300.0, 2600.0)]),
    "c2_adaptive_hwfv1": (lambda: S.config2(16), 300.0, 100.0, 50.0, [(300.0, 2600.0)]),
    "c3_adaptive_mwdg2": (lambda: S.config3(32), 0.1, 0.05, 0.05, [(390.0, 2000.0)]),
    "c4_static_dg2": (lambda: S.config4(64), 14.0, 7.0, 7.0, [(60.0, 60.0), (100.0, 20.0)]),
    "c4_uniform_dg2": (lambda: S.config4(64, uniform=True), 14.0, 7.0, 7.0, [(60.0, 60.0)]),
}


def need_exe():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/run_drive not built (reference sources absent when building)")


def run(mode, cfg, out):
    return subprocess.run([EXE, mode, cfg, out], capture_output=True, text=True, timeout=600)


def stats(path):
    d = {}
    for line in open(path):
        k, v = (x.strip() for x in line.split("=", 1))
        d[k] = v
    return d


def close(a, b, rel=1e-9, abs_=1e-10):
    a, b = np.asarray(a, float), np.asarray(b, float)
    same_nan = np.isnan(a) & np.isnan(b)
    d = np.abs(a - b)
    return bool(np.all(same_nan | (d <= rel * np.abs(b)) | (d <= abs_)))


def asc(path):
    head = {}
    with open(path) as f:
        for _ in range(6):
            k, v = f.readline().split()
            head[k.lower()] = v
        vals = np.loadtxt(f, ndmin=2)
    return head, vals


def compare_dirs(a, b):
    fa, fb = sorted(os.listdir(a)), sorted(os.listdir(b))
    assert fa == fb, (fa, fb)
    sa, sb = stats(os.path.join(a, "stats.txt")), stats(os.path.join(b, "stats.txt"))
    assert sa.keys() == sb.keys(), (sa, sb)
    for k in sa:
        if k == "wall_seconds":
            continue
        if k in ("solver", "steps") or k.startswith("leaf"):
            assert sa[k] == sb[k], (k, sa[k], sb[k])
        elif k == "mass_error_rel":
            assert abs(float(sa[k]) - float(sb[k])) <= 1e-9, (k, sa[k], sb[k])
        else:
            assert close(float(sa[k]), float(sb[k])), (k, sa[k], sb[k])
    for f in fa:
        pa, pb = os.path.join(a, f), os.path.join(b, f)
        if f.endswith(".asc"):
            ha, va = asc(pa)
            hb, vb = asc(pb)
            assert ha == hb, f
            assert close(va, vb), f
        elif f.startswith("gauge_") or f == "elements.csv":
            xa = np.loadtxt(pa, delimiter=",", skiprows=1, ndmin=2)
            xb = np.loadtxt(pb, delimiter=",", skiprows=1, ndmin=2)
            assert xa.shape == xb.shape, f
            if f == "elements.csv":
                assert np.array_equal(xa[:, 1], xb[:, 1]), f  # per-adapt leaf counts
                assert close(xa[:, 0], xb[:, 0]), f
            else:
                assert close(xa, xb), f
        elif f.endswith(".nug"):
            assert open(pa).read() == open(pb).read(), f  # leaf set + topography, bit-identical
    return sa


def test_reference_arm_runs_on_cpu(tmp_path):
    """The harness itself (no GPU needed for the reference arm)."""
    need_exe()
    sc, end, oi, gi, gg = CASES["c2_adaptive_hwfv1"]
    cfg = S.emit_config(sc(), str(tmp_path / "in"), end, oi, gi, gg)
    r = run("ref", cfg, str(tmp_path / "out"))
    assert r.returncode == 0, r.stderr
    files = os.listdir(tmp_path / "out")
    for f in ("stats.txt", "elements.csv", "gauge_0.csv", "depth_0000.asc", "grid_0000.nug"):
        assert f in files
    # the reference's compare_runs of a directory with itself
    rc = subprocess.run([EXE, "compare", str(tmp_path / "out"), str(tmp_path / "out"), "0.01"],
                        capture_output=True, text=True, timeout=300)
    assert rc.returncode == 0, rc.stderr
    rows = [ln.split() for ln in rc.stdout.splitlines()]
    assert any(r[0] == "rmse" for r in rows) and any(r[0] == "extent" for r in rows)
    assert all(float(r[3]) == (0.0 if r[0] == "rmse" or r[2] == "F" else 1.0) for r in rows)


def test_gpu_arm_fails_loudly_without_a_device(tmp_path):
    need_exe()
    try:
        import ctypes
        if ctypes.CDLL("libcuda.so.1").cuInit(0) == 0:
            pytest.skip("a CUDA device is present")
    except OSError:
        pass
    sc, end, oi, gi, gg = CASES["c1_static_acc"]
    cfg = S.emit_config(sc(), str(tmp_path / "in"), end, oi, gi, gg)
    r = run("gpu", cfg, str(tmp_path / "out"))
    assert r.returncode == 1 and "cuda" in r.stderr.lower(), (r.returncode, r.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_drive_gpu_matches_reference_drive(tmp_path, name):
    need_exe()
    sc, end, oi, gi, gg = CASES[name]
    cfg = S.emit_config(sc(), str(tmp_path / "in"), end, oi, gi, gg)
    ra = run("gpu", cfg, str(tmp_path / "gpu"))
    rb = run("ref", cfg, str(tmp_path / "ref"))
    assert rb.returncode == 0, rb.stderr
    assert ra.returncode == 0, ra.stderr
    s = compare_dirs(str(tmp_path / "gpu"), str(tmp_path / "ref"))
    assert int(s["steps"]) > 0
    # the reference's own compare_runs (metrics.cpp:100-143) on the two run
    # directories: gauge RMSEs ~0, identical inundation extents
    rc = subprocess.run([EXE, "compare", str(tmp_path / "gpu"), str(tmp_path / "ref"), "0.01"],
                        capture_output=True, text=True, timeout=300)
    assert rc.returncode == 0, rc.stderr
    rows = [ln.split() for ln in rc.stdout.splitlines() if ln.strip()]
    assert rows and all(r[-1] == "0" for r in rows)  # nothing absent
    for kind, _, metric, value, _ in rows:
        v = float(value)
        if kind == "rmse":
            assert v <= 1e-9 or np.isnan(v), rows
        elif metric in ("H", "C"):
            assert v == 1.0, rows
        else:
            assert v == 0.0, rows
    if name.startswith(("c0", "c1", "c2", "c3", "c4_static")):
        assert int(s["leaf_count"]) > 0  # sim_leaf_count overloads reached (run.cpp:24-33)


@pytest.mark.gpu
def test_drive_gpu_blow_up_exit_code(tmp_path):
    """The reference DG2 dam break diverges: both arms end in
    BlowUpError -> exit code 4 with blow_up_time in stats.txt (run.cpp:97-107)."""
    need_exe()
    cfg = S.emit_config(S.config0(4), str(tmp_path / "in"), 60.0, 20.0, 10.0, [(500.0, 1300.0)])
    for mode in ("gpu", "ref"):
        r = run(mode, cfg, str(tmp_path / mode))
        assert r.returncode == 4, (mode, r.returncode, r.stderr)
        st = stats(str(tmp_path / mode / "stats.txt"))
        assert "blow_up_time" in st and float(st["blow_up_time"]) > 0
