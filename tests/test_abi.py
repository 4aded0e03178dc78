"""The drop-in boundary: libfm_gpu.so loads and exports exactly the C ABI
declared in include/fm_gpu.h, and refuses to run without a CUDA device
(no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import GPU_SO, ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "fm_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for required in ["fm_mra_static", "fm_sim_create", "fm_sim_compute_dt", "fm_sim_step",
                     "fm_sim_apply_inflows", "fm_sim_adapt", "fm_sim_volume", "fm_sim_finite",
                     "fm_sim_download", "fm_sim_upload", "fm_sim_run", "fm_last_error"]:
        assert required in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(GPU_SO), "run __graft_entry__.build() first"
    out = subprocess.run(["nm", "-D", "--defined-only", GPU_SO], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (fm_[a-z_0-9]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_fails_loudly_without_gpu():
    lib = ctypes.CDLL(GPU_SO)
    lib.fm_last_error.restype = ctypes.c_char_p
    n = ctypes.c_int(0)
    has_gpu = False
    try:
        cudart = ctypes.CDLL("libcuda.so.1")
        has_gpu = cudart.cuInit(0) == 0
    except OSError:
        pass
    if has_gpu:
        pytest.skip("a CUDA device is present")
    st = lib.fm_init(0)
    assert st == 7, (st, lib.fm_last_error())
    assert b"CUDA" in lib.fm_last_error() or b"cuda" in lib.fm_last_error()
    del n


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", GPU_SO], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_rmse_restates_metrics_cpp():
    """fm_rmse (host side of the library) against a plain restatement of
    metrics.cpp:20-46 in the same operation order: bit-exact."""
    import bisect
    import numpy as np
    lib = ctypes.CDLL(GPU_SO)
    P = ctypes.POINTER(ctypes.c_double)
    lib.fm_rmse.argtypes = [P, P, ctypes.c_int64, P, P, ctypes.c_int64, P]
    rng = np.random.default_rng(2)
    tt = np.cumsum(rng.uniform(0.5, 3.0, 200))
    tv = rng.normal(size=200)
    rt = np.cumsum(rng.uniform(0.2, 2.0, 300)) + 5.0
    rv = rng.normal(size=300)

    def interp(t):
        hi = bisect.bisect_right(list(tt), t)
        if hi == 0:
            return tv[0]
        if hi == len(tt):
            return tv[-1]
        t0, t1 = tt[hi - 1], tt[hi]
        w = (t - t0) / (t1 - t0)
        return tv[hi - 1] + w * (tv[hi] - tv[hi - 1])

    lo, hi = max(tt[0], rt[0]), min(tt[-1], rt[-1])
    s, n = 0.0, 0
    for t, v in zip(rt, rv):
        if t < lo or t > hi:
            continue
        d = interp(t) - v
        s += d * d
        n += 1
    want = float(np.sqrt(s / n))
    out = ctypes.c_double()
    c = [np.ascontiguousarray(a) for a in (tt, tv, rt, rv)]
    st = lib.fm_rmse(*(a.ctypes.data_as(P) for a in c[:2]), len(tt), *(a.ctypes.data_as(P) for a in c[2:]),
                     len(rt), ctypes.byref(out))
    assert st == 0 and out.value == want
    st = lib.fm_rmse(c[0].ctypes.data_as(P), c[1].ctypes.data_as(P), 0, c[2].ctypes.data_as(P),
                     c[3].ctypes.data_as(P), len(rt), ctypes.byref(out))
    assert st == 3  # empty series: ParseError class
