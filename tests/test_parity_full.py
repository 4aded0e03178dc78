"""Full-size parity of the production path (native libm) against the
UNMODIFIED reference library (oracle/_ref/libfmref.so, built from the
reference's own sources; it travels to the GPU box as a prebuilt file), at
BASELINE.json's full config sizes.

* Free-running: C1 static ACC and C2 static FV1 for their full 2000 steps.
* Lockstep (SURVEY App. A rule 3(ii)): both sides run K steps from the
  reference's state and clock, every window is compared (grids bit-identical,
  flow within 1e-9 rel / 1e-10 abs), then the GPU is re-seeded from the
  reference.  The re-seed bounds the reference DG2's chaotic amplification of
  1-ulp cbrt differences; the horizons end before the
  reference's own state diverges (profiles/parity_lockstep_r1.json).
"""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import isclose_flow

sys.path.insert(0, os.path.join(ROOT, "scripts"))
import parity_lockstep as PL  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def ref_mt(ref):
    ref.fn["set_threads"](os.cpu_count() or 1)
    return ref


@pytest.mark.parametrize("name,mk,steps", [
    ("c1_static_acc", lambda: S.config1(1), 2000),
    ("c2_static_fv1", lambda: S.config2(1, adaptive=False), 2000),
])
def test_free_running_full_length(gpu, ref_mt, name, mk, steps):
    sc = mk()
    a = gpu.sim(sc, gpu.grid(sc.dem, sc.L, sc.eps))
    b = ref_mt.sim(sc, ref_mt.grid(sc.dem, sc.L, sc.eps))
    ca, ra = a.run(steps, gauge_interval=10.0)
    cb, rb = b.run(steps, gauge_interval=10.0)
    assert ra.steps == rb.steps == steps
    assert ca.now == pytest.approx(cb.now, rel=1e-9)
    da, db = a.download(), b.download()
    for x, y in zip(da[:3], db[:3]):
        assert np.array_equal(x, y)
    assert np.array_equal(da[4], db[4])
    ok = isclose_flow(da[3], db[3])
    assert ok.all(), f"{int((~ok).sum())} of {ok.size} coefficients outside tolerance after {steps} steps"


@pytest.mark.parametrize("name,mk,static,total,k", [
    ("c4_static_dg2", lambda: S.config4(1), True, 20, 1),
    ("c0_static_dg2", lambda: S.config0(1), True, 100, 1),
    ("c3_adaptive_mwdg2", lambda: S.config3(1), False, 50, 1),
    ("c2_adaptive_hwfv1", lambda: S.config2(1), False, 200, 50),
])
def test_lockstep_full_size(gpu, ref_mt, name, mk, static, total, k):
    out = PL.run_case(gpu, ref_mt, name, mk, static, total, k)
    assert out["steps"] == total and not out["blew_up"], out
    assert out["grid_mismatch_windows"] == 0, out
    assert out["violations"] == 0, out
