"""Uniform-raster DG2/FV1/ACC on the GPU (UniformSim, solver_uniform.cpp):
config 4's comparator, against the oracle and the reference's own
known-answer tests (test_solver_uniform.cpp)."""
import glob
import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import isclose_flow

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


def uni(solver, dem, **kw):
    sc = S.Scenario(name="u", dem=dem, solver=solver, L=0, grid_mode="uniform", **kw)
    return sc


def dambreak(cells=128, closed=False, h_left=1.0, h_right=0.5):
    # make_dambreak_1d (scenarios.cpp:91-120): flat bed, 4 rows, R = 1
    dem = S.Raster(np.zeros((5, cells + 1)), cellsize=1.0)
    x = np.arange(cells + 1, dtype=float)
    h0 = np.where(x < cells / 2.0, h_left, h_right)[None, :] * np.ones((5, 1))
    bc = (0, 0, 0, 0) if closed else (0, 1, 0, 1)
    return dem, S.Raster(h0, cellsize=1.0), bc


@pytest.mark.parametrize("solver", ["dg2", "fv1", "acc"])
@pytest.mark.parametrize("case", ["c4", "dambreak", "lake"])
def test_uniform_portable_lockstep_bit_exact(gpu, orc, solver, case):
    if case == "c4":
        sc = S.config4(64, uniform=True)
        sc.solver = solver
        steps = 25
    elif case == "dambreak":
        dem, h0, bc = dambreak(100)
        sc = uni(solver, dem, initial_depth_raster=h0, bc=bc, manning=0.03)
        steps = 150
    else:
        from test_flow_gpu import lake
        lk = lake(solver)
        sc = uni(solver, lk.dem, initial_surface=lk.initial_surface, manning=0.03)
        steps = 100
    a, b = gpu.sim(sc, None, libm=1), orc.sim(sc, None, libm=1)
    ca, ra = a.run(steps, gauge_interval=10.0)
    cb, rb = b.run(steps, gauge_interval=10.0)
    assert ra.steps == rb.steps and ca.now == cb.now and ra.dt_min == rb.dt_min
    assert np.array_equal(a.download()[3], b.download()[3])


def test_uniform_native_against_reference_golden(gpu):
    d = np.load(os.path.join(GOLD, "sim_c4_uni_s64.npz"))
    sc = S.from_arrays(d)
    s = gpu.sim(sc, None)
    assert np.array_equal(s.download()[3], d["u0"])
    steps = int(d["run_steps"])  # inside the reference's stable window (make_golden.py)
    ck, r = s.run(steps, gauge_interval=10.0)
    assert r.steps == int(d["steps_done"]) == steps
    u, z = s.download()[3:]
    assert np.array_equal(z, d["z"])
    ok = isclose_flow(u, d["u"])
    assert ok.all(), f"{int((~ok).sum())} coefficients outside 1e-9 rel / 1e-10 abs after {steps} steps"
    assert ck.now == pytest.approx(float(d["now"]), rel=1e-12)


def test_stoker_dam_break(gpu):
    """test_solver_uniform.cpp:144-170: FV1 within 5% of the depth jump, DG2 better."""
    cells, t_end, g = 400, 10.0, 9.80665
    hl, hr = 1.0, 0.5
    # exact wet-bed dam break (stoker.hpp): bisect the star depth
    cl = np.sqrt(g * hl)
    lo, hi = hr, hl
    for _ in range(200):
        hm = 0.5 * (lo + hi)
        mism = 2 * (cl - np.sqrt(g * hm)) - (hm - hr) * np.sqrt(0.5 * g * (hm + hr) / (hm * hr))
        lo, hi = (hm, hi) if mism > 0 else (lo, hm)
    hs = 0.5 * (lo + hi)
    us = 2 * (cl - np.sqrt(g * hs))
    ss = hs * us / (hs - hr)

    def exact(x):
        xi = (x - cells / 2.0) / t_end
        cm = np.sqrt(g * hs)
        return np.where(xi <= -cl, hl, np.where(xi <= us - cm, ((2 * cl - xi) / 3) ** 2 / g,
                                                np.where(xi <= ss, hs, hr)))

    errs = {}
    for solver in ("fv1", "dg2"):
        dem, h0, bc = dambreak(cells)
        s = gpu.sim(uni(solver, dem, initial_depth_raster=h0, bc=bc), None)
        s.run(100000, end_time=t_end, gauge_interval=0.0)
        u = s.download()[3].reshape(4, cells, 9)
        xc = np.arange(cells) + 0.5
        errs[solver] = np.mean(np.abs(u[2, :, 0] - exact(xc)))
    assert errs["fv1"] <= 0.05 * 0.5
    assert errs["dg2"] < errs["fv1"]


def test_radial_symmetry(gpu):
    """test_solver_uniform.cpp:262-301: 8-fold symmetry <= 1e-12."""
    n = 32
    x = np.arange(n + 1, dtype=float)
    X, Y = np.meshgrid(x, x[::-1])
    h0 = np.where((X - 16) ** 2 + (Y - 16) ** 2 < 64.0, 1.0, 0.2)
    dem = S.Raster(np.zeros((n + 1, n + 1)))
    for solver in ("dg2", "fv1"):
        s = gpu.sim(uni(solver, dem, initial_depth_raster=S.Raster(h0)), None)
        s.run(100000, end_time=2.0, gauge_interval=0.0)
        h = s.download()[3][:, 0].reshape(n, n)
        for m in (h[:, ::-1], h[::-1, :], h.T, h[::-1, ::-1].T):
            assert np.abs(h - m).max() <= 1e-12, solver


def test_closed_box_mass(gpu):
    """test_solver_uniform.cpp:129-142."""
    for solver in ("dg2", "fv1", "acc"):
        dem, h0, _ = dambreak(128, closed=True)
        s = gpu.sim(uni(solver, dem, initial_depth_raster=h0, bc=(0, 0, 0, 0),
                        manning=0.03 if solver == "acc" else 0.0), None)
        v0 = s.volume()
        s.run(500, gauge_interval=0.0)
        assert abs(s.volume() - v0) / v0 <= 1e-10, solver


def test_native_uniform_within_tolerance(gpu, orc):
    for solver, steps in (("fv1", 100), ("acc", 100), ("dg2", 20)):
        dem, h0, bc = dambreak(100)
        sc = uni(solver, dem, initial_depth_raster=h0, bc=bc, manning=0.03)
        a, b = gpu.sim(sc, None), orc.sim(sc, None)
        a.run(steps, gauge_interval=10.0)
        b.run(steps, gauge_interval=10.0)
        assert isclose_flow(a.download()[3], b.download()[3]).all(), solver
