"""The reference's remaining known-answer tests, restated
against the GPU path through the C ABI:

* ACC: friction-only decay of a face discharge between level surfaces, flow
  down the surface gradient from rest (test_solver_uniform.cpp:303-326), the
  Manning fixed point within 1 % (:328-338) with the device's pow(h, 7/3);
* the mirrored dam break gives the mirrored solution (:180-198);
* compute_dt follows the CFL rule and halving the cell size halves dt
  (:200-222);
* reflective and open boundaries keep still water still (:340-353);
* convergence on a smooth hump (:369-429): the reference itself misses its
  bar (DG2 >= 1.8, FV1 >= 0.8) on this case, so the GPU is pinned to the
  reference's fields and order instead.
"""
import numpy as np
import pytest

from paper_2107_02750_b200 import scenarios as S

pytestmark = pytest.mark.gpu
G = 9.80665


def dambreak(cells=100, rows=4, R=1.0, h_left=1.0, h_right=0.5, closed=False):
    # make_dambreak_1d (scenarios.cpp:91-120): flat bed, x_dam = cells R / 2
    dem = S.Raster(np.zeros((rows + 1, cells + 1)), cellsize=R)
    x = np.arange(cells + 1, dtype=float) * R
    h0 = np.where(x < cells * R / 2.0, h_left, h_right)[None, :] * np.ones((rows + 1, 1))
    return dem, S.Raster(h0, cellsize=R), (0, 0, 0, 0) if closed else (0, 1, 0, 1)


def uni(solver, dem, **kw):
    return S.Scenario(name="u", dem=dem, solver=solver, L=0, grid_mode="uniform", **kw)


def test_acc_face_discharge_decays_between_level_surfaces(gpu):
    dem, h0, bc = dambreak(h_left=1.0, h_right=1.0)
    s = gpu.sim(uni("acc", dem, initial_depth_raster=h0, bc=bc, manning=0.05), None)
    qx, _ = s.acc_faces()
    qx[1, 50] = 0.4  # face = 1 * (nx + 1) + 50
    s.acc_faces(set_x=qx)
    s.step(0.5)
    q = s.acc_faces()[0][1, 50]
    assert 0.0 < q < 0.4, q


def test_acc_discharge_flows_down_the_surface_gradient(gpu):
    dem, h0, bc = dambreak()
    s = gpu.sim(uni("acc", dem, initial_depth_raster=h0, bc=bc, manning=0.05), None)
    s.step(0.1)
    assert s.acc_faces()[0][1, 50] > 0.0  # higher water west: eastward


def test_acc_fixed_point_matches_manning(gpu):
    """The face update iterated with a frozen surface slope converges to the
    Manning discharge h^(5/3) sqrt(S0) / n within 1 %; h^(7/3) is the device's
    production evaluation (FM_LIBM_NATIVE)."""
    import ctypes
    g, n, h, S0, R, dt = G, 0.03, 0.8, 1e-3, 10.0, 1.0
    x = np.array([h])
    p = np.zeros(1)
    gpu.call("eval_libm", 0, 1, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
             p.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert p[0] == pytest.approx(h ** (7.0 / 3.0), rel=1e-15)
    q = 0.0
    for _ in range(20000):
        q = (q - g * h * dt * (-S0 * R) / R) / (1.0 + g * dt * n * n * abs(q) / p[0])
    assert q == pytest.approx(h ** (5.0 / 3.0) * np.sqrt(S0) / n, rel=0.01)


def test_mirrored_dam_break_gives_the_mirrored_solution(gpu):
    dem, h0, bc = dambreak(128)
    hm = S.Raster(h0.values[:, ::-1].copy(), cellsize=1.0)
    a = gpu.sim(uni("fv1", dem, initial_depth_raster=h0, bc=bc), None)
    b = gpu.sim(uni("fv1", dem, initial_depth_raster=hm, bc=bc), None)
    for s in (a, b):
        s.run(100000, end_time=5.0, gauge_interval=0.0)
    ha = a.download()[3][:, 0].reshape(4, 128)
    hb = b.download()[3][:, 0].reshape(4, 128)
    assert np.allclose(ha, hb[:, ::-1], rtol=1e-12, atol=0.0)


def test_compute_dt_follows_the_cfl_rule(gpu):
    dem, h0, bc = dambreak(100)
    s = gpu.sim(uni("fv1", dem, initial_depth_raster=h0, bc=bc, courant=0.5), None)
    u = np.zeros((s.num_cells, 9))
    u[1 * 100 + 50, 0] = 1.0  # one wet cell of depth 1
    s.upload(u)
    assert s.compute_dt() * 10.0 == pytest.approx(0.5 * 10.0 / np.sqrt(G), rel=1e-12)
    s.upload(np.zeros((s.num_cells, 9)))
    assert s.compute_dt() == np.inf


def test_halving_the_cell_size_halves_dt(gpu):
    da, ha, bc = dambreak(100, R=1.0)
    db, hb, _ = dambreak(200, R=0.5)
    a = gpu.sim(uni("fv1", da, initial_depth_raster=ha, bc=bc), None)
    b = gpu.sim(uni("fv1", db, initial_depth_raster=hb, bc=bc), None)
    assert b.compute_dt() == pytest.approx(0.5 * a.compute_dt(), rel=1e-12)


@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (0, 1, 0, 1)], ids=["reflective", "open"])
def test_still_water_with_reflective_and_open_boundaries(gpu, bc):
    dem, h0, _ = dambreak(100, h_left=0.6, h_right=0.6)
    s = gpu.sim(uni("dg2", dem, initial_depth_raster=h0, bc=bc), None)
    v0 = s.volume()
    s.run(50, gauge_interval=0.0)
    assert abs(s.volume() - v0) <= 1e-12 * v0
    assert np.abs(s.download()[3][:, 3]).max() <= 1e-13


def _hump_run(be, cells, solver):
    x = np.arange(cells + 1) * (96.0 / cells)
    X, Y = np.meshgrid(x, x[::-1])
    h0 = 1.0 + 0.2 * np.exp(-((X - 40.0) ** 2 + (Y - 40.0) ** 2) / 100.0)
    dem = S.Raster(np.zeros((cells + 1, cells + 1)), cellsize=96.0 / cells)
    s = be.sim(uni(solver, dem, initial_depth_raster=S.Raster(h0, cellsize=96.0 / cells)), None)
    u = s.download()[3]
    u[:, 3:6] = 0.3 * u[:, 0:3]  # qx = 0.3 h, qy = 0.3 h: diagonal advection
    u[:, 6:9] = 0.3 * u[:, 0:3]
    s.upload(u)
    s.run(10 ** 6, end_time=3.0, gauge_interval=0.0)
    return s.download()[3][:, 0].reshape(cells, cells)


def _order(h48, h96, h192):
    def l1(coarse, fine):
        avg = 0.25 * (fine[0::2, 0::2] + fine[1::2, 0::2] + fine[0::2, 1::2] + fine[1::2, 1::2])
        return np.abs(coarse - avg).mean()

    return float(np.log2(l1(h48, h96) / l1(h96, h192)))


@pytest.mark.parametrize("solver,ref_threshold", [("dg2", 1.8), ("fv1", 0.8)])
def test_convergence_order_on_a_smooth_hump(gpu, ref, solver, ref_threshold):
    """test_solver_uniform.cpp:369-429 asks for order >= 1.8 (DG2) / 0.8 (FV1).
    The UNMODIFIED reference does not meet its own bar on this case (order
    0.48 DG2, 0.42 FV1, measured with oracle/_ref): the
    reflective 96 m box returns the advected hump's waves within t = 3 s.  So
    the restated test pins the GPU to the reference: the same fields at every
    resolution (no friction: no libm in the path) and the same order."""
    hg = [_hump_run(gpu, c, solver) for c in (48, 96, 192)]
    hr = [_hump_run(ref, c, solver) for c in (48, 96, 192)]
    for a, b in zip(hg, hr):
        assert np.allclose(a, b, rtol=1e-9, atol=1e-10)
    og, orf = _order(*hg), _order(*hr)
    assert og == pytest.approx(orf, abs=1e-6)
    assert orf < ref_threshold  # the reference's own shortfall, reproduced
