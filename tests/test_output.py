"""Output sampling — the gauge samples and raster dumps of drive<Sim>
(run.cpp:56-74): Sim::sample_gauge (solver_nonuniform.cpp:489-506,
solver_uniform.cpp:480-498) and depth/qx/qy_raster (sample_to_raster,
quadgrid.cpp:262-285; field_raster, solver_uniform.cpp:501-520).

CPU: the oracle's restatement against the unmodified reference, bit-exact.
GPU: the device kernels against the oracle on the same trajectory, bit-exact
(portable libm, so the states being sampled are identical)."""
import numpy as np
import pytest

from paper_2107_02750_b200 import scenarios as S

CASES = {
    "c0_dg2": (lambda: S.config0(4), 12),
    "c1_acc": (lambda: S.config1(8), 12),
    "c2_fv1": (lambda: S.config2(8, adaptive=False), 12),
    "c2_hwfv1": (lambda: S.config2(8), 8),
    "c3_mwdg2": (lambda: S.config3(16), 6),
    "c4_uniform_dg2": (lambda: S.config4(64, uniform=True), 8),
}


def gauge_points(sc, n=64, seed=5):
    """Random points over (and slightly beyond) the domain, plus points on
    element edges and corners, where floor() and the containing-leaf search
    must agree with the reference."""
    dem = sc.dem
    w = (dem.ncols - 1) * dem.cellsize
    h = (dem.nrows - 1) * dem.cellsize
    rng = np.random.default_rng(seed)
    x = rng.uniform(dem.xll - 0.05 * w, dem.xll + 1.05 * w, n)
    y = rng.uniform(dem.yll - 0.05 * h, dem.yll + 1.05 * h, n)
    k = np.arange(0, 9)
    ex = dem.xll + k * (w / 8)
    ey = dem.yll + k[::-1] * (h / 8)
    return np.concatenate([x, ex, [dem.xll, dem.xll + w]]), np.concatenate([y, ey, [dem.yll + h, dem.yll]])


def _make(be, sc, libm=None):
    g = be.grid(sc.dem, sc.L, sc.eps) if (sc.solver in ("dg2", "fv1", "acc")
                                          and sc.grid_mode == "nonuniform") else None
    return be.sim(sc, g) if libm is None else be.sim(sc, g, libm=libm)


def _outputs(s, sc):
    x, y = gauge_points(sc)
    return s.raster_shape(), [s.raster(w) for w in range(3)], s.sample_gauges(x, y)


def _compare(a, b):
    sa, ra, ga = a
    sb, rb, gb = b
    assert sa == sb
    for p, q in zip(ra, rb):
        assert p.shape == (sa["nrows"], sa["ncols"])
        assert np.array_equal(p, q)
    assert np.array_equal(ga, gb)


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_outputs_match_reference(orc, ref, name):
    mk, steps = CASES[name]
    sc = mk()
    out = []
    for be in (orc, ref):
        s = _make(be, sc)
        s.run(steps, gauge_interval=10.0)
        out.append(_outputs(s, sc))
    _compare(out[0], out[1])


def test_oracle_raster_of_fresh_lake(orc):
    """A lake at rest: depth raster = eta - z at fine-cell centres on a DG2
    grid, exactly c0 + planes; qx = qy = 0 everywhere."""
    sc = S.config0(8)
    sc.initial_depth_raster = None
    sc.initial_surface = 50.0
    s = _make(orc, sc)
    r = [s.raster(w) for w in range(3)]
    assert (r[0] >= 0).all() and not r[1].any() and not r[2].any()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_outputs_match_oracle(gpu, orc, name):
    mk, steps = CASES[name]
    sc = mk()
    out = []
    for be in (gpu, orc):
        s = _make(be, sc, libm=1)
        s.run(steps, gauge_interval=10.0)
        out.append(_outputs(s, sc))
    _compare(out[0], out[1])


@pytest.mark.gpu
def test_gpu_raster_full_size_c4(gpu):
    """The config-4 fine raster (8192^2) straight from the static grid: every
    fine cell finds a leaf, the depth field is the exact leaf plane there."""
    sc = S.config4(1)
    g = gpu.grid(sc.dem, sc.L, sc.eps)
    sc.initial_surface = None
    s = gpu.sim(sc, g)
    s.run(4, gauge_interval=10.0)
    r = s.raster(0)
    assert r.shape == (8192, 8192) and np.isfinite(r).all()
    lv, i, j, u, z = s.download()
    # coarsest leaf: its block of fine cells carries its plane
    k = int(np.argmin(lv))
    L = sc.L
    f = 1 << (L - int(lv[k]))
    blk = r[8192 - (int(j[k]) + 1) * f: 8192 - int(j[k]) * f, int(i[k]) * f: (int(i[k]) + 1) * f]
    assert blk.shape == (f, f)
    c0, cx, cy = u[k, 0:3]
    if cx == 0 and cy == 0:
        assert (blk == c0).all()


def _rasters(seed, n=(37, 53), nodata_frac=0.05):
    rng = np.random.default_rng(seed)
    a = rng.exponential(0.05, n)
    b = a + rng.normal(0, 0.02, n)
    a[rng.random(n) < nodata_frac] = -9999.0
    b[rng.random(n) < nodata_frac] = -9999.0
    return S.Raster(a, cellsize=2.0), S.Raster(b, cellsize=2.0)


@pytest.mark.parametrize("wet", [0.0, 0.01, 0.05, 1e9])
def test_extent_metrics_oracle_matches_reference(orc, ref, wet):
    t, r = _rasters(3)
    ca, ra = orc.extent_metrics(t, r, wet)
    cb, rb = ref.extent_metrics(t, r, wet)
    assert np.array_equal(ca, cb) and np.array_equal(ra, rb)


def test_extent_metrics_geometry_mismatch(orc, ref):
    from paper_2107_02750_b200.abi import FmError
    t, r = _rasters(4)
    r2 = S.Raster(r.values, cellsize=1.0)
    for be in (orc, ref):
        with pytest.raises(FmError) as e:
            be.extent_metrics(t, r2, 0.01)
        assert e.value.code == 3


@pytest.mark.gpu
@pytest.mark.parametrize("wet", [0.0, 0.01, 0.05, 1e9])
def test_extent_metrics_gpu_matches_oracle(gpu, orc, wet):
    t, r = _rasters(5, n=(1031, 517))
    ca, ra = gpu.extent_metrics(t, r, wet)
    cb, rb = orc.extent_metrics(t, r, wet)
    assert np.array_equal(ca, cb) and np.array_equal(ra, rb)
