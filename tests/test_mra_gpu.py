"""Parity of the sm_100a static MRA (fm_mra_static, through the C ABI) with
the reference: bit-exact grids (leaf set, levels, indices, topography
coefficients, flags, normalised details)."""
import ctypes
import glob
import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2107_02750_b200 import scenarios as S
from test_oracle import random_flag_trees

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


def same_grid(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a.leaves(), b.leaves()))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "grid_*.npz"))),
                         ids=os.path.basename)
def test_grid_matches_reference_golden(gpu, path):
    d = np.load(path)
    dem = S.Raster(d["dem"], cellsize=float(d["cell"]))
    L, kind = int(d["L"]), int(d["kind"])
    g = gpu.grid(dem, L, float(d["eps"]), True, kind)
    lv, i, j, z = g.leaves()
    assert np.array_equal(lv, d["level"]) and np.array_equal(i, d["i"]) and np.array_equal(j, d["j"])
    assert np.array_equal(z, d["topo"])
    assert g.info()["field_norm"] == float(d["field_norm"])
    for l in range(L):
        assert np.array_equal(g.flags(l), d[f"flags{l}"]), l
        assert np.array_equal(g.dhat(l), d[f"dhat{l}"]), l


@pytest.mark.parametrize("cfg,scale,kind", [(0, 1, 0), (0, 1, 1), (1, 1, 0), (1, 1, 1), (3, 1, 0),
                                            (3, 1, 1), (4, 4, 0)])
def test_full_size_grids_bit_exact(gpu, orc, cfg, scale, kind):
    sc = S.CONFIGS[cfg](scale)
    g, o = gpu.grid(sc.dem, sc.L, sc.eps, True, kind), orc.grid(sc.dem, sc.L, sc.eps, True, kind)
    assert g.num_leaves == o.num_leaves
    assert same_grid(g, o)
    # every node within 1e-12 relative of eps is counted
    assert g.near_threshold(1e-12) == o.near_threshold(1e-12)


@pytest.mark.slow
def test_config4_grid_bit_exact(gpu, orc):
    sc = S.config4(1)
    g, o = gpu.grid(sc.dem, sc.L, sc.eps), orc.grid(sc.dem, sc.L, sc.eps)
    assert g.num_leaves == o.num_leaves
    assert same_grid(g, o)


def test_ungraded_and_edge_cases(gpu, orc):
    spike = S.spike(16, 1.0)
    for L, eps, graded in [(4, 1e-3, False), (3, 0.0, True), (3, 1e9, True), (0, 1e-3, True),
                           (2, 1e-3, True), (1, 1e-3, True)]:
        g, o = gpu.grid(spike, L, eps, graded), orc.grid(spike, L, eps, graded)
        assert same_grid(g, o), (L, eps, graded)
    # non-power-of-two raster: padding by edge replication (field.cpp:64-91), M, N > 1
    rng = np.random.default_rng(3)
    dem = S.Raster(rng.uniform(0, 5, (23, 37)), cellsize=2.0)
    for L in (0, 1, 2, 3, 5):
        g, o = gpu.grid(dem, L, 1e-3), orc.grid(dem, L, 1e-3)
        assert same_grid(g, o), L
        assert g.info() == o.info()


def test_nodata_walls(gpu, orc):
    rng = np.random.default_rng(4)
    v = rng.uniform(0, 3, (65, 65))
    v[10:14, 20:30] = -9999.0
    dem = S.Raster(v, cellsize=1.0)
    g, o = gpu.grid(dem, 6, 1e-3), orc.grid(dem, 6, 1e-3)
    assert same_grid(g, o)
    # the norm is recomputed with the wall when the DEM has nodata (k_field_norm_fix)
    assert g.info() == o.info()
    for l in range(6):
        assert np.array_equal(g.dhat(l), o.dhat(l)), l


@pytest.mark.parametrize("kind", [0, 1])
def test_details_bit_exact_all_levels(gpu, orc, kind):
    # normalised details of every node: the encode's zero-tap elision (inputs
    # finite and bounded) gives the same bits as the full filter bank
    sc = S.config1(2)
    g, o = gpu.grid(sc.dem, sc.L, sc.eps, True, kind), orc.grid(sc.dem, sc.L, sc.eps, True, kind)
    assert g.info() == o.info()
    for l in range(sc.L):
        assert np.array_equal(g.dhat(l), o.dhat(l)), l
        assert np.array_equal(g.flags(l), o.flags(l)), l


@pytest.mark.parametrize("scale", [1e306, 1.7e308])
def test_huge_elevations_keep_full_filter_bank(gpu, orc, scale):
    # |z| > 1e300: the encode keeps its zero taps (kBig); at 1.7e308 the planes
    # overflow (norm = inf, NaN details) the same way as the reference's
    rng = np.random.default_rng(5)
    v = rng.uniform(-1.0, 1.0, (33, 33)) * scale
    v[0, 0] = 0.0
    dem = S.Raster(v, cellsize=1.0)
    g, o = gpu.grid(dem, 5, 1e-3), orc.grid(dem, 5, 1e-3)
    assert all(np.array_equal(x, y, equal_nan=x.dtype.kind == "f") for x, y in zip(g.leaves(), o.leaves()))
    for l in range(5):
        assert np.array_equal(g.dhat(l), o.dhat(l), equal_nan=True), l


def test_grading_random_trees_match_oracle(gpu, orc):
    P = ctypes.POINTER(ctypes.c_uint8)
    for L, M, N in [(4, 2, 1), (5, 1, 1), (3, 3, 2)]:
        for flat in random_flag_trees(101 + L, 60, L=L, M=M, N=N):
            for graded in (0, 1):
                a, b = flat.copy(), flat.copy()
                gpu.call("grade_flags", L, M, N, graded, a.ctypes.data_as(P))
                orc.call("grade_flags", L, M, N, graded, b.ctypes.data_as(P))
                assert np.array_equal(a, b)


def test_no_cpu_fallback_symbols_loaded(gpu):
    # the product library is the CUDA build; its kernels actually launched
    before = int(gpu.fn["launch_count"]())
    gpu.grid(S.spike(16, 1.0), 4, 1e-3)
    assert int(gpu.fn["launch_count"]()) > before
