"""Grids from a leaf list (read_nug + make_quadgrid, quadgrid.cpp:85-110,
310-327): the path run_scenario takes for `grid_file` (run.cpp:150-153).

CPU: the oracle's import against the unmodified reference — same leaves,
same topography, same trajectories; same StructureErrors.
GPU: importing a shuffled copy of a generated grid gives that grid back
(leaves, topography) and a bit-identical simulation."""
import numpy as np
import pytest

from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import FmError


def _export(be, sc):
    g = be.grid(sc.dem, sc.L, sc.eps)
    info = g.info()
    lv, i, j, z = g.leaves()
    return g, info, lv, i, j, z


def _shuffled(lv, i, j, z, seed=1):
    p = np.random.default_rng(seed).permutation(len(lv))
    return lv[p], i[p], j[p], z[p]


def _import(be, info, lv, i, j, z):
    return be.grid_import(info["L"], info["M"], info["N"], info["R"], info["x0"], info["y0"],
                          lv, i, j, z)


@pytest.mark.parametrize("backend", ["orc", "ref"])
def test_import_round_trip_cpu(orc, ref, backend):
    be = {"orc": orc, "ref": ref}[backend]
    sc = S.config0(4)
    g, info, lv, i, j, z = _export(be, sc)
    g2 = _import(be, info, *_shuffled(lv, i, j, z))
    for a, b in zip(g.leaves(), g2.leaves()):
        assert np.array_equal(a, b)
    a = be.sim(sc, g)
    b = be.sim(sc, g2)
    a.run(10, gauge_interval=10.0)
    b.run(10, gauge_interval=10.0)
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(x, y)


def _bad_inputs(lv, i, j, z, info):
    L = info["L"]
    out = {}
    k = int(np.argmax(lv))  # a finest leaf
    i2 = i.copy()
    i2[k] = (info["M"] << int(lv[k]))  # just outside
    out["outside"] = (lv, i2, j, z)
    out["gap"] = (lv[1:], i[1:], j[1:], z[1:])
    # a duplicate of one finest leaf replacing another finest leaf: the
    # weights still tile, the leaves overlap (the GPU import rejects it)
    fin = np.nonzero(lv == lv.max())[0]
    i3, j3 = i.copy(), j.copy()
    i3[fin[1]], j3[fin[1]] = i[fin[0]], j[fin[0]]
    out["overlap"] = (lv, i3, j3, z)
    del L
    return out


def test_import_errors_match_reference(orc, ref):
    sc = S.config0(8)
    _, info, lv, i, j, z = _export(ref, sc)
    bad = _bad_inputs(lv, i, j, z, info)
    for name in ("outside", "gap"):
        for be in (orc, ref):
            with pytest.raises(FmError) as e:
                _import(be, info, *bad[name])
            assert e.value.code == 5, (name, e.value)  # StructureError


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale", [(0, 4), (4, 8), (1, 8)])
def test_gpu_import_round_trip(gpu, cfg, scale):
    sc = S.CONFIGS[cfg](scale)
    g, info, lv, i, j, z = _export(gpu, sc)
    g2 = _import(gpu, info, *_shuffled(lv, i, j, z))
    for a, b in zip(g.leaves(), g2.leaves()):
        assert np.array_equal(a, b)
    for order in (1,):
        for a, b in zip(g.leaves(order), g2.leaves(order)):
            assert np.array_equal(a, b)
    a = gpu.sim(sc, g)
    b = gpu.sim(sc, g2)
    a.run(10, gauge_interval=10.0)
    b.run(10, gauge_interval=10.0)
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(x, y)


@pytest.mark.gpu
def test_gpu_import_errors(gpu):
    sc = S.config0(8)
    _, info, lv, i, j, z = _export(gpu, sc)
    for name, args in _bad_inputs(lv, i, j, z, info).items():
        with pytest.raises(FmError) as e:
            _import(gpu, info, *args)
        assert e.value.code == 5, (name, e.value)
