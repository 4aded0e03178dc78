"""The CPU oracle, pinned.

1. Against the golden fixtures in tests/golden (outputs of the unmodified
   reference library, made by scripts/make_golden.py): bit-exact.
2. Against the reference's own known-answer unit tests, restated
   (proj/tests/test_wavelets.cpp, test_mra.cpp, test_quadgrid.cpp,
   test_solver_uniform.cpp).
3. Against the live reference (oracle/_ref) when it was built on this machine.
"""
import glob
import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import dptr

GOLD = os.path.join(ROOT, "tests", "golden")
G = 9.80665


def golden(pattern):
    return sorted(glob.glob(os.path.join(GOLD, pattern)))


# ---------------------------------------------------------------- golden ----
def test_point_kernels_match_golden(orc):
    d = np.load(os.path.join(GOLD, "point_kernels.npz"))
    for kind in (0, 1):
        for r in range(len(d["kids"])):
            k = np.ascontiguousarray(d["kids"][r])
            p, det, back = np.zeros(3), np.zeros(9), np.zeros(12)
            orc.fn["encode"](dptr(k), kind, dptr(p), dptr(det))
            orc.fn["decode"](dptr(p), dptr(det), kind, dptr(back))
            assert np.array_equal(p, d[f"parent{kind}"][r])
            assert np.array_equal(det, d[f"det{kind}"][r])
            assert np.array_equal(back, d[f"back{kind}"][r])
    for c, want in zip(d["hll_in"], d["hll_out"]):
        o = np.zeros(3)
        orc.fn["hll"](*[float(x) for x in c], G, 1e-6, dptr(o))
        assert np.array_equal(o, want), c
    for (h, qx, qy, n, dt), want in zip(d["fr_in"], d["fr_out"]):
        a, b = np.array([qx, 0.1, -0.2]), np.array([qy, 0.3, 0.4])
        orc.fn["friction"](h, dptr(a), dptr(b), n, G, 1e-6, dt)
        assert a[0] == want[0] and b[0] == want[1]


@pytest.mark.parametrize("path", golden("grid_*.npz"), ids=os.path.basename)
def test_static_grid_matches_golden(orc, path):
    d = np.load(path)
    dem = S.Raster(d["dem"], cellsize=float(d["cell"]))
    L, kind = int(d["L"]), int(d["kind"])
    g = orc.grid(dem, L, float(d["eps"]), True, kind)
    lv, i, j, z = g.leaves()
    assert np.array_equal(lv, d["level"]) and np.array_equal(i, d["i"]) and np.array_equal(j, d["j"])
    assert np.array_equal(z, d["topo"])
    assert g.info()["field_norm"] == float(d["field_norm"])
    for l in range(L):
        assert np.array_equal(g.flags(l), d[f"flags{l}"])
        assert np.array_equal(g.dhat(l), d[f"dhat{l}"])


@pytest.mark.parametrize("path", golden("sim_*.npz"), ids=os.path.basename)
def test_simulation_matches_golden(orc, path):
    d = np.load(path)
    sc = S.from_arrays(d)
    grid = None
    if sc.grid_mode == "nonuniform" and sc.solver not in ("mwdg2", "hwfv1"):
        grid = orc.grid(sc.dem, sc.L, sc.eps)
    s = orc.sim(sc, grid)
    assert np.array_equal(s.download()[3], d["u0"])
    ck, r = s.run(int(d["run_steps"]), gauge_interval=10.0)
    lv, i, j, u, z = s.download()
    assert np.array_equal(lv, d["level"]) and np.array_equal(i, d["i"]) and np.array_equal(j, d["j"])
    assert np.array_equal(u, d["u"])
    assert np.array_equal(z, d["z"])
    assert ck.now == float(d["now"]) and r.steps == int(d["steps_done"])
    assert r.dt_min == float(d["dt_min"]) and r.dt_max == float(d["dt_max"])
    assert r.volume_inflow == float(d["vol_in"])
    assert s.volume() == float(d["volume"])
    t, c = s.element_log()
    assert np.array_equal(t, d["elog_t"]) and np.array_equal(c, d["elog_n"])


# ------------------------------------------------- restated unit tests ----
def enc(orc, kids, kind):
    k = np.ascontiguousarray(np.asarray(kids, dtype=np.float64).reshape(12))
    p, d = np.zeros(3), np.zeros(9)
    orc.fn["encode"](dptr(k), kind, dptr(p), dptr(d))
    return p, d


def dec(orc, p, d, kind):
    out = np.zeros(12)
    orc.fn["decode"](dptr(np.ascontiguousarray(p, dtype=np.float64)),
                     dptr(np.ascontiguousarray(d, dtype=np.float64)), kind, dptr(out))
    return out.reshape(4, 3)


def test_constant_children_give_constant_parent(orc):  # test_wavelets.cpp:48-58
    for kind in (0, 1):
        p, d = enc(orc, [[2.0, 0, 0]] * 4, kind)
        assert abs(p[0] - 2.0) <= 1e-15 and abs(p[1]) <= 1e-15 and np.abs(d).max() <= 1e-15


def test_mw_planar_annihilation(orc):  # test_wavelets.cpp:60-73
    rng = np.random.default_rng(5)
    s3 = 1.7320508075688772
    for _ in range(100):
        a, bx, by = rng.uniform(-3, 3, 3)
        kids = []
        for k in range(4):
            cx = 0.25 * (1 if k & 1 else -1)
            cy = 0.25 * (1 if k & 2 else -1)
            kids.append([a + bx * cx + by * cy, bx * 0.5 / (2 * s3), by * 0.5 / (2 * s3)])
        p, d = enc(orc, kids, 0)
        assert np.abs(d).max() <= 1e-13 * max(1.0, abs(a) + abs(bx) + abs(by))
        assert p[0] == pytest.approx(a, rel=1e-13, abs=1e-13)


def test_round_trips(orc):  # test_wavelets.cpp:128-173
    rng = np.random.default_rng(29)
    for _ in range(2000):
        kids = rng.uniform(-10, 10, (4, 3))
        p, d = enc(orc, kids, 0)
        assert np.abs(dec(orc, p, d, 0) - kids).max() / 10.0 <= 1e-13
        hk = kids.copy()
        hk[:, 1:] = 0
        p, d = enc(orc, hk, 1)
        assert np.abs(dec(orc, p, d, 1)[:, 0] - hk[:, 0]).max() <= 1e-12


def test_hw_spike_details(orc):  # test_wavelets.cpp:102-113
    for s in (1.0, 2.0, 8.0):
        p, d = enc(orc, [[s, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]], 1)
        assert p[0] == pytest.approx(s / 4) and abs(d[0]) == pytest.approx(s / 4)
        assert abs(d[3]) == pytest.approx(s / 4) and abs(d[6]) == pytest.approx(s / 4)


def test_hll_known_answers(orc):  # test_solver_uniform.cpp:55-81
    o = np.zeros(3)
    orc.fn["hll"](0, 0, 0, 0, 0, 0, G, 1e-6, dptr(o))
    assert (o == 0).all()
    orc.fn["hll"](1.0, 0, 0, 1.0, 0, 0, G, 1e-6, dptr(o))
    assert abs(o[0]) <= 1e-15 and o[1] == pytest.approx(0.5 * G, rel=1e-14)
    orc.fn["hll"](1.0, 10.0, 2.0, 0.8, 7.2, 0.8, G, 1e-6, dptr(o))
    assert o[0] == pytest.approx(10.0) and o[1] == pytest.approx(100 + 0.5 * G)
    assert o[2] == pytest.approx(20.0)


def test_friction_formula(orc):  # test_solver_uniform.cpp:355-367
    qx, qy = np.array([0.5, 0, 0]), np.array([-0.2, 0, 0])
    h, n, dt = 0.4, 0.05, 2.0
    u, v = 0.5 / h, -0.2 / h
    denom = 1.0 + dt * G * n * n * np.hypot(u, v) / h ** (4.0 / 3.0)
    orc.fn["friction"](h, dptr(qx), dptr(qy), n, G, 1e-6, dt)
    assert qx[0] == pytest.approx(0.5 / denom, rel=1e-13)
    orc.fn["friction"](1e-9, dptr(qx), dptr(qy), n, G, 1e-6, dt)
    assert qx[0] == 0.0


def test_portable_cbrt_is_accurate(orc):
    xs = np.geomspace(1e-7, 50, 2000)
    got = np.array([orc.fn["pcbrt"](float(x)) for x in xs])
    assert np.max(np.abs(got - np.cbrt(xs)) / np.cbrt(xs)) < 5e-16


def random_flag_trees(seed, count=100, L=4, M=2, N=1):  # test_mra.cpp:213-248
    rng = np.random.default_rng(seed)
    for _ in range(count):
        levels = [np.zeros((N << l) * (M << l), np.uint8) for l in range(L)]
        for _ in range(6):
            l = int(rng.integers(0, L))
            w, h = M << l, N << l
            levels[l][int(rng.integers(0, h)) * w + int(rng.integers(0, w))] = 1
        yield np.concatenate(levels)


def flags_graded(flat, L, M, N):  # detail_tree.cpp:76-95
    levels, at = [], 0
    for l in range(L):
        n = (N << l) * (M << l)
        levels.append(flat[at:at + n].reshape(N << l, M << l))
        at += n
    for l in range(1, L):
        h, w = levels[l].shape
        for j, i in zip(*np.nonzero(levels[l])):
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                ni, nj = i + di, j + dj
                if 0 <= ni < w and 0 <= nj < h and not levels[l - 1][nj // 2, ni // 2]:
                    return False
    return True


def u8p(a):
    import ctypes
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def test_grading_random_trees(orc):
    for flat in random_flag_trees(77):
        f = flat.copy()
        orc.call("grade_flags", 4, 2, 1, 1, u8p(f))
        assert flags_graded(f, 4, 2, 1)
        g2 = f.copy()
        orc.call("grade_flags", 4, 2, 1, 1, u8p(g2))
        assert np.array_equal(f, g2)  # idempotent


def gather_grade(flat, L, M, N):
    """The gather form of grading the device runs (mra.cu k_grade_count),
    applied WITHOUT a prior ancestor closure, bottom-up: G(l) = F(l) | any
    child G(l+1) | any G(l+1) among the 8 ring nodes around the child block."""
    levels, at = [], 0
    for l in range(L):
        n = (N << l) * (M << l)
        levels.append(flat[at:at + n].reshape(N << l, M << l).copy())
        at += n
    for l in range(L - 2, -1, -1):
        fine = levels[l + 1]
        h, w = fine.shape
        pad = np.zeros((h + 2, w + 2), np.uint8)
        pad[1:-1, 1:-1] = fine
        G = levels[l].copy()
        for j in range(N << l):
            for i in range(M << l):
                cj, ci = 2 * j + 1, 2 * i + 1  # the child block in padded coordinates
                kids = pad[cj:cj + 2, ci:ci + 2].any()
                ring = (pad[cj:cj + 2, ci - 1].any() or pad[cj:cj + 2, ci + 2].any()
                        or pad[cj - 1, ci:ci + 2].any() or pad[cj + 2, ci:ci + 2].any())
                G[j, i] |= bool(kids or ring)
        levels[l] = G
    return np.concatenate([x.ravel() for x in levels])


def test_closure_subsumed_by_gather_grading(orc):
    """adaptive.cu skips buffer_ring's ancestor closure before grading:
    grading in gather form on the UNCLOSED flags equals the reference's
    closure + grade_flags (the oracle, pinned to the reference)."""
    for L, M, N in [(4, 2, 1), (5, 1, 1), (4, 3, 2)]:
        for flat in random_flag_trees(301 + L, 40, L=L, M=M, N=N):
            a = flat.copy()
            orc.call("grade_flags", L, M, N, 1, u8p(a))
            assert np.array_equal(gather_grade(flat, L, M, N), a)


def test_grid_properties(orc):  # test_mra.cpp:61-211
    flat = S.Raster(np.full((17, 17), 4.0))
    g = orc.grid(flat, 2, 1e-3)
    assert g.num_leaves == 16 and set(g.leaves()[0]) == {0}
    spike = S.spike(16, 1.0)
    g = orc.grid(spike, 4, 1e-3)
    lv, i, j, _ = g.leaves()
    assert 1 < g.num_leaves < 256
    assert all(abs(a - 8) <= 2 and abs(b - 8) <= 2 for l, a, b in zip(lv, i, j) if l == 4)
    g0 = orc.grid(spike, 3, 0.0, False)
    assert g0.num_leaves == 256  # eps = 0 flags everything (M = N = 2 blocks of 8x8)
    gh = orc.grid(spike, 3, 1e9, False)
    assert gh.num_leaves == 4  # the M x N coarsest grid


# ------------------------------------------------------- live reference ----
def test_grading_matches_reference(orc, ref):
    import ctypes
    P = ctypes.POINTER(ctypes.c_uint8)
    for flat in random_flag_trees(11, 50, L=5, M=3, N=2):
        a, b = flat.copy(), flat.copy()
        orc.call("grade_flags", 5, 3, 2, 1, a.ctypes.data_as(P))
        ref.call("grade_flags", 5, 3, 2, 1, b.ctypes.data_as(P))
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg,scale", [(0, 2), (1, 8), (3, 16), (4, 32)])
def test_grid_matches_reference_live(orc, ref, cfg, scale):
    sc = S.CONFIGS[cfg](scale)
    a = orc.grid(sc.dem, sc.L, sc.eps).leaves()
    b = ref.grid(sc.dem, sc.L, sc.eps).leaves()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("name", ["c0", "c1", "c2fv1", "c4uni"])
def test_sim_matches_reference_live(orc, ref, name):
    sc = {"c0": S.config0(4), "c1": S.config1(8), "c2fv1": S.config2(8, adaptive=False),
          "c4uni": S.config4(64, uniform=True)}[name]
    out = []
    for be in (orc, ref):
        g = be.grid(sc.dem, sc.L, sc.eps) if sc.grid_mode == "nonuniform" else None
        s = be.sim(sc, g)
        s.run(25, gauge_interval=10.0)
        out.append(s.download()[3])
    assert np.array_equal(out[0], out[1])


def test_blow_up_matches_reference(orc, ref):
    """The reference's own divergence on the dam break: the
    oracle blows up at the same step, time and first non-finite leaf."""
    from paper_2107_02750_b200.abi import BlowUpError
    sc = S.config0(4)
    out = []
    for be in (orc, ref):
        g = be.grid(sc.dem, sc.L, sc.eps)
        s = be.sim(sc, g)
        with pytest.raises(BlowUpError) as e:
            s.run(3000, gauge_interval=10.0)
        r = e.value.result
        out.append((r.steps, r.blow_up_time, r.bad_x, r.bad_y))
    assert out[0] == out[1]
    assert out[0][0] < 3000
