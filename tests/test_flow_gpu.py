"""Parity of the sm_100a flow updates (DG2 RK2, FV1, ACC on the non-uniform
leaf set; the device-resident drive loop) with the reference, through the C ABI.

Two regimes (DESIGN.md §"Parity"):
* FM_LIBM_PORTABLE: friction's cbrt and ACC's pow(h, 7/3) use the same
  deterministic +,-,*,/ routine on both sides, so every other operation can
  be, and is, compared bit-for-bit after many steps.
* FM_LIBM_NATIVE (the product default): CUDA's cbrt/pow differ from glibc's
  in the last ulp; states agree within the north_star tolerance
  (|d| <= 1e-9 |ref| or <= 1e-10) over the horizons where the reference's own
  sensitivity to a 1-ulp perturbation stays inside it.
"""
import glob
import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import FmError, isclose_flow

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")
PORTABLE = 1


def make(be, sc, libm=0):
    g = None
    if sc.grid_mode == "nonuniform" and sc.solver not in ("mwdg2", "hwfv1"):
        g = be.grid(sc.dem, sc.L, sc.eps)
    return be.sim(sc, g, libm=libm)


def lake(solver, n=64, L=6, emerged=False):
    rng = np.random.default_rng(9)
    x = np.arange(n + 1) * 5.0
    X, Y = np.meshgrid(x, x[::-1])
    z = 1.5 * np.sin(2 * np.pi * X / (n * 5) + 0.3) * np.sin(2 * np.pi * Y / (n * 5) + 1.1)
    z += 0.8 * np.exp(-((X - 120) ** 2 + (Y - 200) ** 2) / 800.0) + rng.uniform(-0.05, 0.05, z.shape)
    eta = z.max() - 0.5 if emerged else z.max() + 2.0
    return S.Scenario(name=f"lake_{solver}", dem=S.Raster(z, cellsize=5.0), solver=solver, L=L,
                      manning=0.03, initial_surface=eta)


STATIC = {
    "c0_dg2": (lambda: S.config0(2), 120),
    "c0_dg2_full": (lambda: S.config0(1), 60),
    "c1_acc": (lambda: S.config1(4), 300),
    "c2_fv1": (lambda: S.config2(4, adaptive=False), 200),
    "c4_nu_dg2": (lambda: S.config4(32), 25),
    "lake_dg2": (lambda: lake("dg2"), 100),
    "lake_fv1_emerged": (lambda: lake("fv1", emerged=True), 100),
}


@pytest.mark.parametrize("name", list(STATIC))
def test_portable_libm_lockstep_bit_exact(gpu, orc, name):
    mk, steps = STATIC[name]
    sc = mk()
    a, b = make(gpu, sc, PORTABLE), make(orc, sc, PORTABLE)
    assert np.array_equal(a.download()[3], b.download()[3])
    ca, ra = a.run(steps, gauge_interval=10.0)
    cb, rb = b.run(steps, gauge_interval=10.0)
    assert ra.steps == rb.steps == steps
    assert ca.now == cb.now and ra.dt_min == rb.dt_min and ra.dt_max == rb.dt_max
    assert ra.volume_inflow == rb.volume_inflow
    da, db = a.download(), b.download()
    for x, y in zip(da, db):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "sim_*.npz"))),
                         ids=os.path.basename)
def test_native_against_reference_golden(gpu, path):
    d = np.load(path)
    sc = S.from_arrays(d)
    if sc.solver in ("mwdg2", "hwfv1"):
        pytest.skip("adaptive: see test_adaptive_gpu.py")
    if sc.solver == "dg2" and sc.grid_mode == "uniform":
        pytest.skip("uniform raster: see test_uniform_gpu.py")
    s = make(gpu, sc)
    assert np.array_equal(s.download()[3], d["u0"])
    # the fixture's horizon lies inside the reference's stable window
    # (scripts/make_golden.py): the production libm must match there
    steps = int(d["run_steps"])
    ck, r = s.run(steps, gauge_interval=10.0)
    lv, i, j, u, z = s.download()
    assert np.array_equal(lv, d["level"]) and np.array_equal(i, d["i"]) and np.array_equal(j, d["j"])
    assert np.array_equal(z, d["z"])
    assert r.steps == int(d["steps_done"]) == steps
    ok = isclose_flow(u, d["u"])
    assert ok.all(), f"{int((~ok).sum())} coefficients outside 1e-9 rel / 1e-10 abs after {steps} steps"
    assert ck.now == pytest.approx(float(d["now"]), rel=1e-12)


@pytest.mark.parametrize("name,steps", [("c0_dg2_full", 40), ("c0_dg2", 10), ("c1_acc", 300),
                                        ("c2_fv1", 200), ("c4_nu_dg2", 15)])
def test_native_libm_within_tolerance(gpu, orc, name, steps):
    sc = STATIC[name][0]()
    a, b = make(gpu, sc), make(orc, sc)
    a.run(steps, gauge_interval=10.0)
    b.run(steps, gauge_interval=10.0)
    assert isclose_flow(a.download()[3], b.download()[3]).all()


def test_host_api_path_lockstep(gpu, orc):
    """compute_dt / step / apply_inflows driven from the host (the reference's
    drive<Sim> calls, run.cpp:80-85), portable libm: bit-exact."""
    for sc in (S.config1(8), S.config0(4)):
        a, b = make(gpu, sc, PORTABLE), make(orc, sc, PORTABLE)
        t = 0.0
        for k in range(40):
            da, db = a.compute_dt(), b.compute_dt()
            assert da == db or (np.isinf(da) and np.isinf(db))
            dt = min(da, 10.0 - (t % 10.0)) if np.isfinite(da) else 10.0
            a.step(dt)
            b.step(dt)
            assert a.apply_inflows(t, dt) == b.apply_inflows(t, dt)
            t += dt
        assert np.array_equal(a.download()[3], b.download()[3])
        assert a.volume() == b.volume()
        assert a.finite_state()[0]


def test_lake_at_rest_is_preserved(gpu):
    for solver in ("dg2", "fv1", "acc"):
        s = make(gpu, lake(solver))
        lv, i, j, u0, z = s.download()
        s.run(200, gauge_interval=10.0)
        u = s.download()[3]
        wet = u0[:, 0] > 1e-6
        eta0 = (u0[:, 0] + z[:, 0])[wet]
        assert np.abs(u[wet, 0] + z[wet, 0] - eta0).max() <= 1e-12, solver
        assert np.abs(u[:, [3, 6]]).max() <= 1e-12, solver


def test_deterministic_across_runs(gpu):
    sc = S.config0(2)
    out = []
    for _ in range(2):
        s = make(gpu, sc)
        s.run(50, gauge_interval=10.0)
        out.append(s.download()[3])
    assert np.array_equal(out[0], out[1])


def test_errors_map_to_reference_exceptions(gpu):
    v = np.zeros((17, 17))
    v[1, 2] = 1.0  # a vertex spike near the NW corner leaves a 2-level jump when ungraded
    spike = S.Raster(v)
    ungraded = gpu.grid(spike, 4, 1e-3, graded=False)
    sc = S.Scenario(name="x", dem=spike, solver="dg2", L=4, initial_depth=0.5)
    with pytest.raises(FmError) as e:  # StructureError (solver_nonuniform.cpp:566-567)
        gpu.sim(sc, ungraded)
    assert e.value.code == 5
    bad = S.Scenario(name="x", dem=spike, solver="acc", L=4,
                     inflows=[S.Inflow([0, 1], [1, 1], 0, 0, 99, 0)])
    with pytest.raises(FmError) as e:  # ConfigError (:613-615)
        gpu.sim(bad, gpu.grid(spike, 4, 1e-3))
    assert e.value.code == 2


def test_event_clock_stops_and_resumes(gpu, orc):
    sc = S.config1(8)
    a, b = make(gpu, sc, PORTABLE), make(orc, sc, PORTABLE)
    ca = cb = None
    for _ in range(6):
        if ca is None:
            ca, ra = a.run(1000, gauge_interval=30.0, output_interval=100.0, stop_at_events=True)
            cb, rb = b.run(1000, gauge_interval=30.0, output_interval=100.0, stop_at_events=True)
        else:
            ca, ra = a.run(1000, clock=ca, stop_at_events=True)
            cb, rb = b.run(1000, clock=cb, stop_at_events=True)
        assert ra.event_due == rb.event_due == 1
        assert ra.steps == rb.steps and ca.now == cb.now
        assert (ca.next_gauge, ca.next_output) == (cb.next_gauge, cb.next_output)
    assert np.array_equal(a.download()[3], b.download()[3])


def test_inline_division_is_ieee(gpu):
    """fmd::quot (reciprocal-refinement division: -DFM_INLINE_DIV builds, and
    the constant-divisor division of project4 in every build) returns exactly
    IEEE a / b on 10^8 random operand pairs, and a / (4 sqrt3) on 10^8
    random numerators; the shared-divisor division of zdiv2 (every build)
    returns exactly IEEE a / b on 10^8 pairs."""
    import ctypes
    fails = ctypes.c_int64(-1)
    for which in (0, 1, 2):
        for seed in (1, 2, 3, 4):
            gpu.call("selftest", which, 25_000_000, seed, ctypes.byref(fails))
            assert fails.value == 0, (which, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("mk", [lambda: S.config0(4), lambda: S.config0(2)], ids=["c0_s4", "c0_s2"])
def test_blow_up_reproduced_bit_exact(gpu, orc, mk):
    """The reference's DG2 has no slope limiter and the dam break diverges
    (DESIGN.md §8).  Lockstep to the end: the GPU blows up at the same step,
    the same time and the same first non-finite leaf as the oracle."""
    from paper_2107_02750_b200.abi import BlowUpError
    sc = mk()
    out = []
    for be in (gpu, orc):
        g = be.grid(sc.dem, sc.L, sc.eps)
        s = be.sim(sc, g, libm=1)
        with pytest.raises(BlowUpError) as e:
            s.run(3000, gauge_interval=10.0)
        r = e.value.result
        out.append((r.steps, r.blow_up_time, r.bad_x, r.bad_y))
    assert out[0] == out[1]


@pytest.mark.gpu
def test_native_pow73_matches_glibc(gpu):
    """ACC's pow(h, 7/3) (solver_nonuniform.cpp:367, 384): the device's
    double-double evaluation is the correctly rounded value.  glibc's pow (the
    reference's) is within 0.52 ulp and misrounds ~5 % of these arguments
    (checked against 60-digit decimal arithmetic), CUDA's pow ~25 %: the
    correctly rounded result agrees with glibc 3x more often."""
    import ctypes
    rng = np.random.default_rng(11)
    x = np.concatenate([10.0 ** rng.uniform(-6, 1.5, 400_000), rng.uniform(0.0, 2.0, 100_000)])
    x = x[x > 0]
    ref = np.power(x, 7.0 / 3.0)  # glibc pow
    out = {}
    for fn in (0, 2):
        y = np.zeros_like(x)
        gpu.call("eval_libm", fn, len(x), x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                 y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        out[fn] = np.mean(y != ref)
    assert out[0] < 0.08, out
    assert out[0] < out[2] / 3, out
    # the fp32 correction terms of the production evaluation (pow73_fast)
    # leave it equal to the all-fp64 double-double (pow73_cr) but for ties
    ys = {}
    for fn in (0, 4):
        y = np.zeros_like(x)
        gpu.call("eval_libm", fn, len(x), x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                 y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        ys[fn] = y
    assert np.mean(ys[0] != ys[4]) < 1e-4, np.mean(ys[0] != ys[4])


def test_download_into_page_locked_buffers(gpu):
    # page-locked destinations take the direct gather (no staging copy): the
    # same arrays as a download into pageable memory
    import torch

    sc = S.config0(4)
    s = make(gpu, sc, PORTABLE)
    s.run(5, gauge_interval=10.0)
    n = s.num_cells
    shapes = [((n,), torch.int32)] * 3 + [((n, 9), torch.float64), ((n, 3), torch.float64)]
    pinned = [torch.zeros(sh, dtype=dt, pin_memory=True) for sh, dt in shapes]
    got = s.download(out=[t.numpy() for t in pinned])
    ref = s.download()
    for x, y in zip(got, ref):
        assert np.array_equal(x, y)


def test_compute_dt_ignores_nan_candidates(gpu, orc):
    # compute_dt (solver_nonuniform.cpp:439-448) folds candidates with
    # std::min, so a leaf whose CFL candidate is NaN never sets dt; the device
    # warp minimum must drop such a lane too, wherever it sits in its warp
    sc = S.config0(4)
    a, b = make(gpu, sc, PORTABLE), make(orc, sc, PORTABLE)
    a.run(20, gauge_interval=10.0)
    b.run(20, gauge_interval=10.0)
    u = b.download()[3]
    wet = np.flatnonzero(u[:, 0] > 1e-3)
    assert len(wet) > 64
    # qx.c0 = NaN on every wet leaf but three: those leaves stay wet and
    # their candidates are NaN, so lane 0 of the warp holding the minimum is
    # almost surely one of them
    keep = wet[[len(wet) // 5, len(wet) // 2, (4 * len(wet)) // 5]]
    nan = np.setdiff1d(wet, keep)
    u[nan, 3] = np.nan
    a.upload(u)
    b.upload(u)
    da, db = a.compute_dt(), b.compute_dt()
    assert np.isfinite(db) and da == db


@pytest.mark.parametrize("solver,uniform", [("fv1", False), ("fv1", True), ("acc", False), ("acc", True),
                                            ("dg2", False), ("dg2", True)])
def test_second_run_resumes_from_the_current_state(gpu, orc, solver, uniform):
    """A second fm_sim_run with a fresh clock takes its first dt from the
    state the first run left (compute_dt, solver_nonuniform.cpp:427-449),
    wherever the device keeps it between steps (FV1: U* or the compact rows;
    ACC: the compact arrays).  Portable libm: bit-exact vs the oracle."""
    import dataclasses
    sc = dataclasses.replace(S.config4(8, uniform=uniform), solver=solver,
                             courant={"fv1": 0.5, "acc": 0.7, "dg2": 0.33}[solver])
    out = []
    for be in (gpu, orc):
        g = None if uniform else be.grid(sc.dem, sc.L, sc.eps)
        s = be.sim(sc, g, libm=PORTABLE)
        s.run(5, gauge_interval=10.0)
        ck, r = s.run(6, gauge_interval=10.0)
        out.append((ck.now, r.dt_min, r.dt_max, s.download()[3]))
    assert out[0][:3] == out[1][:3]
    assert np.array_equal(out[0][3], out[1][3])


@pytest.mark.parametrize("name", ["c0_dg2", "c1_acc", "c2_fv1", "uni_acc", "uni_dg2"])
def test_checkpoint_resume_continues_bit_exact(gpu, tmp_path, name):
    """fm_sim_checkpoint / fm_sim_resume (the binary restart path of SURVEY
    §5): N steps, checkpoint, M steps == a fresh sim resumed from the
    checkpoint then M steps, bit for bit (the clock is the caller's)."""
    import dataclasses
    from paper_2107_02750_b200.abi import c_clock
    sc = {"c0_dg2": lambda: S.config0(4), "c1_acc": lambda: S.config1(8),
          "c2_fv1": lambda: S.config2(8, adaptive=False),
          "uni_acc": lambda: dataclasses.replace(S.config4(64, uniform=True), solver="acc", courant=0.7),
          "uni_dg2": lambda: S.config4(64, uniform=True)}[name]()
    a = make(gpu, sc)
    ck, _ = a.run(12, gauge_interval=10.0)
    path = tmp_path / "state.fmck"
    a.checkpoint(path)
    ck2 = c_clock(ck.end_time, ck.output_interval, ck.gauge_interval, ck.now, ck.next_output, ck.next_gauge)
    a.run(10, clock=ck)
    b = make(gpu, sc)
    b.resume(path)
    b.run(10, clock=ck2)
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(x, y)


def test_resume_rejects_another_scenario_or_leaf_set(gpu, tmp_path):
    from paper_2107_02750_b200.abi import FmError
    sc = S.config0(4)
    a = make(gpu, sc)
    a.run(5, gauge_interval=10.0)
    p = tmp_path / "a.fmck"
    a.checkpoint(p)
    with pytest.raises(FmError) as e:  # another solver
        make(gpu, S.config1(8)).resume(p)
    assert e.value.code == 2
    raw = bytearray(p.read_bytes())
    hdr = 8 + 4 * 8 + 3 * 8 + 6 * 8  # CkptHeader
    raw[hdr] ^= 1  # the first leaf's level
    q = tmp_path / "b.fmck"
    q.write_bytes(bytes(raw))
    with pytest.raises(FmError) as e:  # another leaf set
        make(gpu, sc).resume(q)
    assert e.value.code == 2
    with pytest.raises(FmError) as e:
        make(gpu, sc).resume(tmp_path / "missing.fmck")
    assert e.value.code == 3


def test_manning_raster_read_in_place_when_pinned(gpu):
    """A static sim samples its Manning raster once at creation; from
    page-locked host memory it reads it in place (zero-copy) instead of
    uploading it.  Same trajectory bits as from pageable memory."""
    import dataclasses

    import torch
    sc = S.config4(16)
    g = gpu.grid(sc.dem, sc.L, sc.eps)
    a = gpu.sim(sc, g)
    t = torch.zeros(sc.manning_raster.values.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = sc.manning_raster.values
    scp = dataclasses.replace(sc, manning_raster=dataclasses.replace(sc.manning_raster, values=t.numpy()))
    b = gpu.sim(scp, g)
    del t  # the sim keeps no reference to the caller's raster
    a.run(12, gauge_interval=10.0)
    b.run(12, gauge_interval=10.0)
    assert np.array_equal(a.download()[3], b.download()[3])
