"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

The paper's DEMs are access-restricted and absent, so
every configuration is generated here, on the host, in memory, once; the
CUDA path, the CPU oracle and the reference library all consume the same
arrays.  Choices BASELINE.json leaves open are fixed here and recorded in
DESIGN.md §"Synthetic inputs":

* a DEM of n x n cells is an (n+1) x (n+1) VERTEX raster, row 0 north,
  xll = yll = 0 (field.hpp:93-98, scenarios.cpp:16-25), so M = N = 1 at L = log2 n;
* bumps: centres U[0, n dx]^2, amplitude U[0.5, 3] m, sigma U[20, 80] m,
  z += A exp(-r^2 / 2 sigma^2), evaluated inside a +-5 sigma window;
* channel: -2 m on vertices within 1.5 cells of
  y = (n/2 + (40 n / 256) sin(2 pi x / (n dx))) dx   (C0: y = 128 + 40 sin(2 pi x / 2560) cells);
* RNG: numpy PCG64 seeded SEED + k (k = 0 C0, 1 C1/C2, 2 C3, 3 C4).

`scale` shrinks a configuration for the CPU-sized parity tests: n -> n/scale,
L -> L - log2(scale), cell size and physics unchanged, bump count scaled by
1/scale^2 (at least 2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED = 20210706  # arXiv 2107.02750 submission month, recorded in DESIGN.md

SOLVERS = {"dg2": 0, "fv1": 1, "acc": 2, "mwdg2": 3, "hwfv1": 4}


@dataclass
class Raster:
    """ESRI-style raster (raster.hpp:10-26): values[row, col], row 0 north."""

    values: np.ndarray
    xll: float = 0.0
    yll: float = 0.0
    cellsize: float = 1.0
    nodata: float = -9999.0

    @property
    def nrows(self) -> int:
        return int(self.values.shape[0])

    @property
    def ncols(self) -> int:
        return int(self.values.shape[1])


@dataclass
class Inflow:
    """InflowSpec + Hydrograph (config.hpp:15-18, hydrograph.hpp:10-16)."""

    t: list
    q: list
    i0: int
    j0: int
    i1: int
    j1: int


@dataclass
class Scenario:
    name: str
    dem: Raster
    solver: str
    L: int
    eps: float = 1e-3
    manning: float = 0.0
    manning_raster: Raster | None = None
    initial_depth_raster: Raster | None = None
    initial_surface: float | None = None
    initial_depth: float = 0.0
    courant: float = 0.0
    bc: tuple = (0, 0, 0, 0)  # N, E, S, W; 0 reflective, 1 open
    inflows: list = field(default_factory=list)
    steps: int = 1
    adapt_every: int = 1
    g: float = 9.80665
    h_dry: float = 1e-6
    grid_mode: str = "nonuniform"  # or "uniform"

    @property
    def n_cells(self) -> int:
        return (self.dem.ncols - 1) * (self.dem.nrows - 1)


def _grid(n: int, dx: float):
    """Vertex coordinates (x[col], y[row]) of an (n+1)^2 raster, row 0 north."""
    x = np.arange(n + 1, dtype=np.float64) * dx
    y = (n - np.arange(n + 1, dtype=np.float64)) * dx
    return x, y


def _add_bumps(z: np.ndarray, x: np.ndarray, y: np.ndarray, n: int, dx: float, count: int,
               rng: np.random.Generator) -> None:
    extent = n * dx
    for _ in range(count):
        cx, cy = rng.uniform(0.0, extent, size=2)
        amp = rng.uniform(0.5, 3.0)
        sig = rng.uniform(20.0, 80.0)
        r = 5.0 * sig
        c0 = max(0, int(math.floor((cx - r) / dx)))
        c1 = min(n, int(math.ceil((cx + r) / dx)))
        # rows: y = (n - row) dx
        r0 = max(0, int(math.floor(n - (cy + r) / dx)))
        r1 = min(n, int(math.ceil(n - (cy - r) / dx)))
        if c0 > c1 or r0 > r1:
            continue
        xs = x[c0:c1 + 1] - cx
        ys = y[r0:r1 + 1] - cy
        d2 = ys[:, None] ** 2 + xs[None, :] ** 2
        z[r0:r1 + 1, c0:c1 + 1] += amp * np.exp(-d2 / (2.0 * sig * sig))


def _channel(z: np.ndarray, x: np.ndarray, y: np.ndarray, n: int, dx: float) -> None:
    centre = (n / 2.0 + (40.0 * n / 256.0) * np.sin(2.0 * np.pi * x / (n * dx))) * dx
    mask = np.abs(y[:, None] - centre[None, :]) <= 1.5 * dx
    z[mask] -= 2.0


def terrain(n: int, dx: float, slope: float, bumps: int, seed: int, channel: bool = True):
    rng = np.random.default_rng(seed)
    x, y = _grid(n, dx)
    z = np.broadcast_to(slope * x[None, :], (n + 1, n + 1)).copy()
    _add_bumps(z, x, y, n, dx, bumps, rng)
    if channel:
        _channel(z, x, y, n, dx)
    return z, x, y, rng


def _scaled(n: int, L: int, bumps: int, scale: int):
    if scale < 1 or (scale & (scale - 1)):
        raise ValueError("scale must be a power of two")
    s = int(round(math.log2(scale)))
    return n // scale, L - s, max(2, bumps // (scale * scale))


def config0(scale: int = 1) -> Scenario:
    """Static non-uniform DG2, 256^2 at dx = 10 m, L = 8, dam break, 1000 steps."""
    n, L, nb = _scaled(256, 8, 20, scale)
    dx = 10.0
    z, x, y, _ = terrain(n, dx, 0.001, nb, SEED + 0)
    h0 = np.where(x[None, :] < 0.5 * n * dx, 2.0, 0.0) * np.ones((n + 1, 1))
    return Scenario(name=f"c0_dg2_{n}", dem=Raster(z, cellsize=dx), solver="dg2", L=L,
                    manning=0.03, courant=0.33, initial_depth_raster=Raster(h0, cellsize=dx),
                    steps=1000)


def _c1_dem(scale: int):
    n, L, nb = _scaled(1024, 10, 80, scale)
    dx = 5.0
    z, _, _, _ = terrain(n, dx, 0.001, nb, SEED + 1)
    return n, L, dx, z


def _c1_inflow(n: int) -> Inflow:
    # point source at cell (10, 512) of the 1024^2 grid; triangular hydrograph
    i = max(0, min(n - 1, 10 * n // 1024))
    j = n // 2
    return Inflow(t=[0.0, 1800.0, 3600.0], q=[0.0, 50.0, 0.0], i0=i, j0=j, i1=i, j1=j)


def config1(scale: int = 1) -> Scenario:
    """Static non-uniform ACC, 1024^2 at dx = 5 m, L = 10, point-source inflow, 2000 steps."""
    n, L, dx, z = _c1_dem(scale)
    return Scenario(name=f"c1_acc_{n}", dem=Raster(z, cellsize=dx), solver="acc", L=L,
                    manning=0.035, courant=0.7, bc=(0, 1, 0, 0), inflows=[_c1_inflow(n)],
                    steps=2000)


def config2(scale: int = 1, adaptive: bool = True) -> Scenario:
    """C1 DEM/inflow: static FV1 (adaptive=False) or HWFV1 re-adapted every step."""
    n, L, dx, z = _c1_dem(scale)
    return Scenario(name=f"c2_{'hwfv1' if adaptive else 'fv1'}_{n}", dem=Raster(z, cellsize=dx),
                    solver="hwfv1" if adaptive else "fv1", L=L, manning=0.035, courant=0.5,
                    bc=(0, 1, 0, 0), inflows=[_c1_inflow(n)], steps=2000, adapt_every=1)


def config3(scale: int = 1) -> Scenario:
    """Adaptive MWDG2, 2048^2 at dx = 2 m, ridge with a breach, reservoir, 5000 steps.

    Ridge: +10 m on vertices with |x - 400 m| <= 3 m, except a 50 m breach
    centred on y = domain centre.  Reservoir: water SURFACE at 12 m elevation
    for x < 396 m (upstream of the ridge footprint), dry downstream.
    """
    n, L, nb = _scaled(2048, 11, 200, scale)
    dx = 2.0
    z, x, y, _ = terrain(n, dx, 0.001, nb, SEED + 2)
    xr = 400.0 * (n * dx) / 4096.0 if scale > 1 else 400.0
    ridge = (np.abs(x[None, :] - xr) <= 3.0) & ~(np.abs(y[:, None] - 0.5 * n * dx) < 25.0)
    z = z + 10.0 * ridge
    h0 = np.where(x[None, :] < xr - 4.0, np.maximum(0.0, 12.0 - z), 0.0)
    return Scenario(name=f"c3_mwdg2_{n}", dem=Raster(z, cellsize=dx), solver="mwdg2", L=L,
                    manning=0.025, courant=0.33, initial_depth_raster=Raster(h0, cellsize=dx),
                    steps=5000, adapt_every=1)


def config4(scale: int = 1, uniform: bool = False) -> Scenario:
    """Urban case, 8192^2 at dx = 1 m, L = 13: buildings, street Manning, rainfall.

    Buildings: axis-aligned rectangles 10 m tall with sides U{10..40} m placed
    uniformly until 5 % of the vertices are covered.  Streets: a lattice of
    8 m wide streets every 64 m (cells with i mod 64 < 8 or j mod 64 < 8) that
    are not under a building get n = 0.02; everything else n = 0.05.  The
    Manning raster is cell-centred (n x n).  Rain: 50 mm/h for 3600 s as one
    whole-domain inflow with Q = 50e-3/3600 * (n dx)^2 m^3/s.
    """
    n, L, nb = _scaled(8192, 13, 1000, scale)
    dx = 1.0
    z, x, y, rng = terrain(n, dx, 0.0005, nb, SEED + 3, channel=False)
    cover = np.zeros((n + 1, n + 1), dtype=bool)
    target = 0.05 * cover.size
    covered = 0
    lo, hi = (10, 40) if scale == 1 else (max(2, 10 // scale), max(3, 40 // scale))
    while covered < target:
        w, h = rng.integers(lo, hi + 1, size=2)
        c0 = int(rng.integers(0, n + 1 - w))
        r0 = int(rng.integers(0, n + 1 - h))
        blk = cover[r0:r0 + h + 1, c0:c0 + w + 1]
        covered += int(blk.size - np.count_nonzero(blk))
        blk[...] = True
    z = z + 10.0 * cover
    # cell-centred Manning raster, row 0 north; a cell is "building" when all
    # four of its vertices are covered
    bcell = cover[:-1, :-1] & cover[:-1, 1:] & cover[1:, :-1] & cover[1:, 1:]
    jj = (n - 1 - np.arange(n))[:, None]
    ii = np.arange(n)[None, :]
    period = max(8, 64 // scale)
    width = max(1, 8 // scale)
    street = ((ii % period) < width) | ((jj % period) < width)
    man = np.where(street & ~bcell, 0.02, 0.05)
    q = 50e-3 / 3600.0 * (n * dx) ** 2
    rain = Inflow(t=[0.0, 3600.0, 3600.001], q=[q, q, 0.0], i0=0, j0=0, i1=n - 1, j1=n - 1)
    return Scenario(name=f"c4_{'uni' if uniform else 'nu'}_dg2_{n}", dem=Raster(z, cellsize=dx),
                    solver="dg2", L=L, manning=0.05, manning_raster=Raster(man, cellsize=dx),
                    courant=0.33, inflows=[rain], steps=10000,
                    grid_mode="uniform" if uniform else "nonuniform")


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def to_arrays(sc: Scenario) -> dict:
    """Flatten a scenario into numpy arrays (for the committed golden fixtures)."""
    d = {
        "name": np.array(sc.name), "solver": np.array(sc.solver), "grid_mode": np.array(sc.grid_mode),
        "dem": sc.dem.values, "dem_geo": np.array([sc.dem.xll, sc.dem.yll, sc.dem.cellsize, sc.dem.nodata]),
        "scalars": np.array([sc.L, sc.eps, sc.manning, sc.courant, sc.initial_depth, sc.steps,
                             sc.adapt_every, sc.g, sc.h_dry,
                             np.nan if sc.initial_surface is None else sc.initial_surface]),
        "bc": np.array(sc.bc, dtype=np.int32),
        "n_inflows": np.array(len(sc.inflows)),
    }
    if sc.manning_raster is not None:
        d["manning_raster"] = sc.manning_raster.values
        d["manning_geo"] = np.array([sc.manning_raster.xll, sc.manning_raster.yll,
                                     sc.manning_raster.cellsize, sc.manning_raster.nodata])
    if sc.initial_depth_raster is not None:
        d["h0_raster"] = sc.initial_depth_raster.values
    for k, f in enumerate(sc.inflows):
        d[f"inflow{k}_t"] = np.array(f.t, dtype=np.float64)
        d[f"inflow{k}_q"] = np.array(f.q, dtype=np.float64)
        d[f"inflow{k}_rect"] = np.array([f.i0, f.j0, f.i1, f.j1], dtype=np.int32)
    return d


def from_arrays(d) -> Scenario:
    geo = d["dem_geo"]
    s = d["scalars"]
    dem = Raster(np.array(d["dem"]), xll=float(geo[0]), yll=float(geo[1]), cellsize=float(geo[2]),
                 nodata=float(geo[3]))
    mr = None
    if "manning_raster" in d:
        mg = d["manning_geo"]
        mr = Raster(np.array(d["manning_raster"]), xll=float(mg[0]), yll=float(mg[1]),
                    cellsize=float(mg[2]), nodata=float(mg[3]))
    h0 = Raster(np.array(d["h0_raster"]), xll=float(geo[0]), yll=float(geo[1]),
                cellsize=float(geo[2]), nodata=float(geo[3])) if "h0_raster" in d else None
    infl = []
    for k in range(int(d["n_inflows"])):
        r = d[f"inflow{k}_rect"]
        infl.append(Inflow(t=list(d[f"inflow{k}_t"]), q=list(d[f"inflow{k}_q"]), i0=int(r[0]),
                           j0=int(r[1]), i1=int(r[2]), j1=int(r[3])))
    return Scenario(name=str(d["name"]), dem=dem, solver=str(d["solver"]), L=int(s[0]), eps=float(s[1]),
                    manning=float(s[2]), courant=float(s[3]), initial_depth=float(s[4]),
                    steps=int(s[5]), adapt_every=int(s[6]), g=float(s[7]), h_dry=float(s[8]),
                    initial_surface=None if np.isnan(s[9]) else float(s[9]),
                    manning_raster=mr, initial_depth_raster=h0, bc=tuple(int(x) for x in d["bc"]),
                    inflows=infl, grid_mode=str(d["grid_mode"]))


def spike(n: int = 16, height: float = 1.0) -> Raster:
    """Flat DEM with one raised vertex at the centre (test_mra.cpp:24-29)."""
    v = np.zeros((n + 1, n + 1))
    v[(n + 1) // 2, (n + 1) // 2] = height
    return Raster(v, cellsize=1.0)


def _write_asc(path: str, r: "Raster"):
    # ESRI ASCII grid as the reference reads and writes it (raster.cpp:22-96):
    # 17 significant digits, row 0 north
    v = np.asarray(r.values, dtype=np.float64)
    with open(path, "w") as f:
        f.write(f"ncols {v.shape[1]}\nnrows {v.shape[0]}\nxllcorner {r.xll!r}\nyllcorner {r.yll!r}\n"
                f"cellsize {r.cellsize!r}\nNODATA_value {r.nodata!r}\n")
        np.savetxt(f, v, fmt="%.17g")


def emit_config(sc: "Scenario", out_dir: str, end_time: float, output_interval: float = 0.0,
                gauge_interval: float = 0.0, gauges=(), threads: int = 1) -> str:
    """Write `sc` as the reference's own scenario files (config.cpp:93-245
    `key = value` config, ASCII rasters, `t,Q` hydrograph CSVs) under
    `out_dir`; returns the config path.  The reference's run_scenario and the
    GPU drop-in both read exactly these files."""
    import os
    os.makedirs(out_dir, exist_ok=True)
    _write_asc(os.path.join(out_dir, "dem.asc"), sc.dem)
    names = {"dg2": "dg2", "fv1": "fv1", "acc": "acc", "mwdg2": "mwdg2", "hwfv1": "hwfv1"}
    lines = ["dem_path = dem.asc", f"solver = {names[sc.solver]}", f"grid_mode = {sc.grid_mode}",
             f"epsilon = {sc.eps!r}", f"max_level = {sc.L}", f"end_time = {end_time!r}",
             f"manning = {sc.manning!r}", f"g = {sc.g!r}", f"h_dry = {sc.h_dry!r}",
             f"adapt_every = {sc.adapt_every}", f"threads = {threads}"]
    if output_interval > 0:
        lines.append(f"output_interval = {output_interval!r}")
    if gauge_interval > 0:
        lines.append(f"gauge_interval = {gauge_interval!r}")
    if sc.courant > 0:
        lines.append(f"courant = {sc.courant!r}")
    for key, b in zip(("boundary_n", "boundary_e", "boundary_s", "boundary_w"), sc.bc):
        lines.append(f"{key} = {'open' if b else 'reflective'}")
    if sc.manning_raster is not None:
        _write_asc(os.path.join(out_dir, "manning.asc"), sc.manning_raster)
        lines.append("manning_raster = manning.asc")
    if sc.initial_depth_raster is not None:
        _write_asc(os.path.join(out_dir, "h0.asc"), sc.initial_depth_raster)
        lines.append("initial_depth_raster = h0.asc")
    if sc.initial_surface is not None:
        lines.append(f"initial_surface = {sc.initial_surface!r}")
    if sc.initial_depth:
        lines.append(f"initial_depth = {sc.initial_depth!r}")
    for k, f in enumerate(sc.inflows):
        p = f"hyd{k}.csv"
        with open(os.path.join(out_dir, p), "w") as h:
            h.write("t,Q\n")
            for t, q in zip(f.t, f.q):
                h.write(f"{t!r},{q!r}\n")
        lines.append(f"inflow = {p} @ {f.i0} {f.j0} {f.i1} {f.j1}")
    for x, y in gauges:
        lines.append(f"gauge = {x!r} {y!r}")
    path = os.path.join(out_dir, "scenario.cfg")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    return path
