"""ctypes description of the C ABI declared in include/fm_gpu.h.

`Backend(path, prefix)` binds one shared library exposing that ABI.  The
product binds libfm_gpu.so with prefix "fm_" (see api.py).  The same table
lets the parity tests bind the CPU checkers that mirror the ABI (prefix
"orc_" / "ref_"); those live under oracle/ and are loaded only by tests/,
__graft_entry__.smoke() and bench.py's CPU legs.
"""
from __future__ import annotations

import ctypes as C
import os
import math

import numpy as np

FM_OK = 0
ERRORS = {1: "other", 2: "config", 3: "io", 4: "blowup", 5: "structure", 6: "domain", 7: "cuda"}


class FmError(RuntimeError):
    """A non-zero status from the C ABI (maps to the reference exception types)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERRORS.get(code, code)}] {msg}")
        self.code = code


class BlowUpError(FmError):
    """BlowUpError{t} (errors.hpp:34-37); `result` is the run's fm_run_result
    (steps done, bad_x / bad_y of the first non-finite leaf)."""

    def __init__(self, code: int, msg: str, t: float, result=None):
        super().__init__(code, msg)
        self.t = t
        self.result = result


class c_raster(C.Structure):
    _fields_ = [("values", C.POINTER(C.c_double)), ("ncols", C.c_int32), ("nrows", C.c_int32),
                ("xll", C.c_double), ("yll", C.c_double), ("cellsize", C.c_double),
                ("nodata", C.c_double), ("on_device", C.c_int32)]


class c_inflow(C.Structure):
    _fields_ = [("t", C.POINTER(C.c_double)), ("q", C.POINTER(C.c_double)),
                ("nsamples", C.c_int32), ("i0", C.c_int32), ("j0", C.c_int32),
                ("i1", C.c_int32), ("j1", C.c_int32)]


class c_desc(C.Structure):
    _fields_ = [("solver", C.c_int32), ("g", C.c_double), ("h_dry", C.c_double),
                ("courant", C.c_double), ("bc", C.c_int32 * 4), ("manning", C.c_double),
                ("manning_raster", C.POINTER(c_raster)),
                ("initial_depth_raster", C.POINTER(c_raster)),
                ("has_initial_surface", C.c_int32), ("initial_surface", C.c_double),
                ("initial_depth", C.c_double), ("inflows", C.POINTER(c_inflow)),
                ("n_inflows", C.c_int32), ("epsilon", C.c_double), ("max_level", C.c_int32),
                ("adapt_every", C.c_int32), ("libm", C.c_int32)]


class c_clock(C.Structure):
    _fields_ = [("end_time", C.c_double), ("output_interval", C.c_double),
                ("gauge_interval", C.c_double), ("now", C.c_double),
                ("next_output", C.c_int64), ("next_gauge", C.c_int64)]


class c_result(C.Structure):
    _fields_ = [("steps", C.c_int64), ("dt_min", C.c_double), ("dt_max", C.c_double),
                ("volume_inflow", C.c_double), ("blew_up", C.c_int32),
                ("blow_up_time", C.c_double), ("bad_x", C.c_double), ("bad_y", C.c_double),
                ("finished", C.c_int32), ("event_due", C.c_int32)]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
PD = C.POINTER(C.c_double)
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)
PU8 = C.POINTER(C.c_uint8)

# name -> (restype, argtypes); the common ABI of fm_/orc_/ref_ libraries
SIGS = {
    "last_error": (C.c_char_p, []),
    "mra_static": (C.c_int, [C.POINTER(c_raster), I32, D, I32, I32, PP]),
    "grid_destroy": (C.c_int, [P]),
    "grid_num_leaves": (I64, [P]),
    "grid_info": (C.c_int, [P, PI32, PI32, PI32, PD, PD, PD, PD]),
    "grid_leaves": (C.c_int, [P, I32, PI32, PI32, PI32, PD]),
    "grid_flags": (C.c_int, [P, I32, PU8]),
    "grid_dhat": (C.c_int, [P, I32, PD]),
    "grid_near_threshold": (C.c_int, [P, D, PI64]),
    "sim_create": (C.c_int, [C.POINTER(c_desc), C.POINTER(c_raster), P, PP]),
    "sim_destroy": (C.c_int, [P]),
    "sim_num_cells": (I64, [P]),
    "sim_num_segments": (I64, [P]),
    "sim_compute_dt": (C.c_int, [P, PD]),
    "sim_step": (C.c_int, [P, D]),
    "sim_apply_inflows": (C.c_int, [P, D, D, PD]),
    "sim_adapt": (C.c_int, [P, D]),
    "sim_volume": (C.c_int, [P, PD]),
    "sim_finite": (C.c_int, [P, PI32, PD, PD]),
    "sim_download": (C.c_int, [P, PI32, PI32, PI32, PD, PD]),
    "sim_upload": (C.c_int, [P, PD]),
    "sim_raster_shape": (C.c_int, [P, PI32, PI32, PD, PD, PD, PD]),
    "sim_raster": (C.c_int, [P, I32, PD, I32]),
    "sim_sample_gauges": (C.c_int, [P, I32, PD, PD, PD]),
    "sim_element_log": (I64, [P, PD, PI64, I64]),
    "sim_run": (C.c_int, [P, C.POINTER(c_clock), I64, I32, C.POINTER(c_result)]),
}
OPTIONAL = {
    "init": (C.c_int, [I32]),
    "set_stream": (C.c_int, [P]),
    "synchronize": (C.c_int, []),
    "launch_count": (I64, []),
    "grid_timing": (C.c_int, [P, PD, PD]),
    "sim_last_run_ms": (C.c_int, [P, PD]),
    "grid_details": (C.c_int, [P, I32, PD]),
    "sim_profile": (C.c_int, [P, I64, PD, PI64, I32, PI32]),
    "sim_snapshot": (C.c_int, [P]),
    "sim_restore": (C.c_int, [P]),
    "sim_kernel_name": (C.c_char_p, [P, I32]),
    "sim_acc_q": (C.c_int, [P, PD, PD]),
    "sim_acc_faces": (C.c_int, [P, PD, PD, PD, PD]),
    "sim_checkpoint": (C.c_int, [P, C.c_char_p]),
    "sim_adapt_stats": (C.c_int, [P, PI64, PI64]),
    "sim_resume": (C.c_int, [P, C.c_char_p]),
    "sim_geometry": (C.c_int, [P, PI32, PI32, PI32, PD, PD, PD]),
    "set_threads": (None, [I32]),
    "hw_threads": (I32, []),
    "generate_static_grid": (C.c_int, [C.POINTER(c_raster), I32, D, I32, I32, PI64]),
    "grade_flags": (C.c_int, [I32, I32, I32, I32, PU8]),
    "pcbrt": (D, [D]),
    "selftest": (C.c_int, [I32, I64, C.c_uint64, PI64]),
    "debug_guard_report": (C.c_int, [PI64, PI64]),
    "hll": (None, [D, D, D, D, D, D, D, D, PD]),
    "friction": (None, [D, PD, PD, D, D, D, D]),
    "encode": (None, [PD, I32, PD, PD]),
    "decode": (None, [PD, PD, I32, PD]),
    "bank": (None, [I32, PD]),
    # sharding (libfm_gpu.so) and topology (both)
    "comm_unique_id": (C.c_int, [C.c_char_p]),
    "comm_create_nccl": (C.c_int, [I32, I32, C.c_char_p, PP]),
    "comm_create_local": (C.c_int, [I32, PP]),
    "comm_create_host": (C.c_int, [I32, I32, C.c_char_p, PP]),
    "comm_destroy": (C.c_int, [P]),
    "sim_create_shard": (C.c_int, [C.POINTER(c_desc), C.POINTER(c_raster), P, P, I32, PP]),
    "sim_shard_info": (C.c_int, [P, PI32, PI32, PI64, PI64, PI64, PI64]),
    "group_run": (C.c_int, [C.POINTER(P), I32, C.POINTER(c_clock), I64, I32, C.POINTER(c_result)]),
    "shard_plan": (C.c_int, [I64, I64, PI32, PI32, I32, I32, PI64, PI64, PI64, PI64, PI64, PI32,
                             PI64, PI64]),
    "sim_topology": (C.c_int, [P, PI32, PI32, PI32, PI32, PI32]),
    "grid_import": (C.c_int, [I32, I32, I32, D, D, D, I64, PI32, PI32, PI32, PD, PP]),
    "extent_metrics": (C.c_int, [C.POINTER(c_raster), C.POINTER(c_raster), D, C.POINTER(C.c_int64), PD]),
    "eval_libm": (C.c_int, [I32, I64, PD, PD]),
    # file formats
    "raster_read": (C.c_int, [C.c_char_p, C.POINTER(c_raster)]),
    "raster_release": (C.c_int, [C.POINTER(c_raster)]),
    "raster_write": (C.c_int, [C.POINTER(c_raster), C.c_char_p, I32]),
    "grid_write": (C.c_int, [P, C.c_char_p, I32]),
    "grid_read": (C.c_int, [C.c_char_p, PP]),
}



def _check_array(a, dtype, shape, writable=False):
    """Raise ValueError unless `a` is a C-contiguous ndarray of `dtype` and
    `shape` (the C ABI writes/reads exactly that many elements through a raw
    pointer)."""
    if not isinstance(a, np.ndarray):
        raise ValueError(f"expected a numpy array, got {type(a).__name__}")
    if a.dtype != dtype or a.shape != tuple(shape) or not a.flags.c_contiguous:
        raise ValueError(f"expected a C-contiguous {np.dtype(dtype).name} array of shape {tuple(shape)}, "
                         f"got {a.dtype.name} {a.shape} (c_contiguous={a.flags.c_contiguous})")
    if writable and not a.flags.writeable:
        raise ValueError("output array is read-only")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(PD)


class Backend:
    """One loaded library implementing the ABI under `prefix`."""

    def __init__(self, path: str, prefix: str, mode: int = C.RTLD_LOCAL):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path, mode=mode)
        self.fn = {}
        for name, (res, args) in SIGS.items():
            f = getattr(self.lib, prefix + name)
            f.restype, f.argtypes = res, args
            self.fn[name] = f
        for name, (res, args) in OPTIONAL.items():
            f = getattr(self.lib, prefix + name, None)
            if f is not None:
                f.restype, f.argtypes = res, args
                self.fn[name] = f

    def has(self, name: str) -> bool:
        return name in self.fn

    def check(self, status: int, result: c_result | None = None):
        if status != FM_OK:
            msg = self.fn["last_error"]().decode(errors="replace")
            if status == 4 and result is not None:
                raise BlowUpError(status, msg, result.blow_up_time, result)
            raise FmError(status, msg)

    def call(self, name, *args):
        st = self.fn[name](*args)
        self.check(st)
        return st

    # ---- helpers -------------------------------------------------------
    def grid(self, dem, L: int, eps: float, graded: bool = True, kind: int = 0,
             device_ptr: int | None = None):
        """fm_mra_static; `device_ptr` passes a DEM already resident in HBM."""
        return Grid(self, dem, L, eps, graded, kind, device_ptr)

    def sim(self, scenario, grid=None, libm: int = 0):
        return Sim(self, scenario, grid, libm)

    def grid_import(self, L: int, M: int, N: int, R: float, x0: float, y0: float, level, i, j,
                    topo3) -> "Grid":
        """fm_grid_import: read_nug's NonUniformGrid from a leaf list + topography."""
        lv = np.ascontiguousarray(level, np.int32)
        ii = np.ascontiguousarray(i, np.int32)
        jj = np.ascontiguousarray(j, np.int32)
        z = np.ascontiguousarray(topo3, np.float64)
        h = P()
        self.call("grid_import", L, M, N, R, x0, y0, len(lv), lv.ctypes.data_as(PI32),
                  ii.ctypes.data_as(PI32), jj.ctypes.data_as(PI32), dptr(z), C.byref(h))
        g = Grid.__new__(Grid)
        g.be, g.h, g.eps, g._keep = self, h, 0.0, []
        return g

    def extent_metrics(self, test, ref, wet_threshold: float):
        """extent_metrics (metrics.cpp:51-73): ({hits, misses, false_alarms},
        {hit_rate, false_alarm, csi})."""
        keep: list = []
        a, b = make_raster(test, keep), make_raster(ref, keep)
        cnt = np.zeros(3, np.int64)
        rates = np.zeros(3, np.float64)
        self.call("extent_metrics", C.byref(a), C.byref(b), float(wet_threshold),
                  cnt.ctypes.data_as(C.POINTER(C.c_int64)), dptr(rates))
        return cnt, rates

    # ---- file formats ----
    def read_raster(self, path: str):
        """read_ascii_grid (raster.cpp:22-79) or the binary side format: a
        scenarios.Raster copied out of the library's buffer."""
        from .scenarios import Raster
        r = c_raster()
        self.call("raster_read", os.fsencode(path), C.byref(r))
        try:
            vals = np.ctypeslib.as_array(r.values, shape=(r.nrows, r.ncols)).copy()
        finally:
            self.call("raster_release", C.byref(r))
        return Raster(vals, r.xll, r.yll, r.cellsize, r.nodata)

    def write_raster(self, raster, path: str, binary: bool = False) -> None:
        """write_ascii_grid (raster.cpp:81-96), or the binary side format."""
        keep: list = []
        r = make_raster(raster, keep)
        self.call("raster_write", C.byref(r), os.fsencode(path), 1 if binary else 0)

    def read_grid(self, path: str) -> "Grid":
        """read_nug (quadgrid.cpp:304-327), or the binary side format."""
        h = P()
        self.call("grid_read", os.fsencode(path), C.byref(h))
        g = Grid.__new__(Grid)
        g.be, g.h, g.eps, g._keep = self, h, 0.0, []
        return g

    # ---- sharding ----
    def comm_local(self, nranks: int) -> "Comm":
        h = P()
        self.call("comm_create_local", int(nranks), C.byref(h))
        return Comm(self, h, nranks, None)

    def comm_unique_id(self) -> bytes:
        buf = C.create_string_buffer(128)
        self.call("comm_unique_id", buf)
        return buf.raw

    def comm_nccl(self, nranks: int, rank: int, uid: bytes) -> "Comm":
        h = P()
        self.call("comm_create_nccl", int(nranks), int(rank), C.c_char_p(bytes(uid)), C.byref(h))
        return Comm(self, h, nranks, rank)

    def comm_host(self, nranks: int, rank: int, name: str) -> "Comm":
        """fm_comm_create_host: one process per rank over a shared-memory segment."""
        h = P()
        self.call("comm_create_host", int(nranks), int(rank), name.encode(), C.byref(h))
        return Comm(self, h, nranks, rank)

    def shard_sim(self, scenario, grid, comm: "Comm", rank: int, libm: int = 0):
        return Sim(self, scenario, grid, libm, comm=comm, rank=rank)

    def group_run(self, sims, steps: int, end_time: float = 1e12, gauge_interval: float = 0.0,
                  output_interval: float = 0.0, stop_at_events: bool = False):
        """fm_group_run: the drive loop over every shard of a local group."""
        arr = (P * len(sims))(*[s.h for s in sims])
        clock = c_clock(end_time, output_interval, gauge_interval, 0.0, 1, 1)
        res = c_result()
        st = self.fn["group_run"](arr, len(sims), C.byref(clock), steps, 1 if stop_at_events else 0,
                                  C.byref(res))
        self.check(st, res)
        return clock, res

    def shard_plan(self, n: int, seg_l: np.ndarray, seg_r: np.ndarray, nranks: int, rank: int):
        """fm_shard_plan (host only): dict with first, count, nseg_local, halo,
        halo_owner and send (list per rank of ascending global leaf ids)."""
        sl = np.ascontiguousarray(seg_l, np.int32)
        sr = np.ascontiguousarray(seg_r, np.int32)
        first, count, nsl, nh = I64(), I64(), I64(), I64()
        cnt = np.zeros(nranks, np.int64)
        P64 = C.POINTER(C.c_int64)
        self.call("shard_plan", n, len(sl), sl.ctypes.data_as(PI32), sr.ctypes.data_as(PI32), nranks,
                  rank, C.byref(first), C.byref(count), C.byref(nsl), C.byref(nh), None, None,
                  cnt.ctypes.data_as(P64), None)
        halo = np.zeros(nh.value, np.int64)
        owner = np.zeros(nh.value, np.int32)
        send = np.zeros(int(cnt.sum()), np.int64)
        self.call("shard_plan", n, len(sl), sl.ctypes.data_as(PI32), sr.ctypes.data_as(PI32), nranks,
                  rank, C.byref(first), C.byref(count), C.byref(nsl), C.byref(nh),
                  halo.ctypes.data_as(P64), owner.ctypes.data_as(PI32), cnt.ctypes.data_as(P64),
                  send.ctypes.data_as(P64))
        off = np.concatenate([[0], np.cumsum(cnt)])
        return dict(first=first.value, count=count.value, nseg_local=nsl.value, halo=halo,
                    halo_owner=owner, send=[send[off[r]:off[r + 1]] for r in range(nranks)])


class Comm:
    """fm_comm: the transport between the shards of one partition."""

    def __init__(self, be: Backend, h, nranks: int, rank):
        self.be, self.h, self.nranks, self.rank = be, h, nranks, rank

    def __del__(self):
        if getattr(self, "h", None):
            self.be.fn["comm_destroy"](self.h)
            self.h = None


def make_raster(r, keep: list) -> c_raster:
    vals = np.ascontiguousarray(r.values, dtype=np.float64)
    keep.append(vals)
    return c_raster(dptr(vals), r.ncols, r.nrows, r.xll, r.yll, r.cellsize, r.nodata, 0)


class Grid:
    """A static MRA grid (NonUniformGrid + the DetailTree flags)."""

    def __init__(self, be: Backend, dem, L: int, eps: float, graded: bool, kind: int,
                 device_ptr: int | None = None):
        self.be = be
        keep: list = []
        if device_ptr is not None:
            self._r = c_raster(C.cast(C.c_void_p(device_ptr), PD), dem.ncols, dem.nrows, dem.xll,
                               dem.yll, dem.cellsize, dem.nodata, 1)
        else:
            self._r = make_raster(dem, keep)
        self._keep = keep
        h = P()
        be.call("mra_static", C.byref(self._r), L, eps, 1 if graded else 0, kind, C.byref(h))
        self.h = h
        self.eps = eps

    def __del__(self):
        if getattr(self, "h", None):
            self.be.fn["grid_destroy"](self.h)
            self.h = None

    @property
    def num_leaves(self) -> int:
        return int(self.be.fn["grid_num_leaves"](self.h))

    def info(self) -> dict:
        L, M, N = I32(), I32(), I32()
        R, x0, y0, nm = D(), D(), D(), D()
        self.be.call("grid_info", self.h, C.byref(L), C.byref(M), C.byref(N), C.byref(R),
                     C.byref(x0), C.byref(y0), C.byref(nm))
        return dict(L=L.value, M=M.value, N=N.value, R=R.value, x0=x0.value, y0=y0.value,
                    field_norm=nm.value)

    def write(self, path: str, binary: bool = False) -> None:
        """write_nug (quadgrid.cpp:287-302), or the binary side format."""
        self.be.call("grid_write", self.h, os.fsencode(path), 1 if binary else 0)

    def leaves(self, order: int = 0):
        n = self.num_leaves
        lv = np.zeros(n, np.int32)
        i = np.zeros(n, np.int32)
        j = np.zeros(n, np.int32)
        z = np.zeros((n, 3), np.float64)
        self.be.call("grid_leaves", self.h, order, lv.ctypes.data_as(PI32), i.ctypes.data_as(PI32),
                     j.ctypes.data_as(PI32), dptr(z))
        return lv, i, j, z

    def flags(self, level: int) -> np.ndarray:
        inf = self.info()
        out = np.zeros((inf["N"] << level) * (inf["M"] << level), np.uint8)
        self.be.call("grid_flags", self.h, level, out.ctypes.data_as(PU8))
        return out

    def dhat(self, level: int) -> np.ndarray:
        inf = self.info()
        out = np.zeros((inf["N"] << level) * (inf["M"] << level), np.float64)
        self.be.call("grid_dhat", self.h, level, dptr(out))
        return out

    def near_threshold(self, rel: float = 1e-12) -> int:
        c = I64()
        self.be.call("grid_near_threshold", self.h, rel, C.byref(c))
        return int(c.value)

    def timing(self):
        ms, b = D(), D()
        self.be.call("grid_timing", self.h, C.byref(ms), C.byref(b))
        return ms.value, b.value


class Sim:
    """A drive<Sim>-shaped simulation (run.cpp:35-141) behind the ABI."""

    def __init__(self, be: Backend, sc, grid: Grid | None = None, libm: int = 0,
                 comm: "Comm | None" = None, rank: int = 0):
        from .scenarios import SOLVERS

        self.be = be
        keep: list = []
        d = c_desc()
        d.solver = SOLVERS[sc.solver]
        d.g = sc.g
        d.h_dry = sc.h_dry
        d.courant = sc.courant
        for k in range(4):
            d.bc[k] = int(sc.bc[k])
        d.manning = sc.manning
        if sc.manning_raster is not None:
            mr = make_raster(sc.manning_raster, keep)
            keep.append(mr)
            d.manning_raster = C.pointer(mr)
        if sc.initial_depth_raster is not None:
            hr = make_raster(sc.initial_depth_raster, keep)
            keep.append(hr)
            d.initial_depth_raster = C.pointer(hr)
        if sc.initial_surface is not None:
            d.has_initial_surface = 1
            d.initial_surface = sc.initial_surface
        d.initial_depth = sc.initial_depth
        if sc.inflows:
            arr = (c_inflow * len(sc.inflows))()
            for k, f in enumerate(sc.inflows):
                t = np.ascontiguousarray(f.t, np.float64)
                q = np.ascontiguousarray(f.q, np.float64)
                keep += [t, q]
                arr[k] = c_inflow(dptr(t), dptr(q), len(t), f.i0, f.j0, f.i1, f.j1)
            keep.append(arr)
            d.inflows = C.cast(arr, C.POINTER(c_inflow))
            d.n_inflows = len(sc.inflows)
        d.epsilon = sc.eps
        d.max_level = sc.L
        d.adapt_every = sc.adapt_every
        d.libm = libm
        dem = make_raster(sc.dem, keep)
        h = P()
        if comm is not None:
            be.call("sim_create_shard", C.byref(d), C.byref(dem),
                    grid.h if grid is not None else None, comm.h, int(rank), C.byref(h))
        else:
            be.call("sim_create", C.byref(d), C.byref(dem), grid.h if grid is not None else None,
                    C.byref(h))
        self.comm = comm
        self.h = h
        self.grid = grid
        self.scenario = sc

    def __del__(self):
        if getattr(self, "h", None):
            self.be.fn["sim_destroy"](self.h)
            self.h = None

    @property
    def num_cells(self) -> int:
        return int(self.be.fn["sim_num_cells"](self.h))

    @property
    def num_segments(self) -> int:
        return int(self.be.fn["sim_num_segments"](self.h))

    def compute_dt(self) -> float:
        v = D()
        self.be.call("sim_compute_dt", self.h, C.byref(v))
        return v.value

    def step(self, dt: float):
        self.be.call("sim_step", self.h, dt)

    def apply_inflows(self, t: float, dt: float) -> float:
        v = D()
        self.be.call("sim_apply_inflows", self.h, t, dt, C.byref(v))
        return v.value

    def adapt(self, t: float):
        self.be.call("sim_adapt", self.h, t)

    def volume(self) -> float:
        v = D()
        self.be.call("sim_volume", self.h, C.byref(v))
        return v.value

    def finite_state(self):
        ok, bx, by = I32(), D(), D()
        self.be.call("sim_finite", self.h, C.byref(ok), C.byref(bx), C.byref(by))
        return bool(ok.value), bx.value, by.value

    def download(self, out=None):
        """(level, i, j, u[n,9], z[n,3]) in the reference order; `out` may hold
        preallocated (e.g. pinned) arrays of those shapes to fill."""
        n = self.num_cells
        if out is None:
            lv = np.zeros(n, np.int32)
            i = np.zeros(n, np.int32)
            j = np.zeros(n, np.int32)
            u = np.zeros((n, 9), np.float64)
            z = np.zeros((n, 3), np.float64)
        else:
            lv, i, j, u, z = out
            for a, dt, sh in ((lv, np.int32, (n,)), (i, np.int32, (n,)), (j, np.int32, (n,)),
                              (u, np.float64, (n, 9)), (z, np.float64, (n, 3))):
                _check_array(a, dt, sh, writable=True)
        self.be.call("sim_download", self.h, lv.ctypes.data_as(PI32), i.ctypes.data_as(PI32),
                     j.ctypes.data_as(PI32), dptr(u), dptr(z))
        return lv, i, j, u, z

    def upload(self, u9: np.ndarray):
        u9 = np.ascontiguousarray(u9, np.float64)
        if u9.shape != (self.num_cells, 9):
            raise ValueError(f"upload: u9 must have shape ({self.num_cells}, 9), got {u9.shape}")
        self.be.call("sim_upload", self.h, dptr(u9))

    def acc_faces(self, set_x=None, set_y=None):
        """UniformSim acc_qx / acc_qy (solver_uniform.hpp:53-54): optionally
        overwrite them, then return copies ((nx+1) x ny and nx x (ny+1))."""
        g = self.geometry()
        nx, ny = g["M"], g["N"]
        gx = np.zeros((ny, nx + 1))
        gy = np.zeros((ny + 1, nx))
        sx = None if set_x is None else np.ascontiguousarray(set_x, np.float64).reshape(ny, nx + 1)
        sy = None if set_y is None else np.ascontiguousarray(set_y, np.float64).reshape(ny + 1, nx)
        px = None if sx is None else dptr(sx)
        py = None if sy is None else dptr(sy)
        self.be.call("sim_acc_faces", self.h, dptr(gx), dptr(gy), px, py)
        return gx, gy

    def adapt_stats(self) -> dict:
        """The last adapt's encoded parents and the pyramid's internal nodes."""
        a, b = I64(), I64()
        self.be.call("sim_adapt_stats", self.h, C.byref(a), C.byref(b))
        return dict(n_encoded=a.value, n_internal=b.value)

    def checkpoint(self, path: str):
        """fm_sim_checkpoint: leaf keys, flow state, topography, ACC discharges."""
        self.be.call("sim_checkpoint", self.h, str(path).encode())

    def resume(self, path: str):
        """fm_sim_resume onto the same scenario and leaf set."""
        self.be.call("sim_resume", self.h, str(path).encode())

    def geometry(self) -> dict:
        L, M, N = I32(), I32(), I32()
        R, x0, y0 = D(), D(), D()
        self.be.call("sim_geometry", self.h, C.byref(L), C.byref(M), C.byref(N), C.byref(R),
                     C.byref(x0), C.byref(y0))
        return dict(L=L.value, M=M.value, N=N.value, R=R.value, x0=x0.value, y0=y0.value)

    def shard_info(self) -> dict:
        r, nr = I32(), I32()
        first, owned, halo, ng = I64(), I64(), I64(), I64()
        self.be.call("sim_shard_info", self.h, C.byref(r), C.byref(nr), C.byref(first),
                     C.byref(owned), C.byref(halo), C.byref(ng))
        return dict(rank=r.value, nranks=nr.value, first=first.value, owned=owned.value,
                    halo=halo.value, n_global=ng.value)

    def topology(self):
        """(level, i, j) per leaf and (seg_l, seg_r) per interior segment; device
        order for the GPU library, reference order for the oracle."""
        n, ns = self.num_cells, self.num_segments
        lv, i, j = (np.zeros(n, np.int32) for _ in range(3))
        sl, sr = np.zeros(ns, np.int32), np.zeros(ns, np.int32)
        self.be.call("sim_topology", self.h, lv.ctypes.data_as(PI32), i.ctypes.data_as(PI32),
                     j.ctypes.data_as(PI32), sl.ctypes.data_as(PI32), sr.ctypes.data_as(PI32))
        return lv, i, j, sl, sr

    def raster_shape(self) -> dict:
        nc, nr = I32(), I32()
        xll, yll, cs, nd = D(), D(), D(), D()
        self.be.call("sim_raster_shape", self.h, C.byref(nc), C.byref(nr), C.byref(xll),
                     C.byref(yll), C.byref(cs), C.byref(nd))
        return dict(ncols=nc.value, nrows=nr.value, xll=xll.value, yll=yll.value,
                    cellsize=cs.value, nodata=nd.value)

    def raster(self, which: int) -> np.ndarray:
        """depth_raster / qx_raster / qy_raster (which 0/1/2), row 0 north."""
        sh = self.raster_shape()
        out = np.empty((sh["nrows"], sh["ncols"]), np.float64)
        self.be.call("sim_raster", self.h, int(which), dptr(out), 0)
        return out

    def sample_gauges(self, x, y) -> np.ndarray:
        """sample_gauge at each (x, y): rows of GaugeValue {h, eta, u, v}."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.zeros((len(x), 4), np.float64)
        self.be.call("sim_sample_gauges", self.h, len(x), dptr(x), dptr(y), dptr(out))
        return out

    def element_log(self):
        n = int(self.be.fn["sim_element_log"](self.h, None, None, 0))
        t = np.zeros(n, np.float64)
        c = np.zeros(n, np.int64)
        self.be.fn["sim_element_log"](self.h, dptr(t), c.ctypes.data_as(PI64), n)
        return t, c

    def run(self, steps: int, clock: c_clock | None = None, end_time: float = 1e12,
            gauge_interval: float = 0.0, output_interval: float = 0.0,
            stop_at_events: bool = False):
        """drive<Sim> loop body for `steps` steps (run.cpp:80-111)."""
        if clock is None:
            clock = c_clock(end_time, output_interval, gauge_interval, 0.0, 1, 1)
        res = c_result()
        st = self.be.fn["sim_run"](self.h, C.byref(clock), steps, 1 if stop_at_events else 0,
                                   C.byref(res))
        self.be.check(st, res)
        return clock, res

    def last_run_ms(self) -> float:
        v = D()
        self.be.call("sim_last_run_ms", self.h, C.byref(v))
        return v.value

    def snapshot(self):
        self.be.call("sim_snapshot", self.h)

    def restore(self):
        self.be.call("sim_restore", self.h)

    def profile(self, steps: int) -> dict:
        """Per-kernel device time over `steps` steps: {name: (ms_total, launches)}."""
        ms = np.zeros(16)
        cnt = np.zeros(16, np.int64)
        nf = I32()
        self.be.call("sim_profile", self.h, steps, dptr(ms), cnt.ctypes.data_as(PI64), 16,
                     C.byref(nf))
        out = {}
        for f in range(nf.value):
            if cnt[f]:
                name = self.be.fn["sim_kernel_name"](self.h, f).decode()
                out[name] = (float(ms[f]), int(cnt[f]))
        return out


def default_clock(sc) -> c_clock:
    """The clock the parity harness and bench use: a 10 s gauge cadence so a
    dry domain advances by 10 s steps (SURVEY §8 d2 "Dry start"), no end in reach."""
    return c_clock(1e12, 0.0, 10.0, 0.0, 1, 1)


def isclose_flow(a: np.ndarray, b: np.ndarray, rel: float = 1e-9, abs_: float = 1e-10):
    """The north_star flow tolerance: |d| <= rel*|ref| or |d| <= abs (m, m^2/s)."""
    d = np.abs(a - b)
    return (d <= rel * np.abs(b)) | (d <= abs_)


__all__ = ["Backend", "Grid", "Sim", "FmError", "BlowUpError", "c_clock", "c_result",
           "default_clock", "isclose_flow", "math"]
