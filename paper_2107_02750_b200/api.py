"""Python binding of the product library libfm_gpu.so (include/fm_gpu.h).

Mirrors the reference's solver interface:
`generate_static_grid` (detail_tree.hpp:55-56) and simulation objects with the
drive<Sim> members compute_dt / step / apply_inflows / adapt / volume /
finite_state (run.cpp:35-141), plus `run`, the drive loop resident on the GPU.

There is no CPU fallback: loading fails loudly when the library was not built,
and every call fails with FmError("[cuda] ...") without a CUDA device.
"""
from __future__ import annotations

import os

from .abi import Backend, BlowUpError, FmError, Grid, Sim, c_clock, default_clock  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfm_gpu.so")

_lib: Backend | None = None


def lib() -> Backend:
    """The loaded product library (built by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() first "
                              "(there is no CPU fallback)")
        _lib = Backend(LIB_PATH, "fm_")
        dev = int(os.environ.get("LOCAL_RANK", "0"))
        _lib.call("init", dev)
    return _lib


def generate_static_grid(dem, eps: float, L: int, graded: bool = True, kind: int = 0) -> Grid:
    """generate_static_grid(dem, eps, L, graded, kind) on the GPU."""
    return lib().grid(dem, L, eps, graded, kind)


def make_sim(scenario, grid: Grid | None = None) -> Sim:
    """run_scenario's dispatch (run.cpp:145-164): adaptive solvers ignore `grid`."""
    return lib().sim(scenario, grid)


def launch_count() -> int:
    return int(lib().fn["launch_count"]())
