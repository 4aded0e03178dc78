#!/usr/bin/env python
"""Benchmark of the B200 hot path on BASELINE.json's headline configuration.

Workload (config 4, the 8192^2 urban case the north_star's roofline and
scaling targets are quoted on): multiwavelet MRA (L = 13, eps = 1e-3) of the
seeded synthetic DEM, then static non-uniform DG2 RK2 steps under the 50 mm/h
rain on the resulting ~2.3 M leaves.  A "step" is one RK2 step of every leaf
(cell-updates/s = leaves x steps / time).  Synthetic inputs (DESIGN.md
§6); state ~0.7 GB > the 126 MB L2, so no flush is needed between steps.
With N GPUs (torchrun) the same domain is split into N Morton-range shards
with NCCL halo exchanges (strong scaling: total work fixed).

Legs:
  value    device loop (CUDA graph) with the DEM resident in HBM, CUDA-event time
           of exactly K steps, max over ranks;
  e2e      the public API from host buffers: DEM upload, fm_mra_static,
           fm_sim_create, K steps, final-state download, wall-clock;
  roofline the dominant kernel (k_stage<2>) from a per-launch CUDA-event profile;
  cpu_baseline  the reference library (oracle/_ref, built from the reference's own
           sources) on the host cores, on a bounded sample of the workload.
`--impl reference` runs only the reference arm and prints its line.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2107_02750_b200 import scenarios as S  # noqa: E402
from paper_2107_02750_b200.abi import Backend, c_clock  # noqa: E402

METRIC = "DG2/ACC cell-updates/s and MRA coeffs/s; % of B200 HBM roofline"
UNIT = "cell-updates/s"
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfmref.so")
ORC_SO = os.path.join(ROOT, "oracle", "liboracle.so")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9 and f[1].isdigit():
                    rows.append(f)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def allreduce_max(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def reference_backend():
    if os.path.exists(REF_SO):
        return Backend(REF_SO, "ref_"), "reference"
    return Backend(ORC_SO, "orc_"), "port"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_rate(steps: int, warmup: int, scale: int = 1, serial_steps: int = 2):
    """The reference CPU path on the SAME workload as the GPU line (config 4,
    8192^2, L = 13, static non-uniform DG2): the unmodified
    reference library builds the grid and the sim once (setup untimed), runs
    `warmup` steps, then times `steps` DG2 steps with every host thread and
    `serial_steps` more with one thread (run.cpp:79-113 times the step loop
    only).  The sample is bounded by the step count, not by the grid."""
    be, kind = reference_backend()
    cores = os.cpu_count() or 1
    threaded = be.has("set_threads")
    if threaded:
        be.fn["set_threads"](cores)
    else:
        cores = 1
    sc = S.config4(scale)
    t_setup = time.perf_counter()
    g = be.grid(sc.dem, sc.L, sc.eps)
    s = be.sim(sc, g)
    setup_s = time.perf_counter() - t_setup
    ck, _ = s.run(warmup, gauge_interval=10.0)
    t0 = time.perf_counter()
    ck, r = s.run(steps, clock=ck)
    dt = time.perf_counter() - t0
    n = s.num_cells
    out = {"value": n * r.steps / dt, "unit": UNIT, "cores": cores, "kind": kind,
           "cpu_model": cpu_model(), "nproc": os.cpu_count() or 1,
           "workload": "c4_static_nonuniform_dg2", "leaves": int(n),
           "setup_s": round(setup_s, 2),
           "sample": f"config 4 full size ({8192 // scale}^2 cells, L={sc.L}, {n} leaves): "
                     f"{r.steps} timed DG2 steps after {warmup} warm-up, {cores} threads, "
                     f"{dt:.2f} s; grid + sim setup {setup_s:.1f} s untimed"}
    if threaded and serial_steps > 0:
        be.fn["set_threads"](1)
        t1 = time.perf_counter()
        ck, r1 = s.run(serial_steps, clock=ck)
        d1 = time.perf_counter() - t1
        be.fn["set_threads"](cores)
        out["threads1"] = {"value": n * r1.steps / d1, "steps": int(r1.steps), "seconds": round(d1, 2)}
    return out, r.steps, dt


def run_reference(args, ws, rank):
    if rank != 0:
        return
    steps = max(1, min(args.steps, args.cpu_steps_cap))
    cb, n_done, secs = cpu_rate(steps, args.warmup, serial_steps=0)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": n_done, "warmup": args.warmup,
            "ms_per_step": 1000.0 * secs / max(n_done, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c4_static_nonuniform_dg2", "cells": "8192^2", "L": 13, "eps": 1e-3,
                       "leaves": cb["leaves"], "same_config": True,
                       "sample": cb["sample"],
                       "steps_note": f"K={args.steps} requested, {n_done} timed (cap --cpu-steps-cap)"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import torch

    from paper_2107_02750_b200 import api

    lib = api.lib()
    sc = S.config4(args.scale)
    hbm, peak_kind = peaks()

    # ---- value leg: DEM resident in HBM, device loop, CUDA-event timing ----
    dem_d = torch.from_numpy(np.ascontiguousarray(sc.dem.values)).to(f"cuda:{local}")
    torch.cuda.synchronize()
    # MRA: three untimed builds (the stream-ordered pool's first allocations
    # of the ~2 GB of pyramids run 2-4x slower than steady state), then the
    # measured one; the grid of the measured build feeds the sim
    for _ in range(3):
        del_grid = lib.grid(sc.dem, sc.L, sc.eps, device_ptr=dem_d.data_ptr())
        del del_grid
    grid = lib.grid(sc.dem, sc.L, sc.eps, device_ptr=dem_d.data_ptr())
    mra_ms, mra_bytes = grid.timing()
    n_int = (4 ** sc.L - 1) // 3
    # N > 1: the same domain split into N Morton-range shards,
    # halo exchanges and the dt reduction over NCCL inside each step's graph
    comm = None
    if ws > 1:
        import torch.distributed as dist
        uid = [lib.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = lib.comm_nccl(ws, rank, uid[0])
    elif args.force_shard:  # the sharded path on one GPU (a 1-rank NCCL communicator)
        comm = lib.comm_nccl(1, 0, lib.comm_unique_id())

    def make_sim(g):
        return lib.shard_sim(sc, g, comm, rank) if comm is not None else lib.sim(sc, g)

    sim = make_sim(grid)
    n_leaves, n_seg = sim.num_cells, sim.num_segments
    n_global = sim.shard_info()["n_global"] if comm is not None else n_leaves
    ck, r = sim.run(args.warmup, gauge_interval=10.0)
    # The reference DG2 scheme (no slope limiter) is unstable under this forcing:
    # the CFL step of the still 0.14 mm film after the first dry step is 8.9 s,
    # its update overshoots at the building walls and dt then collapses
    # (profiles/c4_dynamics_r1.txt).  So the K timed steps run in
    # chunks that each restart from the post-warm-up state (device-side
    # snapshot, restored outside the timed region): every leaf is wet there.
    sim.snapshot()
    ck0 = (ck.end_time, ck.output_interval, ck.gauge_interval, ck.now, ck.next_output,
           ck.next_gauge)
    ms = 0.0
    done = 0
    launches = 0
    with Clocks(local) as clocks:
        while done < args.steps:
            n = min(args.chunk, args.steps - done)
            sim.restore()
            ckc = c_clock(*ck0)
            barrier(ws)
            torch.cuda.synchronize()
            launches0 = api.launch_count()
            ckc, r = sim.run(n, clock=ckc)
            torch.cuda.synchronize()
            launches += api.launch_count() - launches0
            barrier(ws)
            if r.steps != n:
                raise SystemExit(f"only {r.steps} of {n} steps ran (blew_up={r.blew_up})")
            ms += sim.last_run_ms()
            done += n
    ms_max = allreduce_max(ms, ws)
    cells_total = allreduce_sum(float(n_leaves) * args.steps, ws)
    value = cells_total / (ms_max / 1000.0)

    # ---- roofline of the dominant kernel (per-launch CUDA events) ----
    sim.restore()
    prof = sim.profile(args.profile_steps)
    stage2_ms, stage2_n = prof.get("k_stage<2>", (0.0, 1))
    avg_ms = stage2_ms / max(stage2_n, 1)
    # DG2 stage 2 reads U^n 72 + U* 72 + z 24 + n 8, writes 72 B per
    # leaf, + 8 B of segment indices per segment
    bytes_launch = 248.0 * n_leaves + 8.0 * n_seg
    achieved = bytes_launch / (avg_ms / 1000.0) / 1e9
    step_ms = sum(v[0] for v in prof.values()) / max(args.profile_steps, 1)
    step_bytes = 424.0 * n_leaves + 16.0 * n_seg
    # dram__bytes_read.sum + dram__bytes_write.sum per launch of k_stage<2>
    # cannot be counted inside this (un-profiled) run: it is read from the
    # committed ncu capture of the same build, named in traffic_source
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("k_stage<2>")
            traffic_src = tj.get("source", "profiles/ncu_traffic.json")
        except Exception:
            traffic = None
    del sim
    solvers = None
    if ws == 1 and args.solver_steps > 0:
        solvers = {name: static_solver_leg(lib, sc, grid, name, cour, bpl, bps, args, hbm)
                   for name, cour, bpl, bps in (("acc", 0.7, 48.0, 24.0), ("fv1", 0.5, 64.0, 8.0))}
    del grid, dem_d

    # ---- e2e leg: public API from host buffers, wall clock ----
    # inputs (DEM, Manning raster) and outputs (final state) in pinned host
    # memory, allocated before the timed region; the copies are inside it
    import dataclasses

    def pinned(a, dtype=np.float64):
        # zero-filled: the host pages are touched when the buffer is made,
        # not by the first transfer into it
        t = torch.zeros(a.shape if hasattr(a, "shape") else a, dtype=getattr(torch, np.dtype(dtype).name),
                        pin_memory=True)
        arr = t.numpy()
        if hasattr(a, "shape"):
            arr[...] = a
        return t, arr

    keep = []
    t_dem, dem_p = pinned(sc.dem.values)
    t_man, man_p = pinned(sc.manning_raster.values)
    keep += [t_dem, t_man]
    sc_p = dataclasses.replace(
        sc, dem=dataclasses.replace(sc.dem, values=dem_p),
        manning_raster=dataclasses.replace(sc.manning_raster, values=man_p))
    outs = []
    for shape, dt in (((n_leaves,), np.int32), ((n_leaves,), np.int32), ((n_leaves,), np.int32),
                      ((n_leaves, 9), np.float64), ((n_leaves, 3), np.float64)):
        t_o, a_o = pinned(shape, dt)
        keep.append(t_o)
        outs.append(a_o)
    barrier(ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ph = {}
    g2 = lib.grid(sc_p.dem, sc_p.L, sc_p.eps)
    ph["upload_mra"] = time.perf_counter()
    s2 = lib.shard_sim(sc_p, g2, comm, rank) if comm is not None else lib.sim(sc_p, g2)
    ph["sim_create"] = time.perf_counter()
    ck2, r2 = s2.run(args.warmup, gauge_interval=10.0)
    s2.snapshot()
    ck0 = (ck2.end_time, ck2.output_interval, ck2.gauge_interval, ck2.now, ck2.next_output,
           ck2.next_gauge)
    ph["warmup"] = time.perf_counter()
    done = 0
    while done < args.steps:
        n = min(args.chunk, args.steps - done)
        s2.restore()
        _, r2 = s2.run(n, clock=c_clock(*ck0))
        done += r2.steps
    ph["steps"] = time.perf_counter()
    out = s2.download(out=outs)
    ph["download"] = time.perf_counter()
    e2e_s = time.perf_counter() - t0
    prev, phases = t0, {}
    for k, v in ph.items():
        phases[k] = round(1000.0 * (v - prev), 2)
        prev = v
    e2e_s = allreduce_max(e2e_s, ws)
    h2d = sc.dem.values.nbytes + sc.manning_raster.values.nbytes
    d2h = sum(a.nbytes for a in out)
    e2e_steps = args.warmup + args.steps
    e2e_value = allreduce_sum(float(n_leaves) * e2e_steps, ws) / e2e_s
    del s2, g2, outs, keep

    # ---- config 4's comparator: the uniform raster at the finest level ----
    uni = None
    if args.uniform_steps > 0:
        uni = uniform_leg(lib, args, ws, rank, comm, hbm)
    comm = None

    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu:
        cpu, _, _ = cpu_rate(args.cpu_steps, args.warmup)
    configs = None
    if ws == 1 and not args.no_configs:
        configs = config_legs(lib, args, with_cpu=not args.no_cpu)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c4_static_nonuniform_dg2", "cells": f"{8192 // args.scale}^2",
                   "L": sc.L, "eps": sc.eps, "leaves": n_global, "segments_rank0": n_seg,
                   "leaves_rank0": n_leaves,
                   "parallelism": f"morton-shards x{ws} (NCCL halo + min-allreduce)" if ws > 1
                   else "single",
                   "l2": "state > 126 MB L2 (no flush needed)",
                   "solver": "static non-uniform DG2 RK2, rain 50 mm/h, Manning street raster"},
        "roofline": {"bound": "hbm", "kernel": "k_stage<2>", "achieved": achieved, "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "bytes_per_launch": bytes_launch,
                     "bytes_formula": "248*N_l + 8*N_s (SURVEY §8 d4, DG2 stage 2)",
                     "avg_launch_ms": avg_ms,
                     "step": {"bytes": step_bytes, "ms": step_ms,
                              "achieved": step_bytes / (step_ms / 1000.0) / 1e9,
                              "frac": step_bytes / (step_ms / 1000.0) / 1e9 / hbm},
                     "kernels_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in prof.items()}},
        "mra": {"coeffs_per_s": 12.0 * n_int / (mra_ms / 1000.0), "ms": mra_ms,
                "bytes": mra_bytes,
                "bytes_formula": "8*(n+1)^2 + 73*N_int + 36*N_l (SURVEY §8 d4, projection fused)", "achieved_gbs": mra_bytes / (mra_ms / 1000.0) / 1e9,
                "frac": mra_bytes / (mra_ms / 1000.0) / 1e9 / hbm},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps, "seconds": e2e_s, "phases_ms": phases,
                "what": "host DEM -> fm_mra_static -> fm_sim_create(_shard) -> W+K steps -> host state"},
        "uniform": uni,
        "solvers": solvers,
        "configs": configs,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def static_solver_leg(lib, sc, grid, solver, courant, b_leaf, b_seg, args, hbm):
    """Config 4's static grid (the same 2.3 M leaves) under the ACC or FV1
    update: SURVEY §8 d4 bytes per step, b_leaf*N_l + b_seg*N_s (ACC 48/24,
    FV1 64/8), against the CUDA-event step time and per-kernel launch times."""
    import dataclasses

    import torch
    sc2 = dataclasses.replace(sc, solver=solver, courant=courant)
    sim = lib.sim(sc2, grid)
    n, ns = sim.num_cells, sim.num_segments
    ck, _ = sim.run(args.warmup, gauge_interval=10.0)
    sim.snapshot()
    ck0 = (ck.end_time, ck.output_interval, ck.gauge_interval, ck.now, ck.next_output, ck.next_gauge)
    ms, done = 0.0, 0
    while done < args.solver_steps:
        k = min(args.chunk, args.solver_steps - done)
        sim.restore()
        torch.cuda.synchronize()
        _, r = sim.run(k, clock=c_clock(*ck0))
        torch.cuda.synchronize()
        if r.steps != k:
            raise SystemExit(f"{solver}: only {r.steps} of {k} steps ran")
        ms += sim.last_run_ms()
        done += k
    sim.restore()
    prof = sim.profile(args.profile_steps)
    step_bytes = b_leaf * n + b_seg * ns
    per = {k: v[0] / max(args.profile_steps, 1) for k, v in prof.items()}
    top = max(per, key=per.get)
    prof_step = sum(per.values())
    ms_step = ms / args.solver_steps
    del sim
    return {"workload": f"c4_static_nonuniform_{solver}", "leaves": int(n), "segments": int(ns),
            "steps": args.solver_steps, "ms_per_step": ms_step, "value": n / (ms_step / 1000.0),
            "unit": UNIT,
            "roofline": {"bound": "hbm", "bytes_per_step": step_bytes,
                         "bytes_formula": f"{b_leaf:g}*N_l + {b_seg:g}*N_s (SURVEY §8 d4)",
                         "achieved": step_bytes / (ms_step / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": step_bytes / (ms_step / 1000.0) / 1e9 / hbm,
                         "profiled_step_ms": prof_step, "top_kernel": top},
            "kernels_ms_per_step": per}


def uniform_leg(lib, args, ws, rank, comm, hbm):
    """Config 4's "uniform-raster DG2 at the finest level": 8192^2 cells, the
    same forcing; N > 1: row bands with one ghost row each side (NCCL)."""
    import torch
    sc = S.config4(args.scale, uniform=True)
    sim = lib.shard_sim(sc, None, comm, rank) if comm is not None else lib.sim(sc, None)
    n = sim.num_cells
    ck, _ = sim.run(3, gauge_interval=10.0)
    sim.snapshot()
    ck0 = (ck.end_time, ck.output_interval, ck.gauge_interval, ck.now, ck.next_output, ck.next_gauge)
    ms = 0.0
    done = 0
    while done < args.uniform_steps:
        k = min(args.chunk, args.uniform_steps - done)
        sim.restore()
        barrier(ws)
        torch.cuda.synchronize()
        _, r = sim.run(k, clock=c_clock(*ck0))
        torch.cuda.synchronize()
        barrier(ws)
        if r.steps != k:
            raise SystemExit(f"uniform: only {r.steps} of {k} steps ran")
        ms += sim.last_run_ms()
        done += k
    ms_max = allreduce_max(ms, ws)
    total = allreduce_sum(float(n) * args.uniform_steps, ws)
    sim.restore()
    prof = sim.profile(3)
    st2_ms, st2_n = prof.get("k_uni_march<2>", (0.0, 1))
    avg = st2_ms / max(st2_n, 1)
    bytes_launch = 248.0 * n  # U^n 72 + U* 72 + z 24 + n 8 read, 72 written per cell
    del sim
    return {"workload": "c4_uniform_dg2", "cells": int(allreduce_sum(float(n), ws)),
            "value": total / (ms_max / 1000.0), "unit": UNIT, "steps": args.uniform_steps,
            "ms_per_step": ms_max / args.uniform_steps,
            "parallelism": f"row-bands x{ws}" if ws > 1 else "single",
            "roofline": {"bound": "hbm", "kernel": "k_uni_march<2>",
                         "achieved": bytes_launch / (avg / 1000.0) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": bytes_launch / (avg / 1000.0) / 1e9 / hbm, "avg_launch_ms": avg},
            "kernels_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in prof.items()}}


CONFIG_LEGS = [
    # (name, scenario factory, static grid?, GPU steps, CPU steps)
    ("c0_static_dg2", lambda: S.config0(1), True, 100, 20),
    ("c1_static_acc", lambda: S.config1(1), True, 400, 40),
    ("c2_static_fv1", lambda: S.config2(1, adaptive=False), True, 400, 40),
    ("c2_adaptive_hwfv1", lambda: S.config2(1), False, 100, 5),
    ("c3_adaptive_mwdg2", lambda: S.config3(1), False, 50, 3),
]


def _leg(be, sc, static, warm, steps, device_time):
    g = be.grid(sc.dem, sc.L, sc.eps) if static else None
    s = be.sim(sc, g)
    ck, _ = s.run(warm, gauge_interval=10.0)
    t0 = time.perf_counter()
    ck, r = s.run(steps, clock=ck)
    wall = time.perf_counter() - t0
    ms = s.last_run_ms() if device_time else 1000.0 * wall
    if static:
        cells = float(s.num_cells) * r.steps
    else:  # adaptive: the leaf count of every step (element_log, one entry per adapt)
        _, counts = s.element_log()
        cells = float(np.sum(counts[-r.steps:])) if len(counts) else float(s.num_cells) * r.steps
    out = {"leaves": int(s.num_cells), "steps": int(r.steps), "ms_per_step": ms / max(r.steps, 1),
           "value": cells / (ms / 1000.0)}
    if device_time and not static and be.has("sim_adapt_stats"):
        # SURVEY §8 d4 per adapted step: the adapt (MW: 72 N_l + 360 N_enc +
        # N_int + 108 N_l' + 32 N_s'; HW: 24 / 120 / 36 for 72 / 360 / 108)
        # plus the flow step (MWDG2: DG2 424 N_l + 16 N_s; HWFV1: FV1 64 N_l + 8 N_s)
        st = s.adapt_stats()
        nl, ns, ne, ni = float(s.num_cells), float(s.num_segments), st["n_encoded"], st["n_internal"]
        mw = sc.solver == "mwdg2"
        a, b, c = (72.0, 360.0, 108.0) if mw else (24.0, 120.0, 36.0)
        adapt_b = a * nl + b * ne + ni + c * nl + 32.0 * ns
        step_b = (424.0 * nl + 16.0 * ns) if mw else (64.0 * nl + 8.0 * ns)
        sec = out["ms_per_step"] / 1000.0
        hbm, _ = peaks()
        out["roofline"] = {"bound": "hbm", "adapt_bytes": adapt_b, "step_bytes": step_b,
                           "n_encoded": int(ne), "n_internal": int(ni),
                           "achieved": (adapt_b + step_b) / sec / 1e9,
                           "frac": (adapt_b + step_b) / sec / 1e9 / hbm}
    return out


def config_legs(lib, args, with_cpu):
    """Every BASELINE config on one GPU (full size), and the reference on the
    host cores on a bounded number of steps of the same run."""
    out = {}
    ref = None
    if with_cpu:
        ref, kind = reference_backend()
        if ref.has("set_threads"):
            ref.fn["set_threads"](os.cpu_count() or 1)
    # every GPU leg first: the small configs are launch-bound, and a host that
    # has just run the 16-thread reference launches graphs measurably slower
    for name, mk, static, gsteps, csteps in CONFIG_LEGS:
        out[name] = {"gpu": _leg(lib, mk(), static, 3, gsteps, True)}
    if ref is not None:
        for name, mk, static, gsteps, csteps in CONFIG_LEGS:
            d = out[name]
            d["cpu_reference"] = _leg(ref, mk(), static, 1, csteps, False)
            d["cpu_reference"]["threads"] = os.cpu_count() or 1
            d["speedup"] = d["gpu"]["value"] / d["cpu_reference"]["value"]
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--scale", type=int, default=1, help="shrink config 4 (tests only)")
    p.add_argument("--profile-steps", type=int, default=10)
    p.add_argument("--chunk", type=int, default=16, help="timed steps between state restores")
    p.add_argument("--cpu-steps", type=int, default=20)
    p.add_argument("--solver-steps", type=int, default=64,
                   help="timed steps of the config-4 ACC and FV1 legs (0: skip)")
    p.add_argument("--cpu-steps-cap", type=int, default=20)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--uniform-steps", type=int, default=32,
                   help="timed steps of the uniform-raster comparator (0: skip)")
    p.add_argument("--no-configs", action="store_true",
                   help="skip the per-config table (configs 0-3 on GPU and CPU)")
    p.add_argument("--force-shard", action="store_true",
                   help="N=1: run the sharded (NCCL) code path with a single rank")
    args = p.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_setup() if args.impl == "ours" else (
        int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
