"""Multi-rank sharding of static non-uniform sims.

CPU: the partition plan (fm_shard_plan, host code of libfm_gpu.so) on
reference topologies from the oracle relabelled to Morton order — partition,
halo and send-list invariants — and the exchange + reduction protocol run by
two gloo ranks (world_size 2), exactly the messages the NCCL path sends.

GPU: a local group of R shards on one device stepped by fm_group_run ends in
the same state bits as the unsharded sim (DG2, FV1, ACC; rain and point
sources; R = 2, 3)."""
import dataclasses
import os
import socket

import numpy as np
import pytest

from conftest import GPU_SO
from paper_2107_02750_b200 import scenarios as S


def _spread(v):
    v = v.astype(np.uint64) & np.uint64(0xFFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
    return v


def morton_relabel(L, lv, i, j, sl, sr):
    """Relabel reference-order leaves to the device's Morton order (M = N = 1):
    returns the permuted (lv, i, j) and the segments in the new indices."""
    sh = (L - lv).astype(np.uint64)
    fi = i.astype(np.uint64) << sh
    fj = j.astype(np.uint64) << sh
    key = _spread(fi) | (_spread(fj) << np.uint64(1))
    order = np.argsort(key, kind="stable")
    new = np.empty_like(order)
    new[order] = np.arange(len(order))
    return lv[order], i[order], j[order], new[sl].astype(np.int32), new[sr].astype(np.int32)


def cpu_lib():
    from paper_2107_02750_b200.abi import Backend
    return Backend(GPU_SO, "fm_")


def oracle_topology(orc, sc):
    g = orc.grid(sc.dem, sc.L, sc.eps)
    s = orc.sim(sc, g)
    lv, i, j, sl, sr = s.topology()
    return morton_relabel(sc.L, lv, i, j, sl, sr)


TOPOS = {"c0_s4": lambda: S.config0(4), "c4_s16": lambda: S.config4(16), "c1_s8": lambda: S.config1(8)}


@pytest.mark.parametrize("name", list(TOPOS))
@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_plan_partition_halo_and_send_lists(orc, name, nranks):
    sc = TOPOS[name]()
    lv, i, j, sl, sr = oracle_topology(orc, sc)
    n = len(lv)
    lib = cpu_lib()
    plans = [lib.shard_plan(n, sl, sr, nranks, r) for r in range(nranks)]
    # contiguous partition of [0, n)
    assert plans[0]["first"] == 0
    for r in range(nranks - 1):
        assert plans[r]["first"] + plans[r]["count"] == plans[r + 1]["first"]
    assert plans[-1]["first"] + plans[-1]["count"] == n
    owner = np.zeros(n, np.int32)
    for r, p in enumerate(plans):
        owner[p["first"]:p["first"] + p["count"]] = r
    for r, p in enumerate(plans):
        mine = (owner[sl] == r) | (owner[sr] == r)
        assert p["nseg_local"] == int(mine.sum())
        ends = np.concatenate([sl[mine], sr[mine]])
        halo = np.unique(ends[owner[ends] != r])
        assert np.array_equal(p["halo"], halo)
        assert np.array_equal(p["halo_owner"], owner[halo])
        for q in range(nranks):
            if q == r:
                assert len(p["send"][q]) == 0
                continue
            # what r sends to q is exactly q's halo slice owned by r, same order
            hq = plans[q]["halo"][plans[q]["halo_owner"] == r]
            assert np.array_equal(p["send"][q], hq)
            assert (owner[p["send"][q]] == r).all()
    # Morton ranges are compact: the halo is a small fraction of the shard
    if n > 10000:
        assert max(len(p["halo"]) for p in plans) < 0.1 * n / nranks


def _gloo_worker(rank, world, port, n, sl, sr, dtc, keys, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lib = cpu_lib()
        p = lib.shard_plan(n, sl, sr, world, rank)
        ntot = p["count"] + len(p["halo"])
        # state: 9 doubles per local leaf; owned leaves carry (global id, id^2, ...)
        u = np.full((ntot, 9), np.nan)
        gid = np.arange(p["first"], p["first"] + p["count"], dtype=np.float64)
        for q in range(9):
            u[:p["count"], q] = gid * (q + 1)
        # one exchange: pack per peer, send/recv, land in the halo slots
        reqs = []
        recv = {}
        for q in range(world):
            if q == rank:
                continue
            send = p["send"][q]
            if len(send):
                buf = torch.from_numpy(np.ascontiguousarray(u[send - p["first"]]).reshape(-1))
                reqs.append(dist.isend(buf, q))
            nh = int((p["halo_owner"] == q).sum())
            if nh:
                recv[q] = torch.empty(9 * nh, dtype=torch.float64)
                reqs.append(dist.irecv(recv[q], q))
        for r_ in reqs:
            r_.wait()
        for q, t in recv.items():
            sel = np.nonzero(p["halo_owner"] == q)[0]
            u[p["count"] + sel] = t.numpy().reshape(-1, 9)
        halo_ok = bool(np.array_equal(u[p["count"]:, 0], p["halo"].astype(np.float64)) and
                       np.array_equal(u[p["count"]:, 8], 9.0 * p["halo"]))
        # the reduction slot: min of the CFL candidates and of the bad keys
        own = slice(p["first"], p["first"] + p["count"])
        slot = torch.tensor([np.min(dtc[own]), np.min(keys[own])], dtype=torch.float64)
        dist.all_reduce(slot, op=dist.ReduceOp.MIN)
        out_q.put((rank, halo_ok, slot.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_two_rank_exchange_and_reduction(orc):
    import torch.multiprocessing as mp
    sc = S.config0(4)
    lv, i, j, sl, sr = oracle_topology(orc, sc)
    n = len(lv)
    rng = np.random.default_rng(3)
    dtc = rng.uniform(0.1, 10.0, n)
    keys = rng.integers(0, 2 ** 40, n).astype(np.float64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, n, sl, sr, dtc, keys, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, slot in res:
        assert ok, f"rank {rank}: halo slots hold the wrong leaves"
        assert slot == [dtc.min(), keys.min()]


# ---------------------------------------------------------------------- GPU

SHARD_CASES = {
    "c0_dg2_s4": (lambda: S.config0(4), 30),
    "c4_dg2_rain_s8": (lambda: S.config4(8), 20),
    "c2_fv1_s8": (lambda: S.config2(8, adaptive=False), 30),
    "c1_acc_s8": (lambda: S.config1(8), 30),
}


def _merged(shards):
    parts = [s.download() for s in shards]
    lv, i, j, u, z = (np.concatenate([p[k] for p in parts]) for k in range(5))
    order = np.lexsort((i, j, lv))
    return lv[order], i[order], j[order], u[order], z[order]


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("name", list(SHARD_CASES))
def test_local_group_matches_unsharded_bit_exact(gpu, name, nranks):
    mk, steps = SHARD_CASES[name]
    sc = mk()
    g = gpu.grid(sc.dem, sc.L, sc.eps)
    ref = gpu.sim(sc, g)
    ck_a, ra = ref.run(steps, gauge_interval=10.0)
    comm = gpu.comm_local(nranks)
    shards = [gpu.shard_sim(sc, g, comm, r) for r in range(nranks)]
    info = [s.shard_info() for s in shards]
    assert sum(x["owned"] for x in info) == ref.num_cells
    assert all(x["halo"] > 0 for x in info)
    ck_b, rb = gpu.group_run(shards, steps, gauge_interval=10.0)
    assert (ra.steps, ra.dt_min, ra.dt_max, ck_a.now) == (rb.steps, rb.dt_min, rb.dt_max, ck_b.now)
    a = ref.download()
    b = _merged(shards)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.gpu
def test_shard_rejects_adaptive(gpu):
    from paper_2107_02750_b200.abi import FmError
    comm = gpu.comm_local(2)
    sc = S.config2(8)  # HWFV1: re-grids every step, replicas only
    with pytest.raises(FmError):
        gpu.shard_sim(sc, None, comm, 0)


UNIFORM_CASES = {
    "c4_uniform_dg2_rain_s32": (lambda: S.config4(32, uniform=True), 20),
    "c0_uniform_dg2_s4": (lambda: dataclasses.replace(S.config0(4), grid_mode="uniform"), 25),
    "c1_uniform_acc_s8": (lambda: dataclasses.replace(S.config1(8), grid_mode="uniform"), 30),
    "c2_uniform_fv1_s8": (lambda: dataclasses.replace(S.config2(8, adaptive=False),
                                                      grid_mode="uniform"), 30),
}


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("name", list(UNIFORM_CASES))
def test_uniform_bands_match_unsharded_bit_exact(gpu, name, nranks):
    """Row-band shards of the uniform raster (one ghost row each side)."""
    mk, steps = UNIFORM_CASES[name]
    sc = mk()
    ref = gpu.sim(sc, None)
    ck_a, ra = ref.run(steps, gauge_interval=10.0)
    comm = gpu.comm_local(nranks)
    shards = [gpu.shard_sim(sc, None, comm, r) for r in range(nranks)]
    info = [s.shard_info() for s in shards]
    assert sum(x["owned"] for x in info) == ref.num_cells
    ck_b, rb = gpu.group_run(shards, steps, gauge_interval=10.0)
    assert (ra.steps, ra.dt_min, ra.dt_max, ck_a.now) == (rb.steps, rb.dt_min, rb.dt_max, ck_b.now)
    a = ref.download()
    parts = [s.download() for s in shards]  # j-major bands in rank order
    for k in range(5):
        assert np.array_equal(a[k], np.concatenate([p[k] for p in parts]))
    # rasters: the bands stack (row 0 north: the last band first)
    full = ref.raster(0)
    assert np.array_equal(full, np.concatenate([s.raster(0) for s in shards[::-1]]))


@pytest.mark.gpu
def test_nccl_single_rank_shard_runs_the_graph_path(gpu):
    """The NCCL transport end to end on one GPU: a 1-rank communicator, the
    shard's device loop captured in a CUDA graph with the ncclAllReduce of the
    reduction slots inside, equal to the unsharded run bit for bit.  (Peer
    exchanges need >= 2 GPUs; their plan and protocol are covered above.)"""
    sc = S.config0(4)
    g = gpu.grid(sc.dem, sc.L, sc.eps)
    ref = gpu.sim(sc, g)
    ck_a, ra = ref.run(40, gauge_interval=10.0)
    comm = gpu.comm_nccl(1, 0, gpu.comm_unique_id())
    sh = gpu.shard_sim(sc, g, comm, 0)
    ck_b, rb = sh.run(40, gauge_interval=10.0)
    assert (ra.steps, ck_a.now) == (rb.steps, ck_b.now)
    for x, y in zip(ref.download(), sh.download()):
        assert np.array_equal(x, y)
    assert sh.compute_dt() == ref.compute_dt()


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_device_plan_matches_host_plan(gpu, nranks):
    """The shards built on the device (segment classification + stream
    compaction) hold exactly the plan of the host function the CPU tests
    check: owned range, halo size and the local segment count."""
    sc = S.config4(16)
    g = gpu.grid(sc.dem, sc.L, sc.eps)
    glob = gpu.sim(sc, g)
    lv, i, j, sl, sr = glob.topology()
    n = glob.num_cells
    comm = gpu.comm_local(nranks)
    for r in range(nranks):
        p = gpu.shard_plan(n, sl, sr, nranks, r)
        sh = gpu.shard_sim(sc, g, comm, r)
        info = sh.shard_info()
        assert (info["first"], info["owned"], info["halo"]) == (p["first"], p["count"], len(p["halo"]))
        assert sh.num_segments == p["nseg_local"]
        del sh


# ------------------------------------------- host transport, real processes

HOST_CASES = {
    "c0_dg2_s4": (lambda: S.config0(4), 30, True),
    "c1_acc_s8": (lambda: S.config1(8), 30, True),
    "c2_fv1_s8": (lambda: S.config2(8, adaptive=False), 30, True),
    "c4_uniform_dg2_s32": (lambda: S.config4(32, uniform=True), 20, False),
}


def _host_rank(name, nranks, rank, shm, out_q):
    """One rank in its own process: the library's shard code (pack, halo
    slots, reduction) over the host transport; reports its owned state."""
    try:
        from paper_2107_02750_b200 import api
        lib = api.lib()
        mk, steps, static = HOST_CASES[name]
        sc = mk()
        comm = lib.comm_host(nranks, rank, shm)
        g = lib.grid(sc.dem, sc.L, sc.eps) if static else None
        sh = lib.shard_sim(sc, g, comm, rank)
        ck, r = sh.run(steps, gauge_interval=10.0)
        dt = sh.compute_dt()
        vol = sh.volume()
        ok, _, _ = sh.finite_state()
        out_q.put((rank, (r.steps, r.dt_min, r.dt_max, ck.now, dt, vol, ok), sh.download()))
        del sh
    except Exception as e:  # surfaced by the parent
        out_q.put((rank, repr(e), None))


def _handshake(nranks, rank, shm, out_q):
    lib = cpu_lib()
    c = lib.comm_host(nranks, rank, shm)  # returns only once every rank has mapped the segment
    out_q.put(rank)
    del c


def test_host_comm_handshake_across_processes():
    """CPU: the host transport's segment and barrier across real processes
    (no device needed to create and join it)."""
    import multiprocessing as mp
    import uuid
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    shm = f"/fm_test_{uuid.uuid4().hex[:12]}"
    procs = [ctx.Process(target=_handshake, args=(3, r, shm, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [0, 1, 2]
    assert not os.path.exists("/dev/shm" + shm)  # rank 0 unlinked it


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("name", list(HOST_CASES))
def test_host_transport_processes_match_unsharded_bit_exact(gpu, name, nranks):
    """nranks processes, one shard each, exchanging halos and reduction slots
    through fm_comm_create_host (shared memory), end in the unsharded sim's
    state bits; the host-API collectives (compute_dt, finite_state) agree and
    volume() is the rank-order sum of the shards' audits."""
    import multiprocessing as mp
    import uuid
    mk, steps, static = HOST_CASES[name]
    sc = mk()
    g = gpu.grid(sc.dem, sc.L, sc.eps) if static else None
    ref = gpu.sim(sc, g)
    ck_a, ra = ref.run(steps, gauge_interval=10.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    shm = f"/fm_test_{uuid.uuid4().hex[:12]}"
    procs = [ctx.Process(target=_host_rank, args=(name, nranks, r, shm, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    for rank, stats, _ in res:
        assert not isinstance(stats, str), f"rank {rank}: {stats}"
    for p in procs:
        assert p.exitcode == 0
    for rank, stats, _ in res:
        steps_b, dtmin, dtmax, now, dt, vol, ok = stats
        assert (ra.steps, ra.dt_min, ra.dt_max, ck_a.now) == (steps_b, dtmin, dtmax, now)
        assert dt == ref.compute_dt() and ok
        assert vol == pytest.approx(ref.volume(), rel=1e-12)
    parts = [r[2] for r in res]
    a = ref.download()
    if static:
        lv, i, j, u, z = (np.concatenate([p[k] for p in parts]) for k in range(5))
        order = np.lexsort((i, j, lv))
        b = (lv[order], i[order], j[order], u[order], z[order])
    else:  # row bands in rank order
        b = tuple(np.concatenate([p[k] for p in parts]) for k in range(5))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
