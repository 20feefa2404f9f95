"""Multi-rank logic on CPU (no GPU): the gloo all-gather used by build_dist's
collective callback, and a virtual-rank simulation of the owner-edge
partition (pin P13: the concatenated slices equal the G = 1
arrays)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allgather_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_04424_b200 as vrb

        # each rank contributes a disjoint part of per-edge counts (others 0),
        # exactly like the library's count exchange; gather + sum = full counts
        E = 1000
        full = np.random.default_rng(0).integers(0, 500, E).astype(np.uint32)
        mine = np.where(np.arange(E) % world == rank, full, 0).astype(np.uint32)
        src = torch.from_numpy(mine.view(np.uint8).copy())
        dst = torch.empty(world * src.numel(), dtype=torch.uint8)
        vrb.allgather_bytes(src, dst)
        parts = dst.numpy().view(np.uint32).reshape(world, E)
        out_q.put((rank, bool((parts.sum(0) == full).all())))
    finally:
        dist.destroy_process_group()


def test_gloo_allgather_count_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allgather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


# ---------------------------------------------------------------------------
# virtual-rank simulation of the level-aligned owner-edge partition, driven
# by the library's own rule (any per-edge work vector; world up to 100)
# ---------------------------------------------------------------------------

def partition_bounds(work_prefix, efilt, world):
    """The library's owner-edge split (vrb_partition_bounds: the same
    __host__ __device__ function the multi-GPU build runs on the device)."""
    import paper_1809_04424_b200 as vrb
    return [int(x) for x in vrb.partition_bounds(np.asarray(work_prefix, dtype=np.uint64), efilt, world)]


def _owner(o, simplex):
    """owner edge of a simplex: its edge of largest position"""
    best = -1
    s = [int(x) for x in simplex]
    for i in range(len(s)):
        for j in range(i + 1, len(s)):
            best = max(best, o.edge_pos(s[i], s[j]))
    return best


@pytest.mark.parametrize("case", range(6))
def test_partition_slices_concatenate_to_global_order(case):
    kind = ["uniform", "lattice", "halfint", "gauss", "dups", "uniform"][case]
    X = workloads.random_cloud(4000 + case, [30, 27, 25, 35, 30, 3][case], 3, kind)
    radius = [0.6, 2.0, 1.6, 1.8, 0.7, math.inf][case]
    o = oracle.Oracle(X, radius)
    ev, ef, el, vor = o.edges()
    for k in (2, 3):
        v, f, r = o.simplices(k)
        owners = np.array([_owner(o, s) for s in v], dtype=np.int64)
        cnt = np.bincount(owners, minlength=o.E) if len(owners) else np.zeros(o.E, np.int64)
        off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        rng = np.random.default_rng(case)
        works = {"counts": off, "random": np.concatenate([[0], np.cumsum(rng.integers(0, 50, o.E))])}
        for (wname, wpre), world in [(w, g) for w in works.items() for g in (1, 2, 3, 4, 8, 64, 100)]:
            b = partition_bounds(wpre, ef, world)
            assert len(b) == world + 1
            assert b[0] == 0 and b[-1] == o.E and all(x <= y for x, y in zip(b, b[1:]))
            pieces = []
            for g in range(world):
                lo, hi = off[b[g]], off[b[g + 1]]
                sl = slice(int(lo), int(hi))
                # every simplex of the slice is owned by an edge of the rank's range
                assert ((owners[sl] >= b[g]) & (owners[sl] < b[g + 1])).all()
                # ranges start at level boundaries (ties are never split)
                if 0 < b[g] < o.E:
                    assert ef[b[g] - 1] != ef[b[g]]
                pieces.append(v[sl])
            cat = np.concatenate(pieces) if pieces else v[:0]
            assert np.array_equal(cat, v)


def test_partition_edge_slices():
    # edge level: rank g reports edges [E g / G, E (g + 1) / G)
    E = 1234
    for world in (1, 2, 4, 8):
        cuts = [E * g // world for g in range(world + 1)]
        assert cuts[0] == 0 and cuts[-1] == E
        assert sum(cuts[g + 1] - cuts[g] for g in range(world)) == E


def test_partition_bounds_balance_and_errors():
    import paper_1809_04424_b200 as vrb
    # distinct levels: the split lands at the first edge reaching g / G of the work
    E = 1000
    ef = np.arange(1, E + 1, dtype=np.uint32)
    pre = np.arange(E + 1, dtype=np.uint64) * 3
    b = vrb.partition_bounds(pre, ef, 4)
    assert b.tolist() == [0, 250, 500, 750, 1000]
    # one level for everything: a level is never split -> all on the last rank
    b = vrb.partition_bounds(pre, np.ones(E, dtype=np.uint32), 4)
    assert b.tolist() == [0, 0, 0, 0, 1000]
    # empty input
    assert vrb.partition_bounds(np.zeros(1, np.uint64), np.zeros(0, np.uint32), 3).tolist() == [0, 0, 0, 0]
    with pytest.raises(vrb.VrbError):
        vrb.partition_bounds(pre, ef, 0)


def _bcast_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_04424_b200 as vrb
        X = np.random.default_rng(1).standard_normal((50, 3))
        buf = torch.from_numpy(X.copy().view(np.uint8).reshape(-1)) if rank == 0 else torch.zeros(X.nbytes, dtype=torch.uint8)
        vrb.broadcast_bytes(buf, 0)
        out_q.put((rank, bool(np.array_equal(buf.numpy().view(np.float64).reshape(50, 3), X))))
    finally:
        dist.destroy_process_group()


def test_gloo_broadcast_points():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
