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
# virtual-rank simulation of the level-aligned owner-edge partition
# ---------------------------------------------------------------------------

def partition_bounds(off, efilt, world):
    """Re-implementation of the library's split (vrb_api.cu k_partition):
    bound g = first owner edge p with off[p] >= floor(T g / G), moved back to
    the start of its filtration level."""
    E = len(efilt)
    T = int(off[E])
    b = [0]
    for g in range(1, world):
        target = (T * g) // world
        p = int(np.searchsorted(off[: E + 1], target, side="left"))
        p = min(p, E)
        while 0 < p < E and efilt[p - 1] == efilt[p]:
            p -= 1
        b.append(p)
    b.append(E)
    return b


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
        for world in (1, 2, 3, 4, 8):
            b = partition_bounds(off, ef, world)
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
