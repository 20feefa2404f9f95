"""vrb_build_dist with several ranks on ONE GPU (gloo process group, so the
ranks may share a device), checked against the ORACLE: the per-rank slices
concatenated in rank order must equal the oracle's arrays element by element
(pin P13), for world sizes 1..8, with length ties, tetrahedra,
ranks that own nothing (row blocks and owner-edge ranges both empty), only
rank 0 holding the points, and a build stream other than torch's current
stream."""
import json
import math
import os
import socket

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _u32(t):
    return t.cpu().numpy().view(np.uint32) if t.dtype == torch.int32 else t.cpu().numpy()


def _worker(rank, world, port, X, maxdim, radius, side_stream, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_04424_b200 as vrb

        torch.cuda.set_device(0)
        stream = torch.cuda.Stream() if side_stream else None
        pts = X if rank == 0 else None      # the library broadcasts rank 0's points
        res = vrb.build_dist(pts, maxdim=maxdim, radius=radius, n=X.shape[0], d=X.shape[1], stream=stream)
        if stream is not None:
            stream.synchronize()
        out = {"rank": rank}
        for k in range(1, maxdim + 2):
            g, off, n = res.count(k)
            v, f = res.simplices(k)
            out[k] = (g, off, n, _u32(v), _u32(f), _u32(res.boundary(k)))
        out["vor"] = res.rank_values().cpu().numpy()
        pos, death, ness = res.h0()   # every rank holds every edge: the whole H0 result
        out["h0"] = (_u32(pos), _u32(death), ness)
        q.put(out)
    except Exception as e:   # surface worker errors in the test
        q.put({"rank": rank, "error": repr(e)})
    finally:
        dist.destroy_process_group()


def run_dist(X, maxdim, radius, world, side_stream=False):
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, maxdim, radius, side_stream, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=900) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=120)
    for o in outs:
        assert "error" not in o, o
    return outs


def check_vs_oracle(outs, X, maxdim, radius):
    o = oracle.Oracle(X, radius)
    ev, ef, _, vor = o.edges()
    want = {1: (ev, ef, ev)}
    for k in range(2, maxdim + 2):
        want[k] = o.simplices(k)
    for k in range(1, maxdim + 2):
        v, f, r = want[k]
        g = v.shape[0]
        assert all(out[k][0] == g for out in outs), k
        offs = [out[k][1] for out in outs]
        ns = [out[k][2] for out in outs]
        # contiguous slices in rank order
        assert offs[0] == 0 and all(offs[i] + ns[i] == offs[i + 1] for i in range(len(outs) - 1))
        assert sum(ns) == g
        for name, idx, arr in (("verts", 3, v), ("filt", 4, f), ("rows", 5, r)):
            cat = np.concatenate([out[k][idx].reshape(-1) for out in outs])
            assert np.array_equal(cat, np.asarray(arr).reshape(-1)), (k, name)
    for out in outs:
        assert out["vor"].tobytes() == vor.tobytes()
    return o


CASES = {
    "c1": lambda: (workloads.WORKLOADS["C1"].points(), 1, math.inf),
    "ties_tets": lambda: (workloads.integer_lattice(4, 3), 2, 1.8),
    "c2_tets": lambda: (workloads.WORKLOADS["C2"].points(), 2, 0.45),
    "gauss_multi_tile": lambda: (workloads.random_cloud(31, 3000, 10, "gauss"), 1, 2.8),
    "five_points": lambda: (np.array(json.load(open(os.path.join(GOLDEN, "ties_five_points.json")))["points"],
                                     dtype=np.float64), 1, 5.0),
}


@pytest.mark.parametrize("case,world", [("c1", 2), ("c1", 8), ("ties_tets", 3), ("ties_tets", 4),
                                        ("c2_tets", 2), ("c2_tets", 8), ("gauss_multi_tile", 4),
                                        ("five_points", 8), ("c1", 1)])
def test_build_dist_slices_equal_oracle(case, world):
    X, maxdim, radius = CASES[case]()
    outs = run_dist(X, maxdim, radius, world)
    check_vs_oracle(outs, X, maxdim, radius)
    if case == "five_points":   # 5 points: one row block, most ranks own no edges
        assert sum(1 for out in outs if out[2][2] == 0) >= world - 2
    import paper_1809_04424_b200 as vrb
    hp, hd, hn = vrb.build(X, maxdim=maxdim, radius=radius).h0()
    for out in outs:
        assert np.array_equal(out["h0"][0], _u32(hp)) and np.array_equal(out["h0"][1], _u32(hd))
        assert out["h0"][2] == hn


def test_build_dist_on_side_stream():
    # the collectives are issued on the library's build stream (a stream that
    # is not torch's current one): the exchange must still be ordered
    X, maxdim, radius = CASES["c2_tets"]()
    outs = run_dist(X, maxdim, radius, 3, side_stream=True)
    check_vs_oracle(outs, X, maxdim, radius)


def _nccl_worker(port, X, maxdim, radius, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_1809_04424_b200 as vrb

        res = vrb.build_dist(torch.from_numpy(X).cuda(), maxdim=maxdim, radius=radius)
        out = {"rank": 0}
        for k in range(1, maxdim + 2):
            g, off, n = res.count(k)
            v, f = res.simplices(k)
            out[k] = (g, off, n, _u32(v), _u32(f), _u32(res.boundary(k)))
        out["vor"] = res.rank_values().cpu().numpy()
        q.put(out)
    except Exception as e:
        q.put({"rank": 0, "error": repr(e)})
    finally:
        dist.destroy_process_group()


def test_build_dist_over_nccl_one_rank():
    # the NCCL code path of the collective callbacks (device tensors, the
    # library's stream as torch's current stream, no host synchronisation):
    # one rank per GPU, so one rank here
    X, maxdim, radius = CASES["c2_tets"]()
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), X, maxdim, radius, q))
    p.start()
    out = q.get(timeout=600)
    p.join(timeout=120)
    assert "error" not in out, out
    check_vs_oracle([out], X, maxdim, radius)
