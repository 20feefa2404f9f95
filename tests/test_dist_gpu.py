"""vrb_build_dist with several ranks on ONE GPU (gloo process group, so the
ranks may share a device): the concatenated per-rank slices must be
byte-identical to vrb_build (pin P13)."""
import math
import os
import socket

import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _u32(t):
    return t.cpu().numpy().view(np.uint32) if t.dtype == torch.int32 else t.cpu().numpy()


def _worker(rank, world, port, X, maxdim, radius, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_04424_b200 as vrb

        torch.cuda.set_device(0)
        res = vrb.build_dist(X, maxdim=maxdim, radius=radius)
        out = {"rank": rank}
        for k in range(1, maxdim + 2):
            g, off, n = res.count(k)
            v, f = res.simplices(k)
            out[k] = (g, off, n, _u32(v), _u32(f), _u32(res.boundary(k)))
        pos, death, ness = res.h0()   # every rank holds every edge: the whole H0 result
        out["h0"] = (_u32(pos), _u32(death), ness)
        q.put(out)
    except Exception as e:   # surface worker errors in the test
        q.put({"rank": rank, "error": repr(e)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["c1", "ties", "c2"])
@pytest.mark.parametrize("world", [2, 3])
def test_build_dist_slices_equal_single_gpu(case, world):
    import paper_1809_04424_b200 as vrb

    if case == "c1":
        w = workloads.WORKLOADS["C1"]
        X, maxdim, radius = w.points(), 1, w.radius
    elif case == "ties":
        X, maxdim, radius = workloads.integer_lattice(4, 3), 2, 1.8
    else:
        w = workloads.WORKLOADS["C2"]
        X, maxdim, radius = w.points(), 2, w.radius
    ref = vrb.build(X, maxdim=maxdim, radius=radius)
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, maxdim, radius, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=600) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=120)
    for o in outs:
        assert "error" not in o, o
    for k in range(1, maxdim + 2):
        g = ref.count(k)[0]
        rv, rf = ref.simplices(k)
        rr = ref.boundary(k)
        assert all(o[k][0] == g for o in outs)
        offs = [o[k][1] for o in outs]
        assert offs == sorted(offs) and offs[0] == 0
        assert sum(o[k][2] for o in outs) == g
        for name, idx, want in (("verts", 3, _u32(rv)), ("filt", 4, _u32(rf)), ("rows", 5, _u32(rr))):
            cat = np.concatenate([o[k][idx] for o in outs])
            assert np.array_equal(cat, want), (k, name)
    hp, hd, hn = ref.h0()
    for o in outs:
        assert np.array_equal(o["h0"][0], _u32(hp)) and np.array_equal(o["h0"][1], _u32(hd)) and o["h0"][2] == hn
