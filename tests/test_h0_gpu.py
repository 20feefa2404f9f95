"""GPU parity of vrb_h0 (dimension-0 persistence from the
ranked edges) against the oracle's textbook GF(2) reduction of D_1
(Algorithm 1; bars by Fig. 4's reading) and, at full size,
against scipy's minimum spanning tree of the edge-position weights (an
independent library routine: with unique weights the Kruskal forest is what
pHcol pairs with vertex rows).
"""
import math

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vrb():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_04424_b200 as m
    return m


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def check_h0(vrb, X, radius, strict=False, maxdim=0):
    res = vrb.build(X, maxdim=maxdim, radius=radius, strict=strict)
    pos, death, ness = res.h0()
    pos, death = _u32(pos), _u32(death)
    o = oracle.Oracle(X, radius, strict)
    bars = o.barcodes(0, keep_zero=True)
    fin = np.sort(bars[(bars[:, 0] == 0) & (bars[:, 2] >= 0)][:, 2])
    inf = int(((bars[:, 0] == 0) & (bars[:, 2] < 0)).sum())
    assert ness == inf
    assert np.all(np.diff(pos.astype(np.int64)) > 0)          # ascending positions
    np.testing.assert_array_equal(death.astype(np.int64), fin)  # sorted deaths = oracle bars
    _, ef, _, _ = o.edges()
    np.testing.assert_array_equal(ef[pos], death)
    assert len(pos) + ness == X.shape[0]
    return res


def test_h0_golden_small(vrb):
    # unit square: three [0,1) bars + [0,inf) (P15 golden 1)
    X = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)
    res = check_h0(vrb, X, math.inf)
    _, death, ness = res.h0()
    assert list(_u32(death)) == [1, 1, 1] and ness == 1
    # five points with ties, full / capped / strict (P15 golden 2)
    X = np.array([[0, 0], [3, 0], [0, 4], [3, 4], [6, 0]], dtype=np.float64)
    for r, st in ((math.inf, False), (5.0, False), (5.0, True), (3.0, True)):
        check_h0(vrb, X, r, st)


@pytest.mark.parametrize("seed", range(24))
def test_h0_random(vrb, seed):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(1, 300))
    kind = seed % 4
    if kind == 0:
        X = rng.uniform(0, 1, (n, 3))
    elif kind == 1:
        X = rng.integers(0, 4, (n, 2)).astype(np.float64)     # lattice: heavy ties, duplicates
    elif kind == 2:
        X = rng.standard_normal((n, 5))
    else:                                                      # clusters: several components
        X = rng.standard_normal((n, 2)) * 0.05 + rng.integers(0, 5, (n, 1)) * 3.0
    _, _, el, _ = oracle.Oracle(X, math.inf).edges()
    r = float(np.quantile(el, 0.3)) if len(el) else 1.0
    check_h0(vrb, X, r)
    check_h0(vrb, X, math.inf, maxdim=1)


def test_h0_c1_c2(vrb):
    for name in ("C1", "C2"):
        w = workloads.WORKLOADS[name]
        check_h0(vrb, w.points(), w.radius, maxdim=w.maxdim)


def test_h0_degenerate(vrb):
    for n in (0, 1, 2):
        X = np.zeros((n, 3))
        res = vrb.build(X, maxdim=0, radius=math.inf)
        pos, death, ness = res.h0()
        assert pos.numel() == (1 if n == 2 else 0) and ness == n - pos.numel()
    X = np.array([[0.0], [10.0]])
    res = vrb.build(X, maxdim=0, radius=1.0)   # no edges: two essential bars
    pos, death, ness = res.h0()
    assert ness == 2 and pos.numel() == 0


@pytest.mark.parametrize("config", ["C5B", "C3"])
def test_h0_full_size_vs_scipy_mst(vrb, config):
    sp = pytest.importorskip("scipy.sparse")
    csgraph = pytest.importorskip("scipy.sparse.csgraph")
    w = workloads.WORKLOADS[config]
    X = w.points()
    vrb.use_torch_allocator(True)
    try:
        res = vrb.build(torch.from_numpy(X).cuda(), maxdim=0, radius=w.radius)
        ev, ef = res.simplices(1)
        ev, ef = _u32(ev).astype(np.int64), _u32(ef)
        pos, death, ness = res.h0()
        pos, death = _u32(pos), _u32(death)
        E, n = ev.shape[0], X.shape[0]
        # weights = position + 1 (unique): the MST is the Kruskal forest of the order
        G = sp.coo_matrix((np.arange(1, E + 1, dtype=np.float64), (ev[:, 0], ev[:, 1])), shape=(n, n)).tocsr()
        T = csgraph.minimum_spanning_tree(G).tocoo()
        ref = np.sort(T.data.astype(np.int64) - 1)
        np.testing.assert_array_equal(pos.astype(np.int64), ref)
        np.testing.assert_array_equal(death, ef[pos])
        ncomp, _ = csgraph.connected_components(G, directed=False)
        assert ness == ncomp and len(pos) + ness == n
    finally:
        del res
        torch.cuda.synchronize()
        vrb.use_torch_allocator(False)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("radius", [math.inf, 30.0])
def test_h0_late_crossing_edges_vs_scipy(vrb, radius):
    # three far-apart blobs: the edges joining them come after ~3e6 intra-blob
    # edges, so the forest is finished in the last filter windows (radius inf:
    # a spanning tree ends the search; radius 30: two blobs never join)
    sp = pytest.importorskip("scipy.sparse")
    csgraph = pytest.importorskip("scipy.sparse.csgraph")
    rng = np.random.default_rng(11)
    X = np.concatenate([rng.normal(0.0, 1.0, (1400, 3)), rng.normal(0.0, 1.0, (1100, 3)) + [100.0, 0, 0],
                        rng.normal(0.0, 1.0, (500, 3)) + [0, 25.0, 0]])
    res = vrb.build(X, maxdim=0, radius=radius)
    ev, ef = res.simplices(1)
    ev, ef = _u32(ev).astype(np.int64), _u32(ef)
    pos, death, ness = res.h0()
    pos, death = _u32(pos), _u32(death)
    E, n = ev.shape[0], X.shape[0]
    G = sp.coo_matrix((np.arange(1, E + 1, dtype=np.float64), (ev[:, 0], ev[:, 1])), shape=(n, n)).tocsr()
    ref = np.sort(csgraph.minimum_spanning_tree(G).tocoo().data.astype(np.int64) - 1)
    np.testing.assert_array_equal(pos.astype(np.int64), ref)
    np.testing.assert_array_equal(death, ef[pos])
    ncomp, _ = csgraph.connected_components(G, directed=False)
    assert ness == ncomp == (1 if math.isinf(radius) else 2)
