"""GPU parity of vrb_h0 (dimension-0 persistence from the
ranked edges) against the oracle's textbook GF(2) reduction of D_1
(Algorithm 1; bars by Fig. 4's reading) and, at full size,
against scipy's minimum spanning tree of the edge-position weights (an
independent library routine: with unique weights the Kruskal forest is what
pHcol pairs with vertex rows).
"""
import math
import os

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


# ---------------------------------------------------------------------------
# "Clear and compress": D_2 without the rows of the
# H0 forest (the D_1 pivot columns).  Checked two ways against the oracle:
# (1) the compressed matrix equals the oracle's D_2 with the rows of the
#     edges whose D_1 column the oracle's textbook reduction leaves nonzero
#     removed and the rest renumbered; (2) the oracle's reduction of the
#     compressed matrix pairs exactly the (edge, triangle) pivots its
#     reduction of the full D_2 pairs -- the compression lemma (every
#     dimension-1 bar is unchanged).
# ---------------------------------------------------------------------------
def _compress_cases():
    import json
    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ties_five_points.json")))
    return {
        "c1": (workloads.WORKLOADS["C1"].points(), math.inf),
        "c2": (workloads.WORKLOADS["C2"].points(), 0.45),
        "lattice": (workloads.integer_lattice(4, 3), 1.5),
        "five": (np.array(g["points"], dtype=np.float64), 5.0),
        "gauss": (workloads.random_cloud(12, 120, 4, "gauss"), 1.6),
        "two_blobs": (np.concatenate([workloads.random_cloud(13, 40, 3, "uniform"),
                                      workloads.random_cloud(14, 40, 3, "uniform") + 10.0]), 0.5),
    }


@pytest.mark.parametrize("case", ["c1", "c2", "lattice", "five", "gauss", "two_blobs"])
def test_compress_d2_vs_oracle(vrb, case):
    X, radius = _compress_cases()[case]
    res = vrb.build(X, maxdim=1, radius=radius)
    cp, rv, rm = res.compress_d2()
    cp, rv, rm = cp.cpu().numpy(), _u32(rv), _u32(rm)
    o = oracle.Oracle(X, radius)
    ev, ef, _, _ = o.edges()
    E = o.E
    _, _, rows = o.simplices(2)
    # the oracle's D_1 reduction: edge columns that stay nonzero are the pivots
    _, zero1 = oracle.reduce(X.shape[0], [list(map(int, e)) for e in ev], "col")
    negative = ~zero1
    keep = np.flatnonzero(~negative)
    newidx = np.full(E, -1, dtype=np.int64)
    newidx[keep] = np.arange(keep.size)
    want_cols = [[int(newidx[r]) for r in col if newidx[r] >= 0] for col in rows]
    assert np.array_equal(rm, keep.astype(np.uint32))
    assert cp[0] == 0 and cp.shape[0] == rows.shape[0] + 1
    got_cols = [rv[cp[j]:cp[j + 1]].astype(np.int64).tolist() for j in range(rows.shape[0])]
    assert got_cols == want_cols
    assert all(1 <= len(c) <= 3 for c in got_cols)
    # compression lemma: identical pivot pairs
    piv_full, _ = oracle.reduce(E, [list(map(int, c)) for c in rows], "col")
    piv_c, _ = oracle.reduce(keep.size, got_cols, "col")
    full_pairs = {(int(r), int(c)) for r, c in enumerate(piv_full) if c >= 0}
    comp_pairs = {(int(rm[r]), int(c)) for r, c in enumerate(piv_c) if c >= 0}
    assert comp_pairs == full_pairs
    # the forest edges are never pivots of D_2
    assert not any(negative[r] for r, _ in full_pairs)


def test_compress_d2_large_forest_index_in_global_memory(vrb):
    # 80 000 points: a forest of ~70 000 edges and hundreds of column tiles
    # chained by the look-back of the one-pass compress; the result must
    # still be D_2 without the forest rows, renumbered (checked against that
    # definition on the GPU's own D_2 and forest, whose parity the tests
    # above establish)
    X = workloads.random_cloud(60, 80000, 3, "uniform")
    res = vrb.build(X, maxdim=1, radius=0.03)
    pos, _, _ = res.h0()
    forest = np.sort(_u32(pos).astype(np.int64))
    rows = _u32(res.boundary(2)).astype(np.int64)
    cp, rv, rm = res.compress_d2()
    cp, rv, rm = cp.cpu().numpy(), _u32(rv).astype(np.int64), _u32(rm).astype(np.int64)
    E = res.count(1)[0]
    keep = np.ones(E, dtype=bool)
    keep[forest] = False
    newidx = np.cumsum(keep) - 1
    assert np.array_equal(rm, np.flatnonzero(keep))
    kept = keep[rows]
    assert np.array_equal(np.diff(cp), kept.sum(1))
    assert np.array_equal(rv, newidx[rows][kept])
    assert kept.sum(1).min() >= 1
