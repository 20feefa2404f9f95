"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Small and medium inputs: every output array is compared element by element
(bit-exact: all outputs are integers or bit-exact float64).  Full-size
configs (C3, C5B, in the launch configuration bench.py times): edge arrays
exactly; triangles by (a) the per-level count histogram against the oracle's
(golden digest written by tools/make_golden.py from oracle/ only), (b) strict
(filt, lex) order of the whole array, (c) every triangle's boundary rows
pointing at its three edges with filt = max edge filt, (d) sampled levels
compared element by element with the oracle's enumeration of that level.
(a)+(b)+(c) imply the sets are equal; (d) spot-checks the exact layout.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def vrb():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_04424_b200 as m
    return m


def _np(t):
    return t.cpu().numpy().view(np.uint32) if t.dtype == torch.int32 else t.cpu().numpy()


def compare(vrb, X, maxdim, radius, strict=False, via_torch_alloc=False, res=None):
    """Element-by-element parity of a build of X (or of `res`, a build of the
    same points passed in another layout) against the oracle on X."""
    if res is None:
        res = vrb.build(X, maxdim=maxdim, radius=radius, strict=strict)
    o = oracle.Oracle(X, radius, strict)
    ev, ef, el, vor = o.edges()
    assert res.count(0)[0] == X.shape[0]
    assert res.count(1)[0] == o.E
    gv, gf = res.simplices(1)
    np.testing.assert_array_equal(_np(gv), ev)
    np.testing.assert_array_equal(_np(gf), ef)
    gvor = _np(res.rank_values())
    assert gvor.shape[0] == o.nvals
    assert gvor.tobytes() == vor.tobytes()          # bit-exact lengths
    np.testing.assert_array_equal(_np(res.boundary(1)), ev)
    if maxdim >= 1:
        tv, tf, tr = o.simplices(2)
        assert res.count(2)[0] == tv.shape[0]
        gtv, gtf = res.simplices(2)
        np.testing.assert_array_equal(_np(gtv), tv)
        np.testing.assert_array_equal(_np(gtf), tf)
        np.testing.assert_array_equal(_np(res.boundary(2)), tr)
        cp = res.boundary_colptr(2).cpu().numpy()
        np.testing.assert_array_equal(cp, 3 * np.arange(tv.shape[0] + 1))
    if maxdim >= 2:
        qv, qf, qr = o.simplices(3)
        assert res.count(3)[0] == qv.shape[0]
        gqv, gqf = res.simplices(3)
        np.testing.assert_array_equal(_np(gqv), qv)
        np.testing.assert_array_equal(_np(gqf), qf)
        np.testing.assert_array_equal(_np(res.boundary(3)), qr)
        cp = res.boundary_colptr(3).cpu().numpy()
        np.testing.assert_array_equal(cp, 4 * np.arange(qv.shape[0] + 1))
    return res, o


def test_golden_unit_square_and_ties(vrb):
    for name in ("unit_square.json", "ties_five_points.json"):
        g = json.load(open(os.path.join(GOLDEN, name)))
        X = np.array(g["points"], dtype=np.float64)
        compare(vrb, X, 1, math.inf)
    X = np.array(json.load(open(os.path.join(GOLDEN, "ties_five_points.json")))["points"], dtype=np.float64)
    compare(vrb, X, 1, 5.0)
    compare(vrb, X, 1, 5.0, strict=True)


def test_c1(vrb):
    w = workloads.WORKLOADS["C1"]
    compare(vrb, w.points(), w.maxdim, w.radius)


def test_c2_triangles(vrb):
    w = workloads.WORKLOADS["C2"]
    compare(vrb, w.points(), 1, w.radius)


def test_c2_tetrahedra(vrb):
    w = workloads.WORKLOADS["C2"]
    compare(vrb, w.points(), w.maxdim, w.radius)


@pytest.mark.parametrize("seed", range(60))
def test_random_small_tetrahedra(vrb, seed):
    rng = np.random.default_rng(5000 + seed)
    kind = ["uniform", "gauss", "lattice", "halfint", "dups"][seed % 5]
    n = int(rng.integers(0, 45))
    d = int(rng.integers(1, 5))
    X = workloads.random_cloud(5000 + seed, n, d, kind)
    radius = [math.inf, 0.5, 1.0, 1.5, 2.0][seed % 5]
    compare(vrb, X, 2, radius, strict=bool(seed % 6 == 1))


def test_lattice_tetrahedra_ties(vrb):
    # 4x4x4 lattice: heavy length ties in dimension 3 too
    X = workloads.integer_lattice(4, 3)
    compare(vrb, X, 2, math.inf)
    compare(vrb, X, 2, 1.8)


@pytest.mark.parametrize("seed", range(4))
def test_wide_list_layout_tetrahedra(vrb, seed, monkeypatch):
    monkeypatch.setenv("VRB_FORCE_WIDE_LISTS", "1")
    X = workloads.random_cloud(900 + seed, 60, 3, ["uniform", "lattice"][seed % 2])
    compare(vrb, X, 2, [0.6, 1.5][seed % 2])


def test_long_apex_runs_tetrahedra(vrb):
    # full filtration of 120 points: owner edges with > 104 triangles, so the
    # face search goes through its 8-ary rounds after the 12-separator record
    compare(vrb, workloads.random_cloud(77, 120, 3, "uniform"), 2, math.inf)


@pytest.mark.parametrize("n,seed", [(20000, 79), (33000, 78)])
def test_sparse_tetrahedra_large_n(vrb, n, seed):
    # n > 16384: the list-based tetrahedron kernel (no dense table); n > 0x7FFF:
    # vertex ids above 15 bits take the scalar separator / apex comparisons
    compare(vrb, workloads.random_cloud(seed, n, 3, "uniform"), 2, 0.045 * (33000 / n) ** (1 / 3))


@pytest.mark.parametrize("n", [0, 1, 2, 3])
def test_tiny(vrb, n):
    compare(vrb, workloads.random_cloud(n, n, 2), 1, math.inf)


def test_zero_radius_duplicates(vrb):
    X = np.array([[0.5, 0.5], [0.5, 0.5], [2.0, 0.0], [0.5, 0.5]])
    compare(vrb, X, 1, 0.0)
    compare(vrb, X, 1, 0.0, strict=True)


@pytest.mark.parametrize("seed", range(200))
def test_random_small(vrb, seed):
    rng = np.random.default_rng(seed)
    kind = ["uniform", "gauss", "lattice", "halfint", "dups"][seed % 5]
    n = int(rng.integers(0, 90))
    d = int(rng.integers(1, 6))
    X = workloads.random_cloud(seed, n, d, kind)
    if n >= 2:
        qs = [math.inf, 0.1, 0.3, 0.6]
        q = qs[seed % 4]
        # caps at data quantiles, sometimes exactly at an attained length
        lens = [oracle.length(X, i, j) for i in range(min(n, 12)) for j in range(i + 1, min(n, 12))]
        radius = math.inf if q == math.inf else float(np.quantile(lens, q, method="nearest")) if lens else 1.0
    else:
        radius = math.inf
    compare(vrb, X, 1, radius, strict=bool(seed % 7 == 3))


def test_multi_tile_ragged(vrb):
    X = workloads.random_cloud(77, 333, 4, "uniform")      # 6 tiles of 64, ragged tail
    compare(vrb, X, 1, 0.45)


def test_lattice_heavy_ties_large_segments(vrb):
    # 5x5x5 lattice: 7750 edges on 25 levels; tie groups hold up to ~10^5
    # triangles (exercises the global-sort path of the tie sort)
    X = workloads.integer_lattice(5, 3)
    compare(vrb, X, 1, math.inf)
    compare(vrb, X, 1, 2.0)


def test_device_points(vrb):
    X = workloads.random_cloud(5, 120, 3, "gauss")
    res, o = compare(vrb, X, 1, 1.3)
    Xd = torch.from_numpy(X).cuda()
    compare(vrb, X, 1, 1.3, res=vrb.build(Xd, maxdim=1, radius=1.3))


# rowsare="dimensions": a d x n array whose COLUMNS are the
# points, passed as is with VRB_DIM_MAJOR; the library transposes on the
# device.  Host and device inputs, several tiles plus a ragged tail, d = 1,
# ties (lattice), tetrahedra, strict caps.
@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("case", range(5))
def test_rowsare_dimensions(vrb, on_device, case):
    n, d, kind, maxdim, radius, strict = [
        (300, 3, "gauss", 2, 0.9, False),
        (257, 7, "uniform", 1, math.inf, False),
        (130, 1, "uniform", 1, 0.05, True),
        (0, 3, "uniform", 1, 1.0, False),
        (None, 3, "lattice", 2, 1.5, False)][case]
    X = workloads.integer_lattice(4, 3) if n is None else workloads.random_cloud(77 + case, n, d, kind)
    Xt = np.ascontiguousarray(X.T)                       # d x n
    arg = torch.from_numpy(Xt).cuda() if on_device else Xt
    res = vrb.build(arg, maxdim=maxdim, radius=radius, strict=strict, rowsare="dimensions")
    assert res.count(0)[0] == X.shape[0]
    compare(vrb, X, maxdim, radius, strict=strict, res=res)


def test_rowsare_dimensions_worldmap_pipeline(vrb):
    # the paper's WorldMap call sequence: latlon (n x 2 degrees)
    # -> latlon2euc -> a 3 x n matrix -> eirene(c, rowsare="dimensions",
    # upperlim=0.15); 2000 synthetic cities uniform on the sphere
    rng = np.random.default_rng(1809)
    n = 2000
    ll = np.stack([np.degrees(np.arcsin(rng.uniform(-1, 1, n))), rng.uniform(-180, 180, n)], 1)
    xyz = vrb.latlon2euc(torch.from_numpy(ll).cuda())     # n x 3, device
    c = xyz.T.contiguous()                                # 3 x n, as the paper's latlon2euc returns
    res = vrb.build(c, maxdim=1, radius=0.15, rowsare="dimensions")
    compare(vrb, xyz.cpu().numpy(), 1, 0.15, res=res)
    with pytest.raises(ValueError):
        vrb.build(c, rowsare="columns")


def test_high_degree_over_apex_bitmap_limit(vrb):
    # hub degree 9000 > 8192: the build falls back to the re-enumerating fill
    test_high_degree_byte_map_rounds(vrb, m=9000)


def test_high_degree_byte_map_rounds(vrb, m=4500):
    # two hubs adjacent to m jittered points of a high-dimensional sphere
    # (mutually almost never adjacent); the hub-hub edge is the longest, so its
    # older-neighbour prefixes hold m entries (> 4096 ranks per round: the
    # fill runs several rounds, and a long prefix is streamed in chunks)
    rng = np.random.default_rng(3)
    dim = 200
    S = rng.standard_normal((m, dim))
    S /= np.linalg.norm(S, axis=1, keepdims=True)
    S *= (1.0 + 0.01 * rng.uniform(size=(m, 1)))
    P = np.zeros((m + 2, dim + 1))
    P[:m, :dim] = S
    P[m, dim] = 0.6
    P[m + 1, dim] = -0.6
    compare(vrb, P, 1, 1.2)


@pytest.mark.parametrize("seed", range(12))
def test_wide_list_layout(vrb, seed, monkeypatch):
    # the unpacked neighbour-list layout used when n or a degree exceeds 65536,
    # forced on small inputs
    monkeypatch.setenv("VRB_FORCE_WIDE_LISTS", "1")
    kind = ["uniform", "lattice", "halfint", "dups"][seed % 4]
    X = workloads.random_cloud(300 + seed, 40 + 20 * seed, 3, kind)
    compare(vrb, X, 1, [0.5, 1.6, 1.2, 0.4][seed % 4])


@pytest.mark.parametrize("wide", ["0", "1"])
def test_sorted_rank_path(vrb, monkeypatch, wide):
    # neighbour ranks by the (vertex, neighbour) radix sort, used when n is too
    # large for the per-vertex bitmap, forced on small inputs
    monkeypatch.setenv("VRB_FORCE_SORT_RANKS", "1")
    monkeypatch.setenv("VRB_FORCE_WIDE_LISTS", wide)
    for seed in range(4):
        X = workloads.random_cloud(700 + seed, 150, 3, ["uniform", "lattice"][seed % 2])
        compare(vrb, X, 1, [0.4, 1.5][seed % 2])


def test_wide_list_layout_multi_round(vrb, monkeypatch):
    monkeypatch.setenv("VRB_FORCE_WIDE_LISTS", "1")
    test_high_degree_byte_map_rounds(vrb)


@pytest.mark.parametrize("seed", range(6))
def test_fill_without_apex_bitmaps(vrb, monkeypatch, seed):
    # the re-enumerating fill (multi-rank builds, degrees > 8192) on the
    # single-rank configs: same bytes as with the count pass's apex bitmaps
    monkeypatch.setenv("VRB_NO_APEX_BITMAPS", "1")
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(50, 700))
    X = workloads.random_cloud(seed, n, 3, ["uniform", "lattice", "gauss"][seed % 3])
    compare(vrb, X, 2 if seed % 2 else 1, [0.35, 1.5, 1.2][seed % 3])


def test_fill_without_apex_bitmaps_high_degree(vrb, monkeypatch):
    monkeypatch.setenv("VRB_NO_APEX_BITMAPS", "1")
    test_high_degree_byte_map_rounds(vrb)
    w = workloads.WORKLOADS["C2"]
    compare(vrb, w.points(), w.maxdim, w.radius)


def test_edge_sort_high_bit_runs_fallback(vrb):
    # lengths 1 + k * 1e-12: they agree in the high bits the partial radix
    # pass sorts on and differ below; runs longer than 64 take the full-sort
    # fallback, shorter runs the in-place fix-up -- both must give (len, i, j)
    for m in (40, 150):
        X = np.zeros((m + 1, 2))
        theta = np.linspace(0.0, 2.0 * np.pi, m, endpoint=False)
        rad = 1.0 + np.arange(m)[::-1] * 1e-12              # reversed: the fix-up has to move every key
        X[1:, 0] = rad * np.cos(theta)
        X[1:, 1] = rad * np.sin(theta)
        o = oracle.Oracle(X, math.inf)
        el = o.edges()[2]
        near = el[(el > 0.999) & (el < 1.001)]
        assert len(near) >= m and len(np.unique(near)) >= m   # a run of distinct keys (m = 150: > 64, fallback)
        compare(vrb, X, 0, math.inf)
        compare(vrb, X, 1, 1.0 + 1e-9)


@pytest.mark.parametrize("m", [20, 50])
def test_edge_sort_high_bit_runs_with_ties(vrb, m):
    # as above, every ring point twice: each run of equal high bits mixes
    # equal lengths (a dense-rank level of 2+ edges) with distinct ones, so
    # the fused ranking pass must count distinct keys per run and keep equal
    # keys in (i, j) order
    theta = np.linspace(0.0, 2.0 * np.pi, m, endpoint=False)
    rad = 1.0 + np.arange(m)[::-1] * 1e-12
    ring = np.stack([rad * np.cos(theta), rad * np.sin(theta)], axis=1)
    X = np.concatenate([np.zeros((1, 2)), ring, ring[::-1], [[1000.0, 0.0]]])
    compare(vrb, X, 0, math.inf)
    compare(vrb, X, 1, 1.0 + 1e-9)


@pytest.mark.parametrize("seed", range(4))
def test_global_host_map_forced(vrb, monkeypatch, seed):
    # the host map in global memory (used when n is too large for shared
    # memory), forced on small inputs: bitmap, re-enumerating and wide paths
    monkeypatch.setenv("VRB_FORCE_GLOBAL_MAP", "1")
    X = workloads.random_cloud(950 + seed, 300, 3, ["uniform", "lattice"][seed % 2])
    compare(vrb, X, 1, [0.35, 1.5][seed % 2])
    monkeypatch.setenv("VRB_NO_APEX_BITMAPS", "1")
    compare(vrb, X, 1, [0.35, 1.5][seed % 2])
    monkeypatch.setenv("VRB_FORCE_WIDE_LISTS", "1")
    compare(vrb, X, 1, [0.35, 1.5][seed % 2])


def test_large_n_global_map_wide_lists(vrb):
    # n = 70000 > 65536 (wide lists) and far beyond the shared-memory host map:
    # properties against an independent neighbour search (scipy cKDTree) and a
    # sparse-matrix triangle count (trace(A^3) / 6)
    spatial = pytest.importorskip("scipy.spatial")
    sp = pytest.importorskip("scipy.sparse")
    rng = np.random.default_rng(70000)
    n = 70000
    X = rng.uniform(0, 1, (n, 3))
    r = 0.03                                     # mean degree ~8: ~2.8e5 edges, ~6e5 triangles
    pairs = spatial.cKDTree(X).query_pairs(r, output_type="ndarray")
    d = np.sqrt(((X[pairs[:, 0]] - X[pairs[:, 1]]) ** 2).sum(1))
    assert np.abs(d - r).min() > 1e-9            # no pair at the cap: the reference set is exact
    vrb.use_torch_allocator(True)
    try:
        res = vrb.build(torch.from_numpy(X).cuda(), maxdim=1, radius=r)
        ev, ef = res.simplices(1)
        ev, ef = _np(ev).astype(np.int64), _np(ef)
        assert ev.shape[0] == pairs.shape[0]
        got = np.sort(ev[:, 0] * n + ev[:, 1])
        want = np.sort(np.minimum(pairs[:, 0], pairs[:, 1]).astype(np.int64) * n + np.maximum(pairs[:, 0], pairs[:, 1]))
        np.testing.assert_array_equal(got, want)
        A = sp.coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(n, n))
        A = (A + A.T).tocsr()
        T = int(round((A @ A).multiply(A).sum() / 6))
        tv, tf = res.simplices(2)
        tv, tf = _np(tv).astype(np.int64), _np(tf)
        assert tv.shape[0] == T and T > 100000
        rows = _np(res.boundary(2)).astype(np.int64)
        assert np.all(np.diff(rows, axis=1) > 0)
        # the rows are the positions of the triangle's three edges
        ekey = ev[:, 0] * n + ev[:, 1]
        from_rows = np.sort(ekey[rows], axis=1)
        from_tri = np.sort(np.stack([tv[:, 0] * n + tv[:, 1], tv[:, 0] * n + tv[:, 2], tv[:, 1] * n + tv[:, 2]], 1),
                           axis=1)
        np.testing.assert_array_equal(from_rows, from_tri)
        # filt = the largest edge filt = the filt of the last (largest-position) row
        np.testing.assert_array_equal(tf, ef[rows[:, 2]])
        assert np.all(ef[rows].max(axis=1) == tf)
        # strict (filt, lex) order: the (filt, v0, v1, v2) sort is the identity, no repeats
        order = np.lexsort((tv[:, 2], tv[:, 1], tv[:, 0], tf))
        np.testing.assert_array_equal(order, np.arange(T))
        dup = (np.diff(tf) == 0) & np.all(np.diff(tv, axis=0) == 0, axis=1)
        assert not dup.any()
        del res
    finally:
        torch.cuda.synchronize()
        vrb.use_torch_allocator(False)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("maxdim", [1, 2])
def test_skip_boundary_same_simplices(vrb, maxdim):
    # VRB_SKIP_BOUNDARY: no D_k row arrays, identical simplices and levels
    X = workloads.random_cloud(77, 400, 3, "uniform")
    o = oracle.Oracle(X, 0.3)
    res = vrb.build(X, maxdim=maxdim, radius=0.3, skip_boundary=True)
    for k in range(2, maxdim + 2):
        v, f, _ = o.simplices(k)
        gv, gf = res.simplices(k)
        np.testing.assert_array_equal(_np(gv), v)
        np.testing.assert_array_equal(_np(gf), f)


def test_sortperm_literal_and_random(vrb):
    g = json.load(open(os.path.join(GOLDEN, "sortperm_literal.json")))
    for case in g["cases"]:
        perm, dense = vrb.sortperm_f64(torch.tensor(case["v"], dtype=torch.float64, device="cuda"))
        assert (perm.cpu().numpy() + 1).tolist() == case["sortperm_1based"]
        assert dense.cpu().numpy().tolist() == case["dense_rank"]
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.standard_normal(100000), rng.integers(-5, 5, 50000).astype(np.float64),
                        [0.0, -0.0, np.inf, -np.inf]])
    rng.shuffle(v)
    perm, dense = vrb.sortperm_f64(torch.from_numpy(v).cuda())
    op, od = oracle.sortperm(v)
    np.testing.assert_array_equal(perm.cpu().numpy(), op)
    np.testing.assert_array_equal(dense.cpu().numpy().view(np.uint32), od)


def test_sortperm_nan_rejected(vrb):
    with pytest.raises(vrb.VrbError):
        vrb.sortperm_f64(torch.tensor([1.0, float("nan")], dtype=torch.float64, device="cuda"))


def test_handle_outlives_allocator_switch(vrb):
    # a handle built through torch's caching allocator and freed after the hook
    # is switched back releases its memory through the hook that allocated it
    # (freeing torch memory with cudaFreeAsync would fail and leave an error
    # pending for the next call)
    X = workloads.random_cloud(9, 150, 3, "uniform")
    vrb.use_torch_allocator(True)
    try:
        res = vrb.build(X, maxdim=1, radius=0.4)
    finally:
        vrb.use_torch_allocator(False)
    res.free()
    compare(vrb, X, 1, 0.4)


def test_torch_allocator_hook(vrb):
    vrb.use_torch_allocator(True)
    try:
        compare(vrb, workloads.random_cloud(8, 200, 3, "uniform"), 1, 0.3)
    finally:
        vrb.use_torch_allocator(False)


# ---------------------------------------------------------------------------
# full-size configs
# ---------------------------------------------------------------------------

def _check_triangles_full(vrb, res, o, golden, n_levels_sampled=40):
    dev = res.device
    E = o.E
    ev, ef, el, vor = o.edges()
    gv, gf = res.simplices(1)
    np.testing.assert_array_equal(_np(gv), ev)
    np.testing.assert_array_equal(_np(gf), ef)
    assert _np(res.rank_values()).tobytes() == vor.tobytes()
    tv, tf = res.simplices(2)
    rows = res.boundary(2)
    T = tv.shape[0]
    assert T == golden["count"]
    # (a) per-level histogram == oracle's
    hist = torch.bincount(tf.to(torch.int64), minlength=o.nvals + 1).cpu().numpy().astype(np.uint64)
    assert hashlib.sha256(hist.tobytes()).hexdigest() == golden["hist_sha256"]
    # (b) strict (filt, lex) order, (c) rows are the three edges, filt = max edge filt
    evd = torch.from_numpy(ev.astype(np.int64)).to(dev)
    efd = torch.from_numpy(ef.astype(np.int64)).to(dev)
    chunk = 1 << 27
    prev = None
    for s in range(0, T, chunk):
        e = min(T, s + chunk + 1)
        v = tv[s:e].to(torch.int64)
        f = tf[s:e].to(torch.int64)
        r = rows[s:e].to(torch.int64) & 0xFFFFFFFF
        assert bool((v[:, 0] < v[:, 1]).all()) and bool((v[:, 1] < v[:, 2]).all())
        code = (v[:, 0] << 42) | (v[:, 1] << 21) | v[:, 2]
        key_f = f[1:] - f[:-1]
        key_c = code[1:] - code[:-1]
        assert bool(((key_f > 0) | ((key_f == 0) & (key_c > 0))).all())
        assert bool((r[:, 0] < r[:, 1]).all()) and bool((r[:, 1] < r[:, 2]).all())
        ea, eb, ec = evd[r[:, 0]], evd[r[:, 1]], evd[r[:, 2]]
        verts = torch.sort(torch.cat([ea, eb, ec], 1), 1).values
        want = torch.stack([v[:, 0], v[:, 0], v[:, 1], v[:, 1], v[:, 2], v[:, 2]], 1)
        assert bool((verts == want).all())
        assert bool((efd[r[:, 2]] == f).all())
        assert bool((torch.maximum(torch.maximum(efd[r[:, 0]], efd[r[:, 1]]), efd[r[:, 2]]) == f).all())
        del v, f, r, ea, eb, ec, verts, want, code
    # (d) sampled levels, element by element
    start = np.concatenate([[0], np.cumsum(hist)]).astype(np.int64)
    rng = np.random.default_rng(0)
    levels = sorted(set(rng.integers(1, o.nvals + 1, n_levels_sampled).tolist()) | {1, o.nvals})
    for lvl in levels:
        sv, sr = o.simplices_at_filt(2, int(lvl))
        a, b = start[lvl], start[lvl + 1]
        assert b - a == len(sv)
        np.testing.assert_array_equal(_np(tv[a:b]), sv)
        np.testing.assert_array_equal(_np(rows[a:b]), sr)


@pytest.mark.parametrize("config", ["C3", "C5B"])
def test_full_size_config(vrb, config):
    path = os.path.join(GOLDEN, f"{config.lower()}_levels.json")
    golden = json.load(open(path))
    w = workloads.WORKLOADS[config]
    X = w.points()
    assert hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest() == golden["points_sha256"]
    vrb.use_torch_allocator(True)
    try:
        res = vrb.build(torch.from_numpy(X).cuda(), maxdim=w.maxdim, radius=w.radius)
        o = oracle.Oracle(X, w.radius)
        assert o.E == golden["E"]
        _check_triangles_full(vrb, res, o, golden)
        del res
    finally:
        torch.cuda.synchronize()
        vrb.use_torch_allocator(False)
        torch.cuda.empty_cache()


def test_hiv_tie_heavy_full(vrb):
    # the paper's tie-heavy benchmark at full size (HIV: 1088 sequences,
    # Hamming distances): 159 distinct lengths for 591,328 edges,
    # so EVERY level is a tie group and all 214,060,736 triangles go through
    # the batched tie-group sort (segsort.cu).  Per-level histogram against the
    # oracle's golden digest, strict (filt, lex) order, rows = edges, and
    # sampled tie levels element by element.
    golden = json.load(open(os.path.join(GOLDEN, "hiv_levels.json")))
    w = workloads.WORKLOADS["HIV"]
    D = w.points()
    assert hashlib.sha256(np.ascontiguousarray(D).tobytes()).hexdigest() == golden["points_sha256"]
    vrb.use_torch_allocator(True)
    try:
        res = vrb.build_dm(torch.from_numpy(D).cuda(), maxdim=1, radius=w.radius)
        o = oracle.Oracle(None, w.radius, D=D)
        assert o.E == golden["E"] and o.nvals == golden["nvals"]
        _check_triangles_full(vrb, res, o, golden, n_levels_sampled=10)
        del res
    finally:
        torch.cuda.synchronize()
        vrb.use_torch_allocator(False)
        torch.cuda.empty_cache()


def test_c5a_edges_full(vrb):
    # C5A: 199,990,000 edges, all pairs (r = inf).  Full edge parity on a
    # sample of positions plus global properties (the oracle's full sort of
    # 2e8 edges is minutes of CPU: checked by sampling rows of the oracle).
    w = workloads.WORKLOADS["C5A"]
    X = w.points()
    res = vrb.build(torch.from_numpy(X).cuda(), maxdim=0, radius=math.inf)
    assert vrb.last_edge_path() == "bucket"   # the path bench.py times for C5A
    n = X.shape[0]
    E = n * (n - 1) // 2
    assert res.count(1)[0] == E
    gv, gf = res.simplices(1)
    vor = res.rank_values()
    v = gv.to(torch.int64)
    f = gf.to(torch.int64)
    assert bool((v[:, 0] < v[:, 1]).all())
    # every pair exactly once
    code = v[:, 0] * n + v[:, 1]
    assert int(torch.unique(code).numel()) == E
    # lengths non-decreasing along the order, (len, i, j) ties in lex order
    lens = vor[f - 1]
    dl = lens[1:] - lens[:-1]
    assert bool((dl >= 0).all())
    tie = dl == 0
    assert bool((code[1:][tie] > code[:-1][tie]).all())
    assert bool(((f[1:] - f[:-1]) == (dl > 0).to(torch.int64)).all())
    # sampled pairs: bit-exact length against the oracle's fold
    rng = np.random.default_rng(1)
    idx = rng.integers(0, E, 2000)
    vv = v[torch.from_numpy(idx).cuda()].cpu().numpy()
    ll = lens[torch.from_numpy(idx).cuda()].cpu().numpy()
    for (i, j), L in zip(vv, ll):
        assert oracle.length(X, int(i), int(j)) == L
    # every element: the oracle's full (len, i, j) order, levels and
    # value_of_rank, as SHA-256 digests (tests/golden/c5a_edges.json, written
    # by tools/make_golden.py from oracle/ only)
    g = json.load(open(os.path.join(GOLDEN, "c5a_edges.json")))
    assert g["points_sha256"] == hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest()
    assert g["E"] == E and g["nvals"] == vor.shape[0]
    del v, f, code, lens, dl, tie
    h = hashlib.sha256()
    gvc = gv.cpu()
    step = 1 << 24
    for a in range(0, E, step):
        h.update(gvc[a:a + step].numpy().view(np.uint32).ravel().astype(np.uint64).tobytes())
    del gvc
    gfc = gf.cpu()
    for a in range(0, E, step):
        h.update(gfc[a:a + step].numpy().view(np.uint32).astype(np.uint64).tobytes())
    assert h.hexdigest() == g["edges_sha256"]
    assert hashlib.sha256(vor.cpu().numpy().tobytes()).hexdigest() == g["value_of_rank_sha256"]


def test_full_size_c4_tetrahedra(vrb):
    # C4: 5000-point noisy sphere, cap 0.40, maxdim 2: edges and triangles
    # element by element; 4.3e8 tetrahedra by (a) the per-level histogram
    # (golden digest from oracle/), (b) strict (filt, lex) order, (c) every D_3
    # row is a face triangle of the column with filt <= and the last row's filt
    # equal to the column's, (d) sampled levels element by element.
    path = os.path.join(GOLDEN, "c4_levels.json")
    golden = json.load(open(path))
    w = workloads.WORKLOADS["C4"]
    X = w.points()
    assert hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest() == golden["points_sha256"]
    vrb.use_torch_allocator(True)
    try:
        res = vrb.build(torch.from_numpy(X).cuda(), maxdim=2, radius=w.radius)
        o = oracle.Oracle(X, w.radius)
        ev, ef, el, vor = o.edges()
        np.testing.assert_array_equal(_np(res.simplices(1)[0]), ev)
        np.testing.assert_array_equal(_np(res.simplices(1)[1]), ef)
        tv, tf, tr = o.simplices(2)
        np.testing.assert_array_equal(_np(res.simplices(2)[0]), tv)
        np.testing.assert_array_equal(_np(res.simplices(2)[1]), tf)
        np.testing.assert_array_equal(_np(res.boundary(2)), tr)
        qv, qf = res.simplices(3)
        qr = res.boundary(3)
        Q = qv.shape[0]
        assert Q == golden["count"]
        hist = torch.bincount(qf.to(torch.int64), minlength=o.E + 1).cpu().numpy().astype(np.uint64)
        assert hashlib.sha256(hist.tobytes()).hexdigest() == golden["hist_sha256"]
        dev = res.device
        tvd = torch.from_numpy(tv.astype(np.int64)).to(dev)
        tfd = torch.from_numpy(tf.astype(np.int64)).to(dev)
        chunk = 1 << 26
        for s in range(0, Q, chunk):
            e = min(Q, s + chunk + 1)
            v = qv[s:e].to(torch.int64)
            f = qf[s:e].to(torch.int64)
            r = qr[s:e].to(torch.int64) & 0xFFFFFFFF
            assert bool((v[:, :-1] < v[:, 1:]).all())
            code = (v[:, 0] << 48) | (v[:, 1] << 32) | (v[:, 2] << 16) | v[:, 3]
            df, dc = f[1:] - f[:-1], code[1:] - code[:-1]
            assert bool(((df > 0) | ((df == 0) & (dc > 0))).all())
            assert bool((r[:, :-1] < r[:, 1:]).all())
            # each row is the face of the column missing one vertex
            for c in range(4):
                face = tvd[r[:, c]]                                  # (m, 3)
                inside = (face.unsqueeze(2) == v.unsqueeze(1)).any(2).all(1)
                assert bool(inside.all())
            assert bool((tfd[r[:, 3]] == f).all())
            assert bool((torch.maximum(tfd[r].max(1).values, tfd[r[:, 3]]) == f).all())
            del v, f, r, code
        start = np.concatenate([[0], np.cumsum(hist)]).astype(np.int64)
        rng = np.random.default_rng(4)
        levels = sorted(set(rng.integers(1, o.nvals + 1, 25).tolist()))
        for lvl in levels:
            sv, _ = o.simplices_at_filt(3, int(lvl))
            a, b = start[lvl], start[lvl + 1]
            assert b - a == len(sv)
            np.testing.assert_array_equal(_np(qv[a:b]), sv)
        del res
    finally:
        torch.cuda.synchronize()
        vrb.use_torch_allocator(False)
        torch.cuda.empty_cache()


@pytest.mark.parametrize("path", ["xmajor", "markfill", "bitmap"])
@pytest.mark.parametrize("case", range(4))
def test_triangle_path_variants(vrb, case, path, monkeypatch):
    # every triangle path (VRB_TRI_PATH=xmajor / markfill / bitmap) must be
    # as exact as the default one
    monkeypatch.setenv("VRB_TRI_PATH", path)
    X, maxdim, radius = [(workloads.random_cloud(21, 300, 4, "gauss"), 1, 1.8),
                         (workloads.integer_lattice(4, 3), 2, 1.5),
                         (workloads.WORKLOADS["C2"].points(), 2, 0.45),
                         (workloads.random_cloud(22, 200, 3, "dups"), 1, 0.35)][case]
    compare(vrb, X, maxdim, radius)
