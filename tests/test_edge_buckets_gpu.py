"""GPU parity of S3's two edge-ranking paths (bucket scatter + on-chip
finish, edge_buckets.cu; LSD radix, radix_sort.cu + edges.cu) against the
oracle's (len, i, j) order, dense ranks and value_of_rank (P:929-936,
readings A3/A4), element by element.  Each case also asserts WHICH path ran
(vrb_last_edge_path), so a silent fallback cannot pass for the bucket path.
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
    return t.cpu().numpy().view(np.uint32) if t.dtype == torch.int32 else t.cpu().numpy()


def edges_equal(vrb, X, radius, strict=False, maxdim=0):
    res = vrb.build(X, maxdim=maxdim, radius=radius, strict=strict)
    path = vrb.last_edge_path()
    o = oracle.Oracle(X, radius, strict)
    ev, ef, _, vor = o.edges()
    assert res.count(1)[0] == o.E
    gv, gf = res.simplices(1)
    np.testing.assert_array_equal(_u32(gv), ev)
    np.testing.assert_array_equal(_u32(gf), ef)
    gvor = _u32(res.rank_values())
    assert gvor.shape[0] == o.nvals
    assert gvor.tobytes() == vor.tobytes()
    return path, res


@pytest.fixture(autouse=True)
def _bucket_path(monkeypatch):
    # the library takes the bucket path by default from 2^24 edges; these
    # cases force it (tests that want the radix path set it themselves)
    monkeypatch.setenv("VRB_EDGE_PATH", "bucket")


@pytest.mark.parametrize("seed", range(24))
def test_bucket_path_random(vrb, seed, monkeypatch):
    # continuous clouds: the bucket path must run and agree with the oracle
    rng = np.random.default_rng(7000 + seed)
    kind = ["uniform", "gauss"][seed % 2]
    n = int(rng.integers(3, 1500))
    d = int(rng.integers(1, 12))
    X = workloads.random_cloud(7000 + seed, n, d, kind)
    radius = [math.inf, 0.8, 1.5, 3.0][seed % 4]
    path, res = edges_equal(vrb, X, radius, strict=seed % 5 == 1)
    if res.count(1)[0] >= 2:
        assert path == "bucket"


@pytest.mark.parametrize("kind", ["lattice", "halfint", "dups", "uniform", "gauss"])
def test_radix_path_forced(vrb, kind, monkeypatch):
    monkeypatch.setenv("VRB_EDGE_PATH", "radix")
    X = workloads.random_cloud(7100, 700, 3, kind)
    path, _ = edges_equal(vrb, X, math.inf)
    assert path == "radix"


@pytest.mark.parametrize("kind", ["lattice", "halfint", "dups"])
def test_ties_either_path(vrb, kind):
    # heavy ties: a bucket over 2048 edges sends the build to the radix
    # path; small tie sets stay on the bucket path (records order equal
    # lengths by lex index)
    for n in (40, 300, 2500):
        X = workloads.random_cloud(7200 + n, n, 2, kind)
        edges_equal(vrb, X, math.inf)
        edges_equal(vrb, X, 2.0)


def test_integer_lattice_large_ties_fall_back(vrb):
    X = workloads.integer_lattice(14, 3)   # 2744 points, few distinct lengths
    path, _ = edges_equal(vrb, X, math.inf)
    assert path == "radix"


def test_full_filtration_both_paths(vrb):
    # every pair kept (lex-index records: E < 2^26 and no room for ids)
    X = workloads.random_cloud(7300, 4000, 10, "gauss")
    path, _ = edges_equal(vrb, X, math.inf)
    assert path == "bucket"
    import os
    os.environ["VRB_EDGE_PATH"] = "radix"
    try:
        path, _ = edges_equal(vrb, X, math.inf)
    finally:
        os.environ["VRB_EDGE_PATH"] = "bucket"
    assert path == "radix"


def test_spiky_distribution(vrb):
    # two tight clusters far apart plus a sparse halo: buckets of very
    # different sizes, chunks spanning many empty buckets
    rng = np.random.default_rng(7400)
    A = rng.normal(0.0, 1e-3, (700, 3))
    B = rng.normal(0.0, 1e-3, (700, 3)) + 50.0
    C = rng.uniform(-100, 100, (200, 3))
    X = np.ascontiguousarray(np.concatenate([A, B, C]))
    edges_equal(vrb, X, math.inf)
    edges_equal(vrb, X, 10.0)


def test_unpacked_ids_large_n(vrb):
    # n > 65536: ids are (i, j) arrays, gathered by lex index.  Too large for
    # the oracle's n x n tables: the reference is the definition itself
    # on an independent neighbour search -- the fixed-order RN
    # fold in numpy, (len, i, j) lexsort, dense ranks
    spatial = pytest.importorskip("scipy.spatial")
    X = workloads.random_cloud(7500, 66000, 3, "uniform")
    r = 0.012
    pr = spatial.cKDTree(X).query_pairs(r * 1.001, output_type="ndarray").astype(np.int64)
    i, j = np.minimum(pr[:, 0], pr[:, 1]), np.maximum(pr[:, 0], pr[:, 1])
    acc = np.zeros(len(i))
    for c in range(X.shape[1]):
        t = X[i, c] - X[j, c]
        acc = acc + t * t
    ln = np.sqrt(acc)
    keep = ln <= r
    i, j, ln = i[keep], j[keep], ln[keep]
    o = np.lexsort((j, i, ln))
    i, j, ln = i[o], j[o], ln[o]
    vals, filt = np.unique(ln, return_inverse=True)
    res = vrb.build(X, maxdim=0, radius=r)
    assert vrb.last_edge_path() == "bucket"
    gv, gf = res.simplices(1)
    gv = _u32(gv).astype(np.int64)
    np.testing.assert_array_equal(gv[:, 0], i)
    np.testing.assert_array_equal(gv[:, 1], j)
    np.testing.assert_array_equal(_u32(gf), filt + 1)
    assert _u32(res.rank_values()).tobytes() == vals.tobytes()


def test_bucket_path_triangles(vrb):
    # the edge order feeds S4-S8: a triangle build on the bucket path is
    # element by element the oracle's
    from test_parity_gpu import compare
    X = workloads.random_cloud(7600, 400, 4, "gauss")
    res, _ = compare(vrb, X, 1, 2.0)
    assert vrb.last_edge_path() == "bucket"


def test_default_choice(vrb, monkeypatch):
    # unset: small builds take the radix passes
    monkeypatch.delenv("VRB_EDGE_PATH")
    X = workloads.random_cloud(7800, 500, 3, "uniform")
    path, _ = edges_equal(vrb, X, math.inf)
    assert path == "radix"


def test_tiny(vrb):
    for n in (0, 1, 2, 3):
        X = workloads.random_cloud(7700 + n, n, 2, "uniform")
        edges_equal(vrb, X, math.inf)


@pytest.mark.parametrize("scale", [1.0, 1e-3, 1e-30, 1e12, 1e17])
def test_cap_at_pair_lengths(vrb, scale, monkeypatch):
    # the cap decision (S2, reading A1) is taken on an FP32 fold with an
    # error bound and re-done in FP64 near the threshold: caps exactly at
    # pair lengths (inclusive keeps the pair, strict drops it) and one ulp
    # around them, at scales where FP32 rounding, subnormals or overflow bite
    monkeypatch.delenv("VRB_EDGE_PATH")
    X = workloads.random_cloud(7900, 300, 5, "gauss") * scale
    rng = np.random.default_rng(7901)
    for _ in range(3):
        i, j = sorted(rng.choice(300, 2, replace=False))
        L = oracle.length(X, int(i), int(j))
        for r in (L, np.nextafter(L, 0.0), np.nextafter(L, np.inf)):
            for strict in (False, True):
                edges_equal(vrb, X, float(r), strict=strict)
