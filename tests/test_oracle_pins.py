"""Pins of the CPU oracle to facts fixed by the paper and by mathematics.

Every test here checks ``oracle/`` against something other than itself:
printed values (tests/golden/*.json, each with its PAPER.md citation), closed
forms, independent brute force, invariants of the definition, and a
rational-arithmetic model of IEEE round-to-nearest.  See DESIGN.md "Oracle
pins" for the table mapping each oracle function to the pins below.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

INF = math.inf


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _radius(v):
    return INF if v == "inf" else float(v)


# --------------------------------------------------------------------------
# Step 1: distances (reading A5).  Pin P1.
# --------------------------------------------------------------------------

def test_length_345_and_unit_square():
    X = np.array([[0.0, 0.0], [3.0, 4.0]])
    assert oracle.length(X, 0, 1) == 5.0
    sq = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)
    got = sorted(oracle.length(sq, i, j) for i in range(4) for j in range(i + 1, 4))
    assert got == [1.0, 1.0, 1.0, 1.0, math.sqrt(2.0), math.sqrt(2.0)]


def test_length_integer_coordinates_exact():
    # Integer coordinates: every partial sum is an exact integer < 2^53, so the
    # fold is exact and len is the correctly rounded sqrt of an integer.
    rng = np.random.default_rng(11)
    X = rng.integers(-1000, 1000, (40, 7)).astype(np.float64)
    for i in range(40):
        for j in range(i + 1, 40):
            d2 = int(sum((int(a) - int(b)) ** 2 for a, b in zip(X[i], X[j])))
            assert oracle.length(X, i, j) == math.sqrt(d2)


def _rn(q: Fraction) -> Fraction:
    """Round an exact rational to the nearest binary64 (float(Fraction) is RN)."""
    return Fraction(float(q))


def test_length_fold_is_unfused_round_to_nearest():
    # Model of reading A5 in exact rationals with explicit RN after every
    # operation (no contraction): acc <- RN(acc + RN(t*t)), t = RN(x - y).
    # A fused multiply-add would round acc + t*t once; the test also checks that
    # the inputs are sensitive to that difference, so an FMA build would fail.
    rng = np.random.default_rng(5)
    X = rng.standard_normal((60, 10))
    fused_differs = 0
    for i in range(0, 60, 2):
        j = i + 1
        acc = Fraction(0)
        acc_fma = Fraction(0)
        for c in range(10):
            t = _rn(Fraction(X[i, c]) - Fraction(X[j, c]))
            acc = _rn(acc + _rn(t * t))
            acc_fma = _rn(acc_fma + t * t)
        want = math.sqrt(float(acc))
        assert oracle.length(X, i, j) == want
        fused_differs += math.sqrt(float(acc_fma)) != want
    assert fused_differs > 0


def test_length_within_error_bound_of_exact():
    # |len - sqrt(exact d2)| <= (d + 3) u len  (u = 2^-53; textbook bound for
    # a d-term recursive sum of rounded squares followed by a rounded sqrt).
    rng = np.random.default_rng(6)
    X = rng.uniform(-3, 3, (50, 5))
    u = 2.0 ** -53
    for i in range(50):
        for j in range(i + 1, 50, 7):
            exact = sum((Fraction(a) - Fraction(b)) ** 2 for a, b in zip(X[i], X[j]))
            ref = math.sqrt(float(exact))
            got = oracle.length(X, i, j)
            assert abs(got - ref) <= (5 + 3) * u * ref + 1e-300


# --------------------------------------------------------------------------
# Step 3: ranking.  Pins P2, P3.
# --------------------------------------------------------------------------

def test_sortperm_literal():
    g = _load("sortperm_literal.json")
    for case in g["cases"]:
        perm, dense = oracle.sortperm(case["v"])
        assert (perm + 1).tolist() == case["sortperm_1based"]
        assert dense.tolist() == case["dense_rank"]


def test_sortperm_matches_counting_definition():
    rng = np.random.default_rng(3)
    v = rng.integers(0, 20, 300).astype(np.float64) * 0.25
    perm, dense = oracle.sortperm(v)
    distinct = sorted(set(v.tolist()))
    for i in range(v.size):                      # dense = 1 + #distinct below
        assert dense[i] == 1 + sum(1 for x in distinct if x < v[i])
    keys = [(v[p], p) for p in perm]               # stable ascending
    assert keys == sorted(keys)


def test_lattice_333_ties():
    g = _load("lattice_333.json")
    X = workloads.integer_lattice(g["side"], g["dim"])
    o = oracle.Oracle(X)
    ev, ef, el, vor = o.edges()
    assert o.E == 351 and o.nvals == 9
    assert np.bincount(ef)[1:].tolist() == g["multiplicity"]
    assert vor.tolist() == [math.sqrt(x) for x in g["d2"]]
    # every edge's length is value_of_rank[filt - 1]
    assert np.array_equal(vor[ef - 1], el)


# --------------------------------------------------------------------------
# Golden arrays (pin P15): unit square and the five-point tie example.
# --------------------------------------------------------------------------

def _check_complex(o, g, maxdim):
    ev, ef, el, vor = o.edges()
    assert ev.tolist() == g["edge_vertices"]
    assert ef.tolist() == g["edge_filt"]
    assert vor.tolist() == g["value_of_rank"]
    tv, tf, tr = o.simplices(2)
    assert tv.tolist() == g["triangles"]
    assert tf.tolist() == g["triangle_filt"]
    assert tr.tolist() == g["d2_rows"]
    assert o.barcodes(maxdim).tolist() == sorted(g["bars"])


def test_golden_unit_square():
    g = _load("unit_square.json")
    o = oracle.Oracle(np.array(g["points"], dtype=np.float64), _radius(g["radius"]))
    _check_complex(o, g, g["maxdim"])
    reals = o.bars_real(o.barcodes(1))
    assert (1, 1.0, math.sqrt(2.0)) in reals      # SPEC S:314 unit square [1, sqrt 2)


def test_golden_ties_and_cap():
    g = _load("ties_five_points.json")
    X = np.array(g["points"], dtype=np.float64)
    _check_complex(oracle.Oracle(X, INF), g["full"], g["maxdim"])
    for key in ("inclusive_r5", "strict_r5"):
        c = g[key]
        o = oracle.Oracle(X, c["radius"], strict=c["strict"])
        assert o.E == c["n_edges"]
        assert o.simplices(2)[0].shape[0] == c["n_triangles"]
        assert o.barcodes(g["maxdim"]).tolist() == sorted(c["bars"])


# --------------------------------------------------------------------------
# Step 8 mapping (pin P4): Fig. 4 pivot (v3, e5) -> bar (3, 5).
# --------------------------------------------------------------------------

@pytest.mark.parametrize("method", ["col", "row"])
def test_fig4_pivot_to_bar(method):
    g = _load("fig4_pivot.json")
    piv, zero = oracle.reduce(4, g["edges"], method)
    r = g["printed_pivot"]["row_1based"] - 1
    c = g["printed_pivot"]["column_1based"] - 1
    assert piv[r] == c
    assert [g["vertex_times"][r], g["edge_times"][c]] == g["printed_pivot"]["bar"]
    # one vertex is never a pivot row: the extra [0, inf) bar
    unpaired = [v for v in range(4) if piv[v] < 0]
    assert [g["vertex_times"][v] for v in unpaired] == [g["printed_infinite_bar"][0]]


# --------------------------------------------------------------------------
# Counts (pins P5, P6).
# --------------------------------------------------------------------------

def test_full_filtration_binomial_counts():
    X = workloads.random_cloud(7, 30, 3)
    o = oracle.Oracle(X)
    assert o.E == math.comb(30, 2)
    assert o.simplices(2)[0].shape[0] == math.comb(30, 3)
    assert o.simplices(3)[0].shape[0] == math.comb(30, 4)


@pytest.mark.parametrize("row", [0, 1])
def test_table_oscmach_size_of_complex(row):
    # "Size of complex" of Table OSCmach = vertices + edges + triangles at full
    # filtration (maxdim 1), printed to two significant figures.
    r = _load("table_oscmach.json")["rows"][row]
    n = r["n"]
    X = workloads.random_cloud(100 + n, n, 3)
    o = oracle.Oracle(X)
    T = int(o.filt_hist(2).sum())
    size = n + o.E + T
    assert size == math.comb(n, 1) + math.comb(n, 2) + math.comb(n, 3)
    assert float(f"{size:.1e}") == r["printed"]


def test_table_oscmach_binomial_reading():
    for r in _load("table_oscmach.json")["rows"]:
        n = r["n"]
        size = math.comb(n, 1) + math.comb(n, 2) + math.comb(n, 3)
        assert float(f"{size:.1e}") == r["printed"], r["name"]


def _adjacency(o):
    ev = o.edges()[0]
    A = np.zeros((o.n, o.n), dtype=np.int64)
    A[ev[:, 0], ev[:, 1]] = 1
    A[ev[:, 1], ev[:, 0]] = 1
    return A


@pytest.mark.parametrize("seed,n,r", [(1, 120, 0.3), (2, 80, 0.45), (3, 150, 0.25)])
def test_capped_counts_by_linear_algebra(seed, n, r):
    X = workloads.random_cloud(seed, n, 3)
    o = oracle.Oracle(X, r)
    A = _adjacency(o)
    T = int(np.trace(A @ A @ A)) // 6
    Q = 0
    for v in range(n):
        nb = np.nonzero(A[v])[0]
        S = A[np.ix_(nb, nb)]
        Q += int(np.trace(S @ S @ S)) // 6
    assert Q % 4 == 0
    assert o.simplices(2)[0].shape[0] == T
    assert o.simplices(3)[0].shape[0] == Q // 4


# --------------------------------------------------------------------------
# Brute force over all subsets for n <= 10 (pin P7).
# --------------------------------------------------------------------------

def _brute(X, radius, strict, K):
    return _brute_len(X.shape[0], lambda i, j: oracle.length(X, i, j), radius, strict, K)   # length pinned above (P1)


def _brute_len(n, length_of, radius, strict, K):
    L = {}
    for i in range(n):
        for j in range(i + 1, n):
            length = length_of(i, j)
            if (length < radius) if strict else (length <= radius):
                L[(i, j)] = length
    vals = sorted(set(L.values()))
    rank = {e: 1 + sum(1 for x in vals if x < v) for e, v in L.items()}
    out = {1: sorted(L, key=lambda e: (L[e], e))}
    filt = {1: {e: rank[e] for e in L}}
    for k in range(2, K + 1):
        simp = []
        for s in itertools.combinations(range(n), k + 1):
            if all(p in L for p in itertools.combinations(s, 2)):
                simp.append(s)
        filt[k] = {s: max(rank[p] for p in itertools.combinations(s, 2)) for s in simp}
        out[k] = sorted(simp, key=lambda s: (filt[k][s], s))
    rows = {}
    for k in range(1, K + 1):
        prev = list(range(n)) if k == 1 else out[k - 1]
        idx = {((s,) if k == 1 else s): q for q, s in enumerate(prev)}
        rows[k] = [sorted(idx[f if k > 1 else (f[0],)] for f in itertools.combinations(s, k))
                   for s in out[k]]
    return out, filt, rows, vals


@pytest.mark.parametrize("seed", range(24))
def test_bruteforce_small(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["uniform", "lattice", "dups", "halfint", "gauss"][seed % 5]
    n = int(rng.integers(0, 11))
    d = int(rng.integers(1, 4))
    X = workloads.random_cloud(seed, n, d, kind)
    radius = [INF, 1.0, 1.5, 0.6, 2.0][seed % 5]
    strict = bool(seed % 3 == 0)
    K = 3
    out, filt, rows, vals = _brute(X, radius, strict, K)
    o = oracle.Oracle(X, radius, strict)
    ev, ef, el, vor = o.edges()
    assert [tuple(e) for e in ev.tolist()] == out[1]
    assert ef.tolist() == [filt[1][e] for e in out[1]]
    assert vor.tolist() == vals
    for k in (2, 3):
        v, f, r = o.simplices(k)
        assert [tuple(s) for s in v.tolist()] == out[k]
        assert f.tolist() == [filt[k][s] for s in out[k]]
        assert r.tolist() == rows[k]


def test_edge_cases_tiny_inputs():
    o = oracle.Oracle(np.zeros((0, 3)))
    assert o.E == 0 and o.simplices(2)[0].shape == (0, 3)
    o = oracle.Oracle(np.zeros((1, 2)))
    assert o.E == 0 and o.barcodes(1).tolist() == [[0, 0, -1]]
    # duplicates at r = 0: zero-length edge of filt 1 (reading A11)
    X = np.array([[0.5, 0.5], [0.5, 0.5], [2.0, 0.0]])
    o = oracle.Oracle(X, 0.0)
    ev, ef, el, vor = o.edges()
    assert ev.tolist() == [[0, 1]] and ef.tolist() == [1] and el.tolist() == [0.0]
    # zero-length bar dropped by default, kept with keep_zero (reading A9)
    assert o.barcodes(0).tolist() == [[0, 0, -1], [0, 0, -1]]
    assert o.barcodes(0, keep_zero=True).tolist() == [[0, 0, -1], [0, 0, -1], [0, 0, 1]]


def test_two_components_give_two_infinite_bars():
    # reading A8: one [0, inf) bar per connected component at the cap
    X = np.concatenate([workloads.random_cloud(1, 8, 2), workloads.random_cloud(2, 8, 2) + 10.0])
    o = oracle.Oracle(X, 3.0)
    bars = o.barcodes(1)
    assert sum(1 for b in bars if b[0] == 0 and b[2] < 0) == 2


# --------------------------------------------------------------------------
# Invariants of order and boundary (pins P8, P9).
# --------------------------------------------------------------------------

def _gf2_product_is_zero(rows_lo, rows_hi, n_mid):
    # (D_k D_{k+1}) over GF(2): column c of the product = sum of columns of D_k
    # at the rows of column c of D_{k+1}.
    for col in rows_hi:
        acc = {}
        for r in col:
            for x in rows_lo[r]:
                acc[x] = acc.get(x, 0) ^ 1
        if any(acc.values()):
            return False
    return True


@pytest.mark.parametrize("seed", range(6))
def test_order_and_boundary_invariants(seed):
    kind = ["uniform", "lattice", "halfint"][seed % 3]
    X = workloads.random_cloud(seed, 24, 3, kind)
    radius = [0.7, 2.0, 1.6][seed % 3]
    o = oracle.Oracle(X, radius)
    ev, ef, el, vor = o.edges()
    fprev = {1: ef}
    vprev = {1: ev}
    d1 = [list(e) for e in ev.tolist()]
    allrows = {1: d1}
    for k in (2, 3):
        v, f, r = o.simplices(k)
        keys = [(int(f[q]), tuple(v[q])) for q in range(len(f))]
        assert all(a < b for a, b in zip(keys, keys[1:]))          # unique total order
        assert (np.diff(v, axis=1) > 0).all() if len(v) else True   # vertices ascending
        for q in range(len(f)):
            rr = r[q].tolist()
            assert len(rr) == k + 1 and rr == sorted(set(rr))
            rf = [int(fprev[k - 1][x]) for x in rr]
            assert max(rf) <= f[q]                                   # face filt <= cofacet filt
            assert rf[-1] == f[q]                                    # lowest row carries the filt
            for t, x in enumerate(rr):                               # rows are the faces
                assert set(vprev[k - 1][x].tolist()) <= set(v[q].tolist())
        fprev[k], vprev[k] = f, v
        allrows[k] = r.tolist()
    assert _gf2_product_is_zero(allrows[1], allrows[2], o.E)
    assert _gf2_product_is_zero(allrows[2], allrows[3], len(fprev[2]))


# --------------------------------------------------------------------------
# Barcodes: known shapes (pin P10), Euler (P11), backend agreement (P12).
# --------------------------------------------------------------------------

def _alive_at_cap(bars, maxdim):
    return tuple(int(sum(1 for b in bars if b[0] == k and b[2] < 0)) for k in range(maxdim + 1))


@pytest.mark.parametrize("cap,betti", [(0.2, (1, 1)), (1.0, (1, 1)), (1.8, (1, 0))])
def test_betti_circle(cap, betti):
    X = workloads.circle_jitter(50, 1e-3, 0)
    o = oracle.Oracle(X, cap)
    assert _alive_at_cap(o.barcodes(1), 1) == betti


@pytest.mark.parametrize("cap", [0.35, 0.45, 0.6])
def test_betti_fibonacci_sphere(cap):
    o = oracle.Oracle(workloads.fibonacci_sphere(300), cap)
    assert _alive_at_cap(o.barcodes(2, method="clear"), 2) == (1, 0, 1)


def test_betti_torus_grid():
    o = oracle.Oracle(workloads.torus_grid(12, 30), 0.4)
    assert _alive_at_cap(o.barcodes(2, method="clear"), 2) == (1, 2, 1)


def test_circle_dominant_bar():
    X = workloads.circle_jitter(50, 1e-3, 0)
    o = oracle.Oracle(X, 1.8)
    bars = o.bars_real(o.barcodes(1))
    one = sorted((d - b for k, b, d in bars if k == 1), reverse=True)
    assert one[0] > 1.0 and (len(one) == 1 or one[1] < 0.1)


@pytest.mark.parametrize("seed", range(8))
def test_euler_characteristic_per_level(seed):
    kind = ["uniform", "lattice", "halfint", "dups"][seed % 4]
    X = workloads.random_cloud(seed, 14, 2 + seed % 2, kind)
    o = oracle.Oracle(X, [0.8, 2.5, 1.5, 0.9][seed % 4])
    maxdim = 2
    bars = o.barcodes(maxdim, keep_zero=True, top=True)
    counts = {0: np.zeros(o.n, dtype=np.int64), 1: o.edges()[1]}
    for k in (2, 3):
        counts[k] = o.simplices(k)[1]
    for f in range(0, o.nvals + 1):
        chi = sum((-1) ** k * int((counts[k] <= f).sum()) for k in range(4))
        betti = sum((-1) ** b[0] for b in bars if b[1] <= f and (b[2] < 0 or f < b[2]))
        assert chi == betti, f


@pytest.mark.parametrize("seed", range(10))
def test_backend_agreement(seed):
    kind = ["uniform", "lattice", "halfint", "dups", "gauss"][seed % 5]
    X = workloads.random_cloud(50 + seed, 12, 3, kind)
    o = oracle.Oracle(X, [1.0, 2.0, 1.3, 0.8, 1.9][seed % 5])
    ref = o.barcodes(2, "col", keep_zero=True, top=True)
    assert np.array_equal(o.barcodes(2, "row", keep_zero=True, top=True), ref)
    assert np.array_equal(o.barcodes(2, "clear", keep_zero=True, top=True), ref)


def test_pivot_pairs_partition_simplices():
    # each simplex is a birth, a death, or unpaired-infinite, exactly once
    X = workloads.random_cloud(9, 14, 3, "uniform")
    o = oracle.Oracle(X, 0.9)
    bars = o.barcodes(2, keep_zero=True, top=True)
    total = o.n + o.E + sum(o.simplices(k)[0].shape[0] for k in (2, 3))
    finite = sum(1 for b in bars if b[2] >= 0)
    infinite = sum(1 for b in bars if b[2] < 0)
    assert 2 * finite + infinite == total


# --------------------------------------------------------------------------
# The per-level helpers used for sampled parity at full size agree with the
# full enumeration (same definitions).
# --------------------------------------------------------------------------

@pytest.mark.parametrize("kind,r", [("uniform", 0.5), ("lattice", 2.3), ("halfint", 1.2)])
def test_level_helpers_match_full_build(kind, r):
    X = workloads.random_cloud(21, 40, 3, kind)
    o = oracle.Oracle(X, r)
    for k in (2, 3):
        v, f, rows = o.simplices(k)
        hist = o.filt_hist(k)
        assert np.array_equal(hist, np.bincount(f, minlength=o.nvals + 1).astype(np.uint64))
        for lvl in sorted(set(f.tolist()))[:: max(1, len(set(f.tolist())) // 7)]:
            sv, sr = o.simplices_at_filt(k, lvl)
            sel = f == lvl
            assert np.array_equal(sv, v[sel])
            if k == 2:
                assert np.array_equal(sr, rows[sel])


def test_c2_mixture_counts_and_betti():
    # C2: torus grid + circle + noise, cap 0.45.  Counts were
    # computed independently in SURVEY 8(a) (scipy pdist + adjacency traces);
    # Betti numbers at the cap (2, 3, 1) are SURVEY 8(c) pin P10.
    w = workloads.WORKLOADS["C2"]
    o = oracle.Oracle(w.points(), w.radius)
    assert o.E == 17169
    assert o.simplices(2)[0].shape[0] == 129438
    assert o.simplices(3)[0].shape[0] == 645405
    assert _alive_at_cap(o.barcodes(2, method="clear"), 2) == (2, 3, 1)


# --------------------------------------------------------------------------
# distance-matrix input ("x is either a point cloud ... or a
# square symmetric matrix (typically a pairwise distance matrix)")
# and latlon2euc.
# --------------------------------------------------------------------------

def test_latlon2euc_printed_worldmap_columns():
    g = _load("latlon2euc_worldmap.json")
    xyz = oracle.latlon2euc(np.array(g["latlon"]))
    np.testing.assert_allclose(xyz, np.array(g["xyz"]), atol=0.6 * 10.0 ** -g["decimals"], rtol=0)
    np.testing.assert_allclose(np.linalg.norm(xyz, axis=1), 1.0, atol=1e-15)     # unit sphere


def _dm_exact(X):
    """Distance matrix of integer-coordinate points: d2 is an exact integer,
    np.sqrt is IEEE correctly rounded, so the entries are the exact lengths."""
    d2 = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    return np.sqrt(d2)


def test_dm_golden_unit_square_and_ties():
    g = _load("unit_square.json")
    X = np.array(g["points"], dtype=np.float64)
    _check_complex(oracle.Oracle(None, _radius(g["radius"]), D=_dm_exact(X)), g, g["maxdim"])
    g = _load("ties_five_points.json")
    X = np.array(g["points"], dtype=np.float64)
    _check_complex(oracle.Oracle(None, INF, D=_dm_exact(X)), g["full"], g["maxdim"])
    for key in ("inclusive_r5", "strict_r5"):
        c = g[key]
        o = oracle.Oracle(None, c["radius"], strict=c["strict"], D=_dm_exact(X))
        assert o.E == c["n_edges"]
        assert o.barcodes(g["maxdim"]).tolist() == sorted(c["bars"])


@pytest.mark.parametrize("seed", range(12))
def test_dm_hamming_bruteforce(seed):
    # HIV-like input (Hamming distances of sequences): integer
    # lengths, heavy ties; against brute force over all subsets
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.integers(0, 10))
    seqs = rng.integers(0, 2, (n, 10))
    D = (seqs[:, None, :] != seqs[None, :, :]).sum(-1).astype(np.float64)
    radius = [INF, 3.0, 4.0, 5.0][seed % 4]
    strict = seed % 3 == 0
    out, filt, rows, vals = _brute_len(n, lambda i, j: D[i, j], radius, strict, 3)
    o = oracle.Oracle(None, radius, strict, D=D)
    ev, ef, el, vor = o.edges()
    assert [tuple(e) for e in ev.tolist()] == out[1]
    assert ef.tolist() == [filt[1][e] for e in out[1]]
    assert vor.tolist() == vals
    for k in (2, 3):
        v, f, r = o.simplices(k)
        assert [tuple(x) for x in v.tolist()] == out[k]
        assert f.tolist() == [filt[k][x] for x in out[k]]
        assert r.tolist() == rows[k]


def test_dm_negative_zero_is_length_zero():
    D = np.array([[0.0, -0.0], [-0.0, 0.0]])
    o = oracle.Oracle(None, 0.0, D=D)
    ev, ef, el, vor = o.edges()
    assert o.E == 1 and np.signbit(el[0]) == 0 and el[0] == 0.0


# --------------------------------------------------------------------------
# blockprodsum S = D + C E over GF(2) (sec. 4.6).
# --------------------------------------------------------------------------

def _rand_csc(rng, nr, nc, density):
    cols = [np.flatnonzero(rng.random(nr) < density).astype(np.uint32) for _ in range(nc)]
    cp = np.zeros(nc + 1, dtype=np.int64)
    for j, c in enumerate(cols):
        cp[j + 1] = cp[j] + len(c)
    rv = np.concatenate(cols) if cols and cp[-1] else np.zeros(0, dtype=np.uint32)
    return cp, rv


def _dense(m, nr):
    cp, rv = m
    M = np.zeros((nr, len(cp) - 1), dtype=np.int64)
    for j in range(len(cp) - 1):
        M[rv[cp[j]:cp[j + 1]], j] = 1
    return M


@pytest.mark.parametrize("seed", range(10))
def test_blockprodsum_matches_dense_mod2_algebra(seed):
    rng = np.random.default_rng(8000 + seed)
    nr, k, nc = (int(x) for x in rng.integers(1, 40, 3))
    D, C, E = _rand_csc(rng, nr, nc, 0.2), _rand_csc(rng, nr, k, 0.15), _rand_csc(rng, k, nc, 0.2)
    S = oracle.blockprodsum(nr, D, C, E)
    ref = (_dense(D, nr) + _dense(C, nr) @ _dense(E, k)) % 2      # numpy integer algebra, then mod 2
    np.testing.assert_array_equal(_dense(S, nr), ref)
    for j in range(nc):                                            # rows strictly ascending
        assert np.all(np.diff(S[1][S[0][j]:S[0][j + 1]].astype(np.int64)) > 0)


def test_blockprodsum_identities_and_worker_partition():
    rng = np.random.default_rng(8100)
    nr, k, nc = 30, 20, 25
    D, C, E = _rand_csc(rng, nr, nc, 0.3), _rand_csc(rng, nr, k, 0.3), _rand_csc(rng, k, nc, 0.3)
    zeroE = (np.zeros(nc + 1, dtype=np.int64), np.zeros(0, dtype=np.uint32))
    S = oracle.blockprodsum(nr, D, C, zeroE)                       # E = 0: S = D
    np.testing.assert_array_equal(S[0], D[0]); np.testing.assert_array_equal(S[1], D[1])
    I = (np.arange(k + 1, dtype=np.int64), np.arange(k, dtype=np.uint32))
    zeroD = (np.zeros(nc + 1, dtype=np.int64), np.zeros(0, dtype=np.uint32))
    S = oracle.blockprodsum(k, zeroD, I, E)                         # D = 0, C = I: S = E
    np.testing.assert_array_equal(S[0], E[0]); np.testing.assert_array_equal(S[1], E[1])
    S = oracle.blockprodsum(nr, D, C, E)
    S2 = oracle.blockprodsum(nr, S, C, E)                           # (D + CE) + CE = D
    np.testing.assert_array_equal(S2[0], D[0]); np.testing.assert_array_equal(S2[1], D[1])
    # master/workers (Fig. BlkProdSum): column blocks computed
    # separately, colptr "adjusted one after the other" on concatenation
    cuts = [0, 7, 8, 19, nc]
    parts_cp, parts_rv, base = [np.zeros(1, dtype=np.int64)], [], 0
    for a, b in zip(cuts[:-1], cuts[1:]):
        Db = (D[0][a:b + 1] - D[0][a], D[1][D[0][a]:D[0][b]])
        Eb = (E[0][a:b + 1] - E[0][a], E[1][E[0][a]:E[0][b]])
        cp, rv = oracle.blockprodsum(nr, Db, C, Eb)
        parts_cp.append(cp[1:] + base)
        parts_rv.append(rv)
        base += cp[-1]
    np.testing.assert_array_equal(np.concatenate(parts_cp), S[0])
    np.testing.assert_array_equal(np.concatenate(parts_rv), S[1])
