"""GPU parity of vrb_gf2_blockprodsum (S = D + C E over GF(2),
sec. 4.6) against the oracle's dense-accumulator definition and,
at size, against scipy's sparse integer product reduced mod 2 (an
independent library routine)."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vrb():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_04424_b200 as m
    return m


def rand_csc_fast(rng, nr, nc, per_col):
    """Vectorised: per column up to per_col distinct sorted rows."""
    cnt = rng.integers(0, per_col + 1, nc)
    col = np.repeat(np.arange(nc, dtype=np.int64), cnt)
    key = np.unique(col * nr + rng.integers(0, nr, col.size))
    c, r = key // nr, (key % nr).astype(np.uint32)
    cp = np.zeros(nc + 1, dtype=np.int64)
    np.add.at(cp, c + 1, 1)
    return np.cumsum(cp), r


def rand_csc(rng, nr, nc, per_col, sort=True, dups=False):
    cols = []
    for _ in range(nc):
        m = int(rng.integers(0, per_col + 1))
        if nr == 0:
            m = 0
        c = rng.integers(0, max(nr, 1), m).astype(np.uint32)
        if not dups:
            c = np.unique(c)
        if sort:
            c = np.sort(c)
        else:
            rng.shuffle(c)
        cols.append(c)
    cp = np.zeros(nc + 1, dtype=np.int64)
    for j, c in enumerate(cols):
        cp[j + 1] = cp[j] + len(c)
    rv = np.concatenate(cols).astype(np.uint32) if cp[-1] else np.zeros(0, dtype=np.uint32)
    return cp, rv


def dev(m):
    cp, rv = m
    return torch.from_numpy(cp).cuda(), torch.from_numpy(rv.view(np.int32)).cuda()


def run(vrb, nr, D, C, E):
    S = vrb.gf2_blockprodsum(nr, dev(D), dev(C), dev(E))
    return S.colptr.cpu().numpy(), S.rowval.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("seed", range(16))
def test_blockprodsum_vs_oracle(vrb, seed):
    rng = np.random.default_rng(9000 + seed)
    nr, k, nc = (int(x) for x in rng.integers(0, 300, 3))
    kw = dict(sort=seed % 3 != 0, dups=seed % 4 == 0)
    D, C, E = rand_csc(rng, nr, nc, 6, **kw), rand_csc(rng, nr, k, 5, **kw), rand_csc(rng, k, nc, 7, **kw)
    cp, rv = run(vrb, nr, D, C, E)
    ocp, orv = oracle.blockprodsum(nr, D, C, E)
    np.testing.assert_array_equal(cp, ocp)
    np.testing.assert_array_equal(rv, orv)


def test_blockprodsum_boundary_shaped(vrb):
    # C = D_2 of a VR complex (3 rows per column), built by the oracle;
    # E selects a few triangles per column, D is sparse noise
    import workloads
    w = workloads.WORKLOADS["C2"]
    o = oracle.Oracle(w.points(), w.radius)
    _, _, rows = o.simplices(2)
    T, Ecount = rows.shape[0], o.E
    C = (3 * np.arange(T + 1, dtype=np.int64), rows.reshape(-1).astype(np.uint32))
    rng = np.random.default_rng(42)
    nc = 20000
    E = rand_csc(rng, T, nc, 6)
    D = rand_csc(rng, Ecount, nc, 3)
    cp, rv = run(vrb, Ecount, D, C, E)
    ocp, orv = oracle.blockprodsum(Ecount, D, C, E)
    np.testing.assert_array_equal(cp, ocp)
    np.testing.assert_array_equal(rv, orv)


def test_blockprodsum_large_vs_scipy(vrb):
    sp = pytest.importorskip("scipy.sparse")
    rng = np.random.default_rng(7)
    nr, k, nc = 2_000_000, 1_000_000, 1_000_000
    D, C, E = rand_csc_fast(rng, nr, nc, 4), rand_csc_fast(rng, nr, k, 5), rand_csc_fast(rng, k, nc, 4)
    cp, rv = run(vrb, nr, D, C, E)

    def mat(m, nrows):
        return sp.csc_matrix((np.ones(len(m[1]), dtype=np.int64), m[1].astype(np.int64), m[0]),
                             shape=(nrows, len(m[0]) - 1))
    ref = (mat(D, nr) + mat(C, nr) @ mat(E, k)).tocsc()
    ref.data %= 2
    ref.eliminate_zeros()
    ref.sort_indices()
    np.testing.assert_array_equal(cp, ref.indptr.astype(np.int64))
    np.testing.assert_array_equal(rv, ref.indices.astype(np.uint32))


def test_blockprodsum_edge_cases(vrb):
    empty = (np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.uint32))
    cp, rv = run(vrb, 5, empty, (np.zeros(3, dtype=np.int64), np.zeros(0, dtype=np.uint32)), empty)
    assert cp.tolist() == [0] and rv.size == 0
    # x + x = 0: a column of D equal to C E cancels
    C = (np.array([0, 2], dtype=np.int64), np.array([1, 3], dtype=np.uint32))
    E = (np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.uint32))
    D = (np.array([0, 2], dtype=np.int64), np.array([3, 1], dtype=np.uint32))
    cp, rv = run(vrb, 4, D, C, E)
    assert cp.tolist() == [0, 0] and rv.size == 0
    with pytest.raises(vrb.VrbError):
        run(vrb, 2, D, C, E)          # row 3 >= nrows = 2


@pytest.mark.parametrize("which", ["D", "C", "E"])
def test_blockprodsum_index_minus_one_rejected(vrb, which):
    # an int32 -1 is the u32 index 0xFFFFFFFF: out of range in every operand
    # (the range check once wrapped it to 0 and passed)
    ok = {"D": (np.array([0, 1], dtype=np.int64), np.array([1], dtype=np.uint32)),
          "C": (np.array([0, 2], dtype=np.int64), np.array([0, 2], dtype=np.uint32)),
          "E": (np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.uint32))}
    cp, rv = ok[which]
    bad = rv.copy()
    bad[-1] = 0xFFFFFFFF
    ops = dict(ok)
    ops[which] = (cp, bad)
    with pytest.raises(vrb.VrbError) as ei:
        run(vrb, 4, ops["D"], ops["C"], ops["E"])
    assert ei.value.status == vrb.VRB_EINVAL
    run(vrb, 4, ok["D"], ok["C"], ok["E"])   # the unmodified operands are accepted


def test_blockprodsum_bad_colptr_rejected(vrb):
    C = (np.array([0, 2], dtype=np.int64), np.array([1, 3], dtype=np.uint32))
    E = (np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.uint32))
    for cp in ([1, 2], [0, 3, 2]):   # not starting at 0; decreasing
        nc = len(cp) - 1
        D = (np.array(cp, dtype=np.int64), np.array([0, 1, 2], dtype=np.uint32)[:max(cp)])
        Ek = (np.arange(nc + 1, dtype=np.int64), np.zeros(nc, dtype=np.uint32))
        with pytest.raises(vrb.VrbError) as ei:
            run(vrb, 4, D, C, Ek)
        assert ei.value.status == vrb.VRB_EINVAL
