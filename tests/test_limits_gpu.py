"""GPU parity on inputs at the edges of the layout:
an owner edge whose apex set exceeds the 512-entry warp scratch of the
tetrahedron kernels (handled by k_tets_big), through the dense pair-table
kernel and the sparse one, with the owner edge alone at its level (direct
face positions) and sharing it (face search by triple).

Definition: a tetrahedron is built when all six of its edges
are; its owner is its longest edge in the (len, i, j) order.  The inputs are
distance matrices (F3) so the combinatorics can be set exactly.
"""
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


def _np(t):
    return t.cpu().numpy().view(np.uint32) if t.dtype == torch.int32 else t.cpu().numpy()


def big_apex_matrix(m_apex=600, clique=14, tie=False, seed=0):
    """Vertices 0, 1 at distance 1 (the longest kept edge, its own level
    unless tie); m_apex apexes at ~0.9 from both (so edge (0, 1) owns
    m_apex triangles); apexes mutually at 2.0 (not kept at r = 1) except a
    clique of `clique` apexes at ~0.5 (so (0, 1) owns C(clique, 2)
    tetrahedra).  tie: two more vertices at distance exactly 1.0 share the
    owner's level."""
    rng = np.random.default_rng(seed)
    extra = 2 if tie else 0
    n = 2 + m_apex + extra
    D = np.full((n, n), 2.0)
    np.fill_diagonal(D, 0.0)
    D[0, 1] = D[1, 0] = 1.0
    a = np.arange(2, 2 + m_apex)
    d0 = 0.9 + rng.uniform(-0.05, 0.05, m_apex)
    d1 = 0.9 + rng.uniform(-0.05, 0.05, m_apex)
    D[0, a] = D[a, 0] = d0
    D[1, a] = D[a, 1] = d1
    c = a[rng.choice(m_apex, clique, replace=False)]
    for i in range(clique):
        for j in range(i + 1, clique):
            v = 0.5 + rng.uniform(-0.1, 0.1)
            D[c[i], c[j]] = D[c[j], c[i]] = v
    if tie:
        u, w = n - 2, n - 1
        D[u, w] = D[w, u] = 1.0
    return D


@pytest.mark.parametrize("tie", [False, True])
@pytest.mark.parametrize("sparse", [False, True])
def test_owner_edge_with_more_than_512_triangles(vrb, monkeypatch, tie, sparse):
    if sparse:
        monkeypatch.setenv("VRB_FORCE_SPARSE_TETS", "1")
    D = big_apex_matrix(tie=tie, seed=3 + tie)
    res = vrb.build_dm(D, maxdim=2, radius=1.0)
    o = oracle.Oracle(None, 1.0, False, D=D)
    ev, ef, _, vor = o.edges()
    np.testing.assert_array_equal(_np(res.simplices(1)[0]), ev)
    for k in (2, 3):
        v, f, r = o.simplices(k)
        gv, gf = res.simplices(k)
        np.testing.assert_array_equal(_np(gv), v)
        np.testing.assert_array_equal(_np(gf), f)
        np.testing.assert_array_equal(_np(res.boundary(k)), r)
    # the owner edge (0, 1) is the last kept edge of length 1 and owns every
    # apex triangle and every clique-pair tetrahedron
    tv, tf, _ = o.simplices(2)
    top = ef.max()
    assert ((tv[:, 0] == 0) & (tv[:, 1] == 1) & (tf == top)).sum() == 600
    assert o.simplices(3)[0].shape[0] >= 14 * 13 // 2


def test_tetrahedra_vertex_limit_is_rejected_before_work(vrb):
    # K = 3 needs n <= tets_max_n() (38 784 on a B200: the sparse kernel's
    # shared-memory host map) -- rejected up front, not after the triangles
    import time
    X = np.random.default_rng(0).uniform(0, 1, (40000, 3))
    t0 = time.time()
    with pytest.raises(vrb.VrbError) as ei:
        vrb.build(X, maxdim=2, radius=0.01)
    assert ei.value.status == vrb.VRB_ENOTSUP
    assert time.time() - t0 < 5.0
    res = vrb.build(X, maxdim=1, radius=0.01)   # triangles have no such limit
    assert res.count(2)[0] >= 0
