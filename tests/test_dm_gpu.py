"""GPU parity of the distance-matrix build (vrb_build_dm) and latlon2euc
(vrb_latlon2euc) -- SURVEY 8(f) F3: "x is either a point cloud ... or a
square symmetric matrix (typically a pairwise distance matrix)",
latlon2euc -- against the CPU oracle on the same inputs.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

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


def compare_dm(vrb, D, maxdim, radius, strict=False, on_device=False):
    Din = torch.from_numpy(D).cuda() if on_device else D
    res = vrb.build_dm(Din, maxdim=maxdim, radius=radius, strict=strict)
    o = oracle.Oracle(None, radius, strict, D=D)
    ev, ef, el, vor = o.edges()
    assert res.count(1)[0] == o.E
    gv, gf = res.simplices(1)
    np.testing.assert_array_equal(_np(gv), ev)
    np.testing.assert_array_equal(_np(gf), ef)
    assert _np(res.rank_values()).tobytes() == vor.tobytes()
    for k in range(2, maxdim + 2):
        v, f, r = o.simplices(k)
        assert res.count(k)[0] == v.shape[0]
        gv, gf = res.simplices(k)
        np.testing.assert_array_equal(_np(gv), v)
        np.testing.assert_array_equal(_np(gf), f)
        np.testing.assert_array_equal(_np(res.boundary(k)), r)
    return res, o


def _hamming(rng, n, L):
    s = rng.integers(0, 2, (n, L)).astype(np.int8)
    return (s[:, None, :] != s[None, :, :]).sum(-1).astype(np.float64)


@pytest.mark.parametrize("seed", range(8))
def test_dm_hamming_heavy_ties(vrb, seed):
    # HIV analog: integer Hamming distances, heavy ties
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(2, 260))
    D = _hamming(rng, n, 24)
    radius = [math.inf, 8.0, 9.0, 10.0][seed % 4]
    compare_dm(vrb, D, 1 if seed % 2 else 2, radius, strict=seed % 3 == 0, on_device=seed % 2 == 0)


@pytest.mark.parametrize("seed", range(6))
def test_dm_random_metric(vrb, seed):
    rng = np.random.default_rng(6000 + seed)
    n = int(rng.integers(40, 400))
    X = rng.standard_normal((n, 4))
    D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    D = np.minimum(D, D.T)                      # exactly symmetric
    np.fill_diagonal(D, 0.0)
    r = float(np.quantile(D[np.triu_indices(n, 1)], 0.05))
    compare_dm(vrb, D, 2 if n < 150 else 1, r)


def test_dm_golden_and_degenerate(vrb):
    X = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)
    D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    compare_dm(vrb, D, 1, math.inf)
    for n in (0, 1, 2):
        compare_dm(vrb, np.zeros((n, n)), 1, math.inf)
    D = np.array([[0.0, -0.0, 2.0], [-0.0, 0.0, 1.0], [2.0, 1.0, 0.0]])   # -0.0 is length 0
    compare_dm(vrb, D, 1, 1.0)


def test_dm_rejects_bad_matrices(vrb):
    good = np.array([[0.0, 1.0], [1.0, 0.0]])
    for bad in (np.array([[0.0, 1.0], [2.0, 0.0]]), np.array([[0.0, -1.0], [-1.0, 0.0]]),
                np.array([[0.0, np.nan], [np.nan, 0.0]]), np.array([[0.0, np.inf], [np.inf, 0.0]])):
        with pytest.raises(vrb.VrbError) as ei:
            vrb.build_dm(bad, maxdim=1)
        assert ei.value.status == vrb.VRB_EINVAL
    np.fill_diagonal(good, np.nan)            # the diagonal is not read
    vrb.build_dm(good, maxdim=1)


def test_latlon2euc_printed_worldmap(vrb):
    g = json.load(open(os.path.join(GOLDEN, "latlon2euc_worldmap.json")))
    xyz = vrb.latlon2euc(torch.tensor(g["latlon"], dtype=torch.float64, device="cuda")).cpu().numpy()
    np.testing.assert_allclose(xyz, np.array(g["xyz"]), atol=0.6 * 10.0 ** -g["decimals"], rtol=0)


def test_latlon2euc_vs_oracle_and_worldmap_build(vrb):
    # a WorldMap-sized synthetic catalogue (7322 points): uniform on the
    # sphere; cap 0.15 as in the paper's demo
    rng = np.random.default_rng(7322)
    n = 7322
    lat = np.degrees(np.arcsin(rng.uniform(-1, 1, n)))
    lon = rng.uniform(-180, 180, n)
    ll = np.stack([lat, lon], 1)
    g = vrb.latlon2euc(torch.from_numpy(ll).cuda())
    ref = oracle.latlon2euc(ll)
    np.testing.assert_allclose(g.cpu().numpy(), ref, rtol=0, atol=4e-16)
    # the build from the device coordinates, parity against the oracle on the same bytes
    X = g.cpu().numpy()
    res = vrb.build(g, maxdim=1, radius=0.15)
    o = oracle.Oracle(X, 0.15)
    ev, ef, _, vor = o.edges()
    gv, gf = res.simplices(1)
    np.testing.assert_array_equal(_np(gv), ev)
    np.testing.assert_array_equal(_np(gf), ef)
    v, f, r = o.simplices(2)
    gtv, gtf = res.simplices(2)
    np.testing.assert_array_equal(_np(gtv), v)
    np.testing.assert_array_equal(_np(gtf), f)
    np.testing.assert_array_equal(_np(res.boundary(2)), r)
