"""GPU error paths of the C ABI (include/vrb.h "Errors"): non-finite input,
out-of-range accessors, skipped boundary arrays, allocation failure through
the hook, and u32 position overflow -- each a status code, no handle, no
leak, and the library stays usable afterwards."""
import ctypes
import math

import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vrb():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_04424_b200 as m
    return m


def _status(vrb, fn):
    with pytest.raises(vrb.VrbError) as ei:
        fn()
    return ei.value.status


def test_non_finite_coordinates(vrb):
    for bad in (np.nan, np.inf, -np.inf):
        X = workloads.random_cloud(1, 100, 3, "uniform")
        X[37, 1] = bad
        assert _status(vrb, lambda: vrb.build(X, maxdim=1)) == vrb.VRB_EINVAL
        assert _status(vrb, lambda: vrb.build(torch.from_numpy(X).cuda(), maxdim=1)) == vrb.VRB_EINVAL
    vrb.build(workloads.random_cloud(1, 100, 3, "uniform"), maxdim=1)   # still usable


def test_accessor_ranges_and_skipped_boundary(vrb):
    X = workloads.random_cloud(2, 60, 3, "uniform")
    res = vrb.build(X, maxdim=1, radius=0.5, skip_boundary=True)
    assert _status(vrb, lambda: res.simplices(3)) == vrb.VRB_EINVAL      # K = 2
    assert _status(vrb, lambda: res.count(-1)) == vrb.VRB_EINVAL
    assert _status(vrb, lambda: res.boundary(2)) == vrb.VRB_EINVAL       # VRB_SKIP_BOUNDARY
    assert res.boundary(1).shape[1] == 2                                    # D_1 aliases the edges
    assert _status(vrb, lambda: res.boundary(0)) == vrb.VRB_EINVAL


def test_allocation_failure_through_the_hook(vrb):
    L = vrb.lib()
    calls = {"n": 0}

    def alloc(nbytes, dev, stream, ctx):
        calls["n"] += 1
        if calls["n"] > 6:           # fail part-way through a build
            return None
        return torch.cuda.caching_allocator_alloc(int(nbytes), int(dev), int(stream or 0))

    def free(ptr, nbytes, dev, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    hooks = (vrb.ALLOC_FN(alloc), vrb.FREE_FN(free))
    assert L.vrb_set_allocator(hooks[0], hooks[1], None) == 0
    try:
        X = workloads.random_cloud(3, 400, 3, "uniform")
        assert _status(vrb, lambda: vrb.build(X, maxdim=2, radius=0.3)) == vrb.VRB_ENOMEM
    finally:
        vrb.use_torch_allocator(False)
    res = vrb.build(workloads.random_cloud(3, 400, 3, "uniform"), maxdim=2, radius=0.3)
    assert res.count(3)[0] >= 0


def test_triangle_positions_overflow_u32(vrb):
    # C(2960, 3) = 4.32e9 triangles at full filtration >= 2^32: the count pass
    # runs, then the build stops with VRB_EOVERFLOW before allocating outputs
    X = workloads.random_cloud(4, 2960, 3, "uniform")
    assert math.comb(2960, 3) >= 1 << 32
    vrb.use_torch_allocator(True)
    try:
        assert _status(vrb, lambda: vrb.build(torch.from_numpy(X).cuda(), maxdim=1)) == vrb.VRB_EOVERFLOW
    finally:
        vrb.use_torch_allocator(False)
        torch.cuda.empty_cache()


def test_h0_and_gf2_reject_bad_handles(vrb):
    L = vrb.lib()
    assert L.vrb_h0(None, None, None, None, None, None) == vrb.VRB_EINVAL
    assert L.vrb_gf2_csc(None, None, None, None) == vrb.VRB_EINVAL
    assert L.vrb_gf2_free(None) == vrb.VRB_OK
    out = ctypes.c_void_p()
    assert L.vrb_gf2_blockprodsum(-1, 0, 0, None, None, None, None, None, None, None, ctypes.byref(out)) == \
        vrb.VRB_EINVAL
