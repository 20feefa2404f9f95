"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/vrb.h declares, and rejects bad arguments before touching a device."""
import ctypes
import math
import os
import re

import pytest

import paper_1809_04424_b200 as vrb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "vrb.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(vrb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding_exports():
    assert _declared_symbols() == sorted(vrb.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = vrb.lib()
    for name in _declared_symbols():
        assert hasattr(L, name), name
    assert vrb.abi_version() == 2


def test_binding_has_no_oracle_or_cpu_path():
    pkg = os.path.join(ROOT, "paper_1809_04424_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "vr_oracle" not in src and "liboracle" not in src, f


def _build_status(n, d, maxdim, radius, X=True):
    L = vrb.lib()
    opts = vrb.vrb_opts(maxdim, radius, 0)
    h = ctypes.c_void_p()
    buf = (ctypes.c_double * 4)(0.0, 0.0, 1.0, 1.0)
    st = L.vrb_build(ctypes.cast(buf, ctypes.c_void_p) if X else None, n, d, ctypes.byref(opts), None,
                     ctypes.byref(h))
    return st, h.value, L.vrb_last_error().decode()


@pytest.mark.parametrize("n,d,maxdim,radius", [(-1, 2, 1, 1.0), (2, 0, 1, 1.0), (2, 2, 3, 1.0),
                                               (2, 2, -1, 1.0), (2, 2, 1, -0.5), (2, 2, 1, math.nan)])
def test_build_rejects_bad_arguments(n, d, maxdim, radius):
    st, h, msg = _build_status(n, d, maxdim, radius)
    assert st == vrb.VRB_EINVAL and h is None and msg


def test_build_rejects_null_points():
    st, h, msg = _build_status(2, 2, 1, 1.0, X=False)
    assert st == vrb.VRB_EINVAL


def test_too_many_vertices_is_overflow():
    st, h, msg = _build_status(1 << 21, 2, 1, 1.0)
    assert st == vrb.VRB_EOVERFLOW


def test_allocator_hooks_must_come_in_pairs():
    L = vrb.lib()
    st = L.vrb_set_allocator(vrb.ALLOC_FN(lambda *a: None), vrb.FREE_FN(), None)
    assert st == vrb.VRB_EINVAL
    assert L.vrb_set_allocator(vrb.ALLOC_FN(), vrb.FREE_FN(), None) == vrb.VRB_OK


def test_accessors_reject_null_handle():
    L = vrb.lib()
    g = ctypes.c_int64()
    assert L.vrb_count(None, 1, ctypes.byref(g), None, None) == vrb.VRB_EINVAL
    assert L.vrb_free(None) == vrb.VRB_OK
