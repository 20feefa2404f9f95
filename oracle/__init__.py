"""CPU oracle for the Vietoris-Rips filtration build -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1809_04424_b200``) never imports it and shares no code with it.

This is a thin ctypes wrapper over ``oracle/liboracle.so`` (plain C, see
``vr_oracle.c`` for the step-by-step citations of PAPER.md).  It adds no
arithmetic of the method: it marshals numpy arrays in and out.

Parity status of each function:
  length, sortperm, build (edges), simplices, boundary, barcodes, the
  distance-matrix build, latlon2euc and blockprodsum: pinned by
  tests/test_oracle_pins.py.  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared"]


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc; building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        c_i64, c_i32, c_d, c_p = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        lib.or_length.restype = c_d
        lib.or_length.argtypes = [c_p, c_i32, c_i64, c_i64]
        lib.or_sortperm.restype = None
        lib.or_sortperm.argtypes = [c_p, c_i64, c_p, c_p]
        lib.or_new.restype = c_p
        lib.or_new.argtypes = [c_p, c_i64, c_i32, c_d, c_i32]
        lib.or_new_dm.restype = c_p
        lib.or_new_dm.argtypes = [c_p, c_i64, c_d, c_i32]
        lib.or_latlon2euc.restype = None
        lib.or_latlon2euc.argtypes = [c_p, c_i64, c_p]
        lib.or_free.restype = None
        lib.or_free.argtypes = [c_p]
        lib.or_n_edges.restype = c_i64
        lib.or_n_edges.argtypes = [c_p]
        lib.or_n_vals.restype = c_i64
        lib.or_n_vals.argtypes = [c_p]
        lib.or_get_edges.restype = None
        lib.or_get_edges.argtypes = [c_p, c_p, c_p, c_p, c_p]
        lib.or_edge_pos.restype = c_i64
        lib.or_edge_pos.argtypes = [c_p, c_i64, c_i64]
        lib.or_build_simplices.restype = c_i64
        lib.or_build_simplices.argtypes = [c_p, c_i32]
        lib.or_get_simplices.restype = None
        lib.or_get_simplices.argtypes = [c_p, c_i32, c_p, c_p, c_p]
        lib.or_filt_hist.restype = None
        lib.or_filt_hist.argtypes = [c_p, c_i32, c_p]
        lib.or_simplices_at_filt.restype = c_i64
        lib.or_simplices_at_filt.argtypes = [c_p, c_i32, ctypes.c_uint32, c_p, c_p, c_i64]
        lib.or_barcodes.restype = c_i64
        lib.or_barcodes.argtypes = [c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_i64]
        lib.or_blockprodsum.restype = c_i64
        lib.or_blockprodsum.argtypes = [c_i64, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]
        lib.or_reduce.restype = None
        lib.or_reduce.argtypes = [c_i64, c_i64, c_p, c_p, c_i32, c_p, c_p]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def length(X: np.ndarray, i: int, j: int) -> float:
    """Step 1 (reading A5): sqrt of the fixed-order fold."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    return _L().or_length(_ptr(X), X.shape[1], i, j)


def latlon2euc(latlon) -> np.ndarray:
    """(n, 2) degrees (lat, lon) -> (n, 3) unit-sphere xyz."""
    a = np.ascontiguousarray(latlon, dtype=np.float64).reshape(-1, 2)
    out = np.empty((a.shape[0], 3), dtype=np.float64)
    _L().or_latlon2euc(_ptr(a), a.shape[0], _ptr(out))
    return out


def sortperm(v) -> tuple[np.ndarray, np.ndarray]:
    """(0-based stable ascending permutation, 1-based dense ranks)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    perm = np.empty(v.size, dtype=np.int64)
    dense = np.empty(v.size, dtype=np.uint32)
    _L().or_sortperm(_ptr(v), v.size, _ptr(perm), _ptr(dense))
    return perm, dense


METHOD = {"col": 0, "row": 1, "clear": 2}


def reduce(nrows: int, columns, method: str = "col"):
    """Textbook GF(2) reduction of an arbitrary matrix given as a list of
    ascending row-index lists (Algorithms 1/2).  Returns
    (pivot_row (nrows,) int64: reducing column or -1, zero (ncols,) bool)."""
    colptr = np.zeros(len(columns) + 1, dtype=np.int64)
    for j, col in enumerate(columns):
        colptr[j + 1] = colptr[j] + len(col)
    rowval = np.asarray([r for col in columns for r in col] or [0], dtype=np.uint32)
    piv = np.empty(max(nrows, 1), dtype=np.int64)
    zero = np.empty(max(len(columns), 1), dtype=np.uint8)
    _L().or_reduce(nrows, len(columns), _ptr(colptr), _ptr(rowval), METHOD[method] & 1,
                   _ptr(piv), _ptr(zero))
    return piv[:nrows], zero[:len(columns)].astype(bool)


def blockprodsum(nrows: int, D, C, E):
    """S = D + C E over GF(2).  D (nrows x ncols), C (nrows x k),
    E (k x ncols) given as (colptr int64, rowval uint32) CSC pairs with rows
    ascending; returns S as (colptr int64 (ncols+1,), rowval uint32)."""
    def arr(m):
        cp = np.ascontiguousarray(m[0], dtype=np.int64)
        rv = np.ascontiguousarray(m[1], dtype=np.uint32)
        return cp, (rv if rv.size else np.zeros(1, dtype=np.uint32))
    (dc, dr), (cc, cr), (ec, er) = arr(D), arr(C), arr(E)
    nc = dc.shape[0] - 1
    scp = np.empty(nc + 1, dtype=np.int64)
    nnz = _L().or_blockprodsum(nrows, nc, _ptr(dc), _ptr(dr), _ptr(cc), _ptr(cr), _ptr(ec), _ptr(er),
                               _ptr(scp), None)
    srv = np.empty(max(nnz, 1), dtype=np.uint32)
    _L().or_blockprodsum(nrows, nc, _ptr(dc), _ptr(dr), _ptr(cc), _ptr(cr), _ptr(ec), _ptr(er),
                         _ptr(scp), _ptr(srv))
    return scp, srv[:nnz]


class Oracle:
    """Steps 1-4 on construction; steps 5-7 via ``simplices(k)``; step 8 via
    ``barcodes``.  ``X`` is (n, d) row-major float64 (points are rows)."""

    def __init__(self, X: np.ndarray, radius: float = np.inf, strict: bool = False, D: np.ndarray = None):
        """X: (n, d) point cloud; or X=None and D: (n, n) distance matrix (upper
        triangle = edge lengths)."""
        if D is not None:
            self.D = np.ascontiguousarray(D, dtype=np.float64)
            if self.D.ndim != 2 or self.D.shape[0] != self.D.shape[1]:
                raise ValueError("D must be (n, n)")
            self.n, self.d = self.D.shape[0], 0
            self.X = np.zeros((self.n, 0))
            self._h = _L().or_new_dm(_ptr(self.D), self.n, float(radius), int(bool(strict)))
        else:
            self.X = np.ascontiguousarray(X, dtype=np.float64)
            if self.X.ndim != 2:
                raise ValueError("X must be (n, d)")
            self.n, self.d = self.X.shape
            self._h = _L().or_new(_ptr(self.X), self.n, self.d, float(radius), int(bool(strict)))
        if not self._h:
            raise MemoryError("oracle allocation failed")
        self.E = _L().or_n_edges(self._h)
        self.nvals = _L().or_n_vals(self._h)
        self._built = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L().or_free(h)
            self._h = None

    def edges(self):
        """(edge_vertices (E,2) u32, edge_filt (E,) u32, edge_len (E,) f64, value_of_rank (nvals,) f64)."""
        ev = np.empty((self.E, 2), dtype=np.uint32)
        ef = np.empty(self.E, dtype=np.uint32)
        el = np.empty(self.E, dtype=np.float64)
        vor = np.empty(self.nvals, dtype=np.float64)
        _L().or_get_edges(self._h, _ptr(ev), _ptr(ef), _ptr(el), _ptr(vor))
        return ev, ef, el, vor

    def edge_pos(self, i: int, j: int) -> int:
        return _L().or_edge_pos(self._h, i, j)

    def simplices(self, k: int):
        """(vertices (N,k+1) u32, filt (N,) u32, boundary rows (N,k+1) u32) for k = 2, 3."""
        if k not in self._built:
            if k == 3 and 2 not in self._built:
                self.simplices(2)
            N = _L().or_build_simplices(self._h, k)
            if N < 0:
                raise ValueError("bad dimension")
            self._built[k] = N
        N = self._built[k]
        v = np.empty((N, k + 1), dtype=np.uint32)
        f = np.empty(N, dtype=np.uint32)
        r = np.empty((N, k + 1), dtype=np.uint32)
        _L().or_get_simplices(self._h, k, _ptr(v), _ptr(f), _ptr(r))
        return v, f, r

    def filt_hist(self, k: int) -> np.ndarray:
        """hist[f] = number of k-simplices (k = 2, 3) with filt f."""
        h = np.empty(self.nvals + 1, dtype=np.uint64)
        _L().or_filt_hist(self._h, k, _ptr(h))
        return h

    def simplices_at_filt(self, k: int, f: int, cap: int = 1 << 20):
        """k-simplices with filt == f in lex order (+ boundary rows for k = 2)."""
        v = np.empty((cap, k + 1), dtype=np.uint32)
        r = np.empty((cap, 3), dtype=np.uint32)
        N = _L().or_simplices_at_filt(self._h, k, f, _ptr(v), _ptr(r), cap)
        if N > cap:
            return self.simplices_at_filt(k, f, cap=int(N))
        return v[:N], (r[:N] if k == 2 else None)

    def barcodes(self, maxdim: int, method: str = "col", keep_zero: bool = False,
                 top: bool = False) -> np.ndarray:
        """Bars (dim, birth filt, death filt or -1 for infinity) sorted, int64 (B, 3).
        Requires the simplices up to dimension maxdim + 1 (built on demand).
        top=True also reports unkilled cycles of dimension maxdim + 1."""
        for k in range(2, maxdim + 2):
            self.simplices(k)
        cap = 1 << 16
        while True:
            out = np.empty((cap, 3), dtype=np.int64)
            nb = _L().or_barcodes(self._h, maxdim, METHOD[method], int(keep_zero), int(top),
                                  _ptr(out), cap)
            if nb <= cap:
                out = out[:nb]
                break
            cap = int(nb)
        order = np.lexsort((out[:, 2], out[:, 1], out[:, 0]))
        return out[order]

    def bars_real(self, bars: np.ndarray):
        """Map integer filtration levels to lengths via value_of_rank (filt 0 -> 0.0)."""
        _, _, _, vor = self.edges()
        table = np.concatenate([[0.0], vor])
        res = []
        for dim, b, d in bars:
            res.append((int(dim), float(table[b]), float("inf") if d < 0 else float(table[d])))
        return res
