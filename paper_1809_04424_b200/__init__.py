"""Python binding of libvrb.so -- the B200 Vietoris-Rips filtration build.

Argument marshalling only: every step of the build runs in the CUDA kernels of
``libvrb.so`` (``csrc/``); PyTorch supplies device memory (through the
allocator hook), streams and ``torch.distributed``.  There is no CPU path: if
the library is missing or no CUDA device is present, calls raise.

Names follow ``include/vrb.h`` (``vrb_build`` -> ``build`` ...).  The paper's
problem statement: a point cloud, the max homology
dimension and an optional radius give ranked edges, ranked simplices and the
boundary matrices in filtration order.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# VRB_LIB_PATH: an alternative build of the same library (tools/variants.py
# experiment builds); the default is the in-tree libvrb.so
LIB_PATH = os.environ.get("VRB_LIB_PATH") or os.path.join(_PKG, "libvrb.so")

VRB_OK, VRB_EINVAL, VRB_ENOMEM, VRB_EOVERFLOW, VRB_ECUDA, VRB_ECOMM, VRB_ENOTSUP = range(7)
STATUS_NAMES = {0: "VRB_OK", 1: "VRB_EINVAL", 2: "VRB_ENOMEM", 3: "VRB_EOVERFLOW", 4: "VRB_ECUDA",
                5: "VRB_ECOMM", 6: "VRB_ENOTSUP"}
VRB_STRICT_RADIUS = 0x1
VRB_DIM_MAJOR = 0x2
VRB_POINTS_ON_DEVICE = 0x4
VRB_SKIP_BOUNDARY = 0x8

# Every symbol include/vrb.h declares (checked by tests/test_abi.py).
EXPORTS = ("vrb_abi_version", "vrb_last_error", "vrb_set_allocator", "vrb_build", "vrb_build_dist",
           "vrb_count", "vrb_simplices", "vrb_rank_values", "vrb_boundary", "vrb_boundary_colptr",
           "vrb_free", "vrb_sortperm_f64", "vrb_partition_bounds", "vrb_compress_d2", "vrb_set_profiling", "vrb_last_stage_ms", "vrb_last_stage_ms_n", "vrb_launch_count", "vrb_last_edge_path", "vrb_h0",
           "vrb_build_dm",
           "vrb_latlon2euc", "vrb_gf2_blockprodsum", "vrb_gf2_csc", "vrb_gf2_free")

STAGES = ("distance", "edge_rank", "csr", "count", "fill", "tie_sort", "exchange", "total", "tet_count",
          "tet_fill")


class VrbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class vrb_opts(ctypes.Structure):
    _fields_ = [("maxdim", ctypes.c_int32), ("radius", ctypes.c_double), ("flags", ctypes.c_uint32)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_void_p, ctypes.c_void_p)
BCAST_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                            ctypes.c_void_p)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p)


class vrb_comm(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("allgather", ALLGATHER_FN),
                ("broadcast", BCAST_FN), ("ctx", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libvrb.so; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    p, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    P = ctypes.POINTER
    L.vrb_abi_version.restype = ctypes.c_int
    L.vrb_abi_version.argtypes = []
    L.vrb_last_error.restype = ctypes.c_char_p
    L.vrb_last_error.argtypes = []
    L.vrb_set_allocator.restype = ctypes.c_int
    L.vrb_set_allocator.argtypes = [ALLOC_FN, FREE_FN, p]
    L.vrb_build.restype = ctypes.c_int
    L.vrb_build.argtypes = [p, i64, i32, P(vrb_opts), p, P(p)]
    L.vrb_build_dist.restype = ctypes.c_int
    L.vrb_build_dist.argtypes = [p, i64, i32, P(vrb_opts), P(vrb_comm), p, P(p)]
    L.vrb_count.restype = ctypes.c_int
    L.vrb_count.argtypes = [p, i32, P(i64), P(i64), P(i64)]
    L.vrb_simplices.restype = ctypes.c_int
    L.vrb_simplices.argtypes = [p, i32, P(p), P(p)]
    L.vrb_rank_values.restype = ctypes.c_int
    L.vrb_rank_values.argtypes = [p, P(p), P(i64)]
    L.vrb_boundary.restype = ctypes.c_int
    L.vrb_boundary.argtypes = [p, i32, P(i64), P(i64), P(p)]
    L.vrb_boundary_colptr.restype = ctypes.c_int
    L.vrb_boundary_colptr.argtypes = [p, i32, p, p]
    L.vrb_free.restype = ctypes.c_int
    L.vrb_free.argtypes = [p]
    L.vrb_sortperm_f64.restype = ctypes.c_int
    L.vrb_sortperm_f64.argtypes = [p, i64, p, p, p]
    L.vrb_set_profiling.restype = ctypes.c_int
    L.vrb_set_profiling.argtypes = [i32]
    L.vrb_last_stage_ms.restype = ctypes.c_int
    L.vrb_last_stage_ms.argtypes = [P(ctypes.c_double)]
    L.vrb_last_stage_ms_n.restype = ctypes.c_int
    L.vrb_last_stage_ms_n.argtypes = [P(ctypes.c_double), ctypes.c_int32]
    L.vrb_launch_count.restype = ctypes.c_ulonglong
    L.vrb_launch_count.argtypes = []
    L.vrb_last_edge_path.restype = ctypes.c_int32
    L.vrb_last_edge_path.argtypes = []
    L.vrb_build_dm.restype = ctypes.c_int
    L.vrb_build_dm.argtypes = [p, i64, P(vrb_opts), p, P(p)]
    L.vrb_latlon2euc.restype = ctypes.c_int
    L.vrb_latlon2euc.argtypes = [p, i64, p, p]
    L.vrb_gf2_blockprodsum.restype = ctypes.c_int
    L.vrb_gf2_blockprodsum.argtypes = [i64, i64, i64, p, p, p, p, p, p, p, P(p)]
    L.vrb_gf2_csc.restype = ctypes.c_int
    L.vrb_gf2_csc.argtypes = [p, P(i64), P(p), P(p)]
    L.vrb_gf2_free.restype = ctypes.c_int
    L.vrb_gf2_free.argtypes = [p]
    L.vrb_partition_bounds.restype = ctypes.c_int
    L.vrb_partition_bounds.argtypes = [p, p, i64, i32, p]
    L.vrb_compress_d2.restype = ctypes.c_int
    L.vrb_compress_d2.argtypes = [p, p, P(i64), P(i64), P(p), P(p), P(p)]
    L.vrb_h0.restype = ctypes.c_int
    L.vrb_h0.argtypes = [p, p, P(p), P(p), P(i64), P(i64)]
    _lib = L
    return L


def _check(st: int):
    if st != VRB_OK:
        raise VrbError(st, lib().vrb_last_error().decode(errors="replace"))


def abi_version() -> int:
    return lib().vrb_abi_version()


# ---------------------------------------------------------------------------
# allocator hook -> PyTorch caching allocator
# ---------------------------------------------------------------------------
_hooks = None
_hooks_ever = []   # every hook pair ever installed: a handle frees through the hook
                   # that allocated it, so its C callback must outlive the switch


def use_torch_allocator(enable: bool = True):
    """Route the library's device allocations through torch's caching allocator."""
    global _hooks
    import torch

    if not enable:
        _check(lib().vrb_set_allocator(ALLOC_FN(), FREE_FN(), None))
        _hooks = None
        return

    def _alloc(nbytes, dev, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), int(dev), int(stream or 0))
        except Exception:   # reported as VRB_ENOMEM by the library
            return None

    def _free(ptr, nbytes, dev, stream, ctx):
        try:
            torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:
            pass

    hooks = (ALLOC_FN(_alloc), FREE_FN(_free))
    _check(lib().vrb_set_allocator(hooks[0], hooks[1], None))
    _hooks = hooks
    _hooks_ever.append(hooks)


def set_profiling(enable: bool):
    _check(lib().vrb_set_profiling(1 if enable else 0))


def launch_count() -> int:
    """Kernels launched by libvrb.so so far in this process."""
    return int(lib().vrb_launch_count())


def last_edge_path() -> str:
    """S3 path of the last build on this thread: "bucket", "radix" or "none"."""
    return {1: "bucket", 0: "radix"}.get(int(lib().vrb_last_edge_path()), "none")


def last_stage_ms() -> dict:
    arr = (ctypes.c_double * len(STAGES))()
    _check(lib().vrb_last_stage_ms_n(arr, len(STAGES)))
    return {k: float(v) for k, v in zip(STAGES, arr)}


# ---------------------------------------------------------------------------
# zero-copy device views of handle-owned arrays
# ---------------------------------------------------------------------------
class _CAI:
    def __init__(self, ptr, shape, typestr, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}
        self._owner = owner


def _view(ptr, shape, typestr, owner, device):
    import torch

    n = int(np.prod(shape)) if len(shape) else 1
    if n == 0 or not ptr:
        dt = {"<i4": torch.int32, "<f8": torch.float64, "<i8": torch.int64}[typestr]
        return torch.empty(shape, dtype=dt, device=device)
    return torch.as_tensor(_CAI(ptr, shape, typestr, owner), device=device)


class VRResult:
    """A built filtration (owns the vrb handle).  Arrays are zero-copy CUDA
    tensors in filtration order; u32 arrays are exposed as int32 tensors
    holding the u32 bit patterns (use ``.view(torch.uint32)`` or ``u64()``)."""

    def __init__(self, handle: int, device):
        self._h = ctypes.c_void_p(handle)
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().vrb_free(h)
            finally:
                self._h = None

    def free(self):
        self.__del__()

    # counts
    def count(self, dim: int):
        g, o, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().vrb_count(self._h, dim, ctypes.byref(g), ctypes.byref(o), ctypes.byref(n)))
        return g.value, o.value, n.value

    @property
    def num_edges(self) -> int:
        return self.count(1)[0]

    def simplices(self, dim: int):
        """(vertices (N, dim+1) int32[u32], filt (N,) int32[u32]) of this handle's slice."""
        v, f = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().vrb_simplices(self._h, dim, ctypes.byref(v), ctypes.byref(f)))
        n = self.count(dim)[2]
        return (_view(v.value, (n, dim + 1), "<i4", self, self.device),
                _view(f.value, (n,), "<i4", self, self.device))

    def h0(self, stream=None):
        """Dimension-0 persistence (vrb_h0): (forest_pos, death_filt,
        n_essential).  forest_pos: ascending positions of the minimum-spanning-forest
        edges (the D_1 pivot columns); death_filt: their filt, so the finite bars are
        [0, death_filt[i]); n_essential: number of [0, inf) bars (components)."""
        pos, dth = ctypes.c_void_p(), ctypes.c_void_p()
        nf, ne = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().vrb_h0(self._h, _stream_ptr(stream), ctypes.byref(pos), ctypes.byref(dth),
                            ctypes.byref(nf), ctypes.byref(ne)))
        return (_view(pos.value, (nf.value,), "<i4", self, self.device),
                _view(dth.value, (nf.value,), "<i4", self, self.device), ne.value)

    def compress_d2(self, stream=None):
        """vrb_compress_d2 ("clear and compress"): D_2
        without the rows of the H0 forest edges (the D_1 pivot columns).
        Returns (colptr (ncols+1,) int64, rowval (nnz,) int32[u32] compressed
        rows, rowmap (nrows,) int32[u32] compressed row -> edge position)."""
        nr, nz = ctypes.c_int64(), ctypes.c_int64()
        cp, rv, rm = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().vrb_compress_d2(self._h, _stream_ptr(stream), ctypes.byref(nr), ctypes.byref(nz),
                                     ctypes.byref(cp), ctypes.byref(rv), ctypes.byref(rm)))
        nc = self.count(2)[2]
        return (_view(cp.value, (nc + 1,), "<i8", self, self.device),
                _view(rv.value, (nz.value,), "<i4", self, self.device),
                _view(rm.value, (nr.value,), "<i4", self, self.device))

    def rank_values(self):
        p, nv = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().vrb_rank_values(self._h, ctypes.byref(p), ctypes.byref(nv)))
        return _view(p.value, (nv.value,), "<f8", self, self.device)

    def boundary(self, k: int):
        """D_k row values (ncols, k+1) int32[u32]: positions of the faces, ascending."""
        nr, nc, p = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_void_p()
        _check(lib().vrb_boundary(self._h, k, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(p)))
        return _view(p.value, (nc.value, k + 1), "<i4", self, self.device)

    def boundary_colptr(self, k: int, stream=None):
        import torch

        nc = self.count(k)[2]
        out = torch.empty(nc + 1, dtype=torch.int64, device=self.device)
        _check(lib().vrb_boundary_colptr(self._h, k, ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out


def u64(t):
    """int32 tensor holding u32 bit patterns -> int64 values."""
    import torch

    return t.to(torch.int64) & 0xFFFFFFFF


def _stream_ptr(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(int(s.cuda_stream))


def _prepare_points(points, device, rowsare: str = "points"):
    """Returns (pointer, n, d, flags, keepalive).  rowsare="points": the array
    is (n, d), one point per row; rowsare="dimensions" (Eirene's keyword,
    P:385-386): it is (d, n), one point per column, passed to the
    library as is with VRB_DIM_MAJOR (the transpose runs on the device)."""
    import torch

    if rowsare not in ("points", "dimensions"):
        raise ValueError('rowsare must be "points" or "dimensions"')
    dm = rowsare == "dimensions"
    flags = VRB_DIM_MAJOR if dm else 0
    if isinstance(points, torch.Tensor):
        t = points.detach()
        if t.dtype != torch.float64:
            raise TypeError("points must be float64")
        if t.ndim != 2:
            raise ValueError("points must be 2-D")
        t = t.contiguous()
        n, d = (t.shape[1], t.shape[0]) if dm else (t.shape[0], t.shape[1])
        if t.is_cuda:
            flags |= VRB_POINTS_ON_DEVICE
        return t.data_ptr(), n, d, flags, t
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("points must be 2-D")
    n, d = (a.shape[1], a.shape[0]) if dm else (a.shape[0], a.shape[1])
    return a.ctypes.data, n, d, flags, a


def build(points, maxdim: int = 1, radius: float = math.inf, strict: bool = False,
          skip_boundary: bool = False, stream=None, rowsare: str = "points") -> VRResult:
    """vrb_build: points (n, d) float64, or (d, n) with rowsare="dimensions"
    (numpy / CPU tensor -> copied H2D inside the call; CUDA tensor -> used in
    place on its device)."""
    import torch

    ptr, n, d, flags, keep = _prepare_points(points, None, rowsare)
    if flags & VRB_POINTS_ON_DEVICE:
        device = keep.device
    else:
        device = torch.device("cuda", torch.cuda.current_device())
    if strict:
        flags |= VRB_STRICT_RADIUS
    if skip_boundary:
        flags |= VRB_SKIP_BOUNDARY
    opts = vrb_opts(int(maxdim), float(radius), flags)
    h = ctypes.c_void_p()
    with torch.cuda.device(device):
        _check(lib().vrb_build(ctypes.c_void_p(ptr), n, max(d, 1), ctypes.byref(opts), _stream_ptr(stream),
                               ctypes.byref(h)))
    del keep
    return VRResult(h.value, device)


def build_dm(D, maxdim: int = 1, radius: float = math.inf, strict: bool = False,
             skip_boundary: bool = False, stream=None) -> VRResult:
    """vrb_build_dm: D (n, n) float64 symmetric distance matrix (numpy / CPU
    tensor -> copied H2D inside the call; CUDA tensor -> used in place)."""
    import torch

    ptr, n, n2, flags, keep = _prepare_points(D, None)
    if n != n2:
        raise ValueError("D must be square (n, n)")
    device = keep.device if (flags & VRB_POINTS_ON_DEVICE) else torch.device("cuda", torch.cuda.current_device())
    if strict:
        flags |= VRB_STRICT_RADIUS
    if skip_boundary:
        flags |= VRB_SKIP_BOUNDARY
    opts = vrb_opts(int(maxdim), float(radius), flags)
    h = ctypes.c_void_p()
    with torch.cuda.device(device):
        _check(lib().vrb_build_dm(ctypes.c_void_p(ptr), n, ctypes.byref(opts), _stream_ptr(stream), ctypes.byref(h)))
    del keep
    return VRResult(h.value, device)


def latlon2euc(latlon, stream=None):
    """vrb_latlon2euc: (n, 2) float64 CUDA tensor of (lat, lon) degrees -> (n, 3)
    unit-sphere coordinates."""
    import torch

    if not (isinstance(latlon, torch.Tensor) and latlon.is_cuda and latlon.dtype == torch.float64):
        raise TypeError("latlon must be a float64 CUDA tensor")
    a = latlon.detach().contiguous().reshape(-1, 2)
    out = torch.empty((a.shape[0], 3), dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        _check(lib().vrb_latlon2euc(ctypes.c_void_p(a.data_ptr()), a.shape[0], ctypes.c_void_p(out.data_ptr()),
                                    _stream_ptr(stream)))
    return out


class Gf2Matrix:
    """A GF(2) CSC matrix owned by the library (vrb_gf2_blockprodsum result):
    ``colptr`` (ncols+1,) int64 and ``rowval`` (nnz,) int32[u32] CUDA tensors."""

    def __init__(self, handle: int, ncols: int, device):
        self._h = ctypes.c_void_p(handle)
        nnz, cp, rv = ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().vrb_gf2_csc(self._h, ctypes.byref(nnz), ctypes.byref(cp), ctypes.byref(rv)))
        self.nnz = nnz.value
        self.colptr = _view(cp.value, (ncols + 1,), "<i8", self, device)
        self.rowval = _view(rv.value, (nnz.value,), "<i4", self, device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().vrb_gf2_free(h)
            finally:
                self._h = None


def gf2_blockprodsum(nrows: int, D, C, E, stream=None) -> Gf2Matrix:
    """vrb_gf2_blockprodsum: S = D + C E over GF(2).  D, C, E are
    (colptr, rowval) pairs of CUDA tensors (int64 colptr, int32/uint32 rows)."""
    import torch

    def prep(m):
        cp, rv = m
        if not (cp.is_cuda and rv.is_cuda):
            raise TypeError("CSC arrays must be CUDA tensors")
        cp = cp.to(torch.int64).contiguous()
        rv = rv.contiguous()
        if rv.dtype not in (torch.int32, torch.uint32):
            raise TypeError("row indices must be 32-bit")
        return cp, rv

    (dc, dr), (cc, cr), (ec, er) = prep(D), prep(C), prep(E)
    ncols, k = dc.numel() - 1, cc.numel() - 1
    h = ctypes.c_void_p()
    with torch.cuda.device(dc.device):
        _check(lib().vrb_gf2_blockprodsum(int(nrows), ncols, k, *(ctypes.c_void_p(t.data_ptr()) for t in
                                                                  (dc, dr, cc, cr, ec, er)),
                                          _stream_ptr(stream), ctypes.byref(h)))
    return Gf2Matrix(h.value, ncols, dc.device)


def allgather_bytes(src, dst, group=None):
    """dst (world * nbytes, uint8) <- all-gather of src (nbytes, uint8) over the
    process group, on the current stream: NCCL on the device tensors directly,
    other backends (gloo) through host memory."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl" or src.device.type == "cpu":
        dist.all_gather_into_tensor(dst, src, group=group)
        return
    hs = src.cpu()
    hd = torch.empty(dst.numel(), dtype=dst.dtype)
    dist.all_gather_into_tensor(hd, hs, group=group)
    dst.copy_(hd)


def broadcast_bytes(buf, root: int, group=None):
    """buf (nbytes, uint8) <- rank root's buf, on the current stream (NCCL on
    device, other backends through host memory)."""
    import torch.distributed as dist

    src = dist.get_global_rank(group, root) if group is not None else root
    if dist.get_backend(group) == "nccl" or buf.device.type == "cpu":
        dist.broadcast(buf, src, group=group)
        return
    h = buf.cpu()
    dist.broadcast(h, src, group=group)
    buf.copy_(h)


def _torch_stream(ptr, device):
    """torch view of the library's stream.  0 is the legacy default stream:
    torch.cuda.ExternalStream(0) would hand out a fresh pool stream instead,
    so stream 0 maps to torch's default stream (the legacy one)."""
    import torch

    return torch.cuda.ExternalStream(int(ptr), device=device) if ptr else torch.cuda.default_stream(device)


def _comm_callbacks(device, world, group):
    """The vrb_comm callbacks over torch.distributed.  Each one runs its
    collective with the library's build stream as torch's current stream, so
    it is ordered after the work the library enqueued and the library's later
    work is ordered after it (NCCL: no host synchronisation)."""
    import torch

    def _allgather(send, recv, nbytes, stream_, ctx):
        try:
            with torch.cuda.stream(_torch_stream(stream_, device)):
                src = torch.as_tensor(_CAI(send, (nbytes,), "|u1", None), device=device)
                dst = torch.as_tensor(_CAI(recv, (nbytes * world,), "|u1", None), device=device)
                allgather_bytes(src, dst, group)
            return 0
        except Exception as e:   # reported as VRB_ECOMM
            print("vrb allgather failed:", e)
            return 1

    def _broadcast(buf, nbytes, root, stream_, ctx):
        try:
            with torch.cuda.stream(_torch_stream(stream_, device)):
                t = torch.as_tensor(_CAI(buf, (nbytes,), "|u1", None), device=device)
                broadcast_bytes(t, root, group)
            return 0
        except Exception as e:   # reported as VRB_ECOMM
            print("vrb broadcast failed:", e)
            return 1

    return ALLGATHER_FN(_allgather), BCAST_FN(_broadcast)


def build_dist(points, maxdim: int = 1, radius: float = math.inf, strict: bool = False,
               skip_boundary: bool = False, group=None, stream=None, rowsare: str = "points", n: int = None,
               d: int = None) -> VRResult:
    """vrb_build_dist: one process per GPU.  Rank 0 passes the points (as
    build()); the other ranks may pass None with n and d (the library
    broadcasts rank 0's points).  The collectives the library asks for run
    over torch.distributed on the build stream."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if points is None:
        if n is None or d is None:
            raise ValueError("ranks without points must pass n and d")
        ptr, flags, keep = 0, 0, None
        device = torch.device("cuda", torch.cuda.current_device())
    else:
        ptr, n, d, flags, keep = _prepare_points(points, None, rowsare)
        device = keep.device if (flags & VRB_POINTS_ON_DEVICE) else torch.device("cuda", torch.cuda.current_device())
    if strict:
        flags |= VRB_STRICT_RADIUS
    if skip_boundary:
        flags |= VRB_SKIP_BOUNDARY
    ag, bc = _comm_callbacks(device, world, group)
    comm = vrb_comm(rank, world, ag, bc, None)
    opts = vrb_opts(int(maxdim), float(radius), flags)
    h = ctypes.c_void_p()
    with torch.cuda.device(device):
        _check(lib().vrb_build_dist(ctypes.c_void_p(ptr), n, max(d, 1), ctypes.byref(opts), ctypes.byref(comm),
                                    _stream_ptr(stream), ctypes.byref(h)))
    del keep
    return VRResult(h.value, device)


def partition_bounds(prefix, efilt, world: int):
    """vrb_partition_bounds on host arrays (the owner-edge split rule of
    build_dist): prefix (E + 1,) uint64 work prefix, efilt (E,) uint32 levels
    -> (world + 1,) int64 first owner edge of each rank."""
    pre = np.ascontiguousarray(prefix, dtype=np.uint64)
    ef = np.ascontiguousarray(efilt, dtype=np.uint32)
    if pre.shape[0] != ef.shape[0] + 1:
        raise ValueError("prefix must have E + 1 entries")
    out = np.zeros(world + 1, dtype=np.int64)
    _check(lib().vrb_partition_bounds(pre.ctypes.data, ef.ctypes.data if ef.size else None, ef.shape[0], int(world),
                                      out.ctypes.data))
    return out


def sortperm_f64(keys):
    """vrb_sortperm_f64: (0-based stable permutation int64, dense ranks int32[u32])."""
    import torch

    if not (isinstance(keys, torch.Tensor) and keys.is_cuda and keys.dtype == torch.float64):
        raise TypeError("keys must be a CUDA float64 tensor")
    k = keys.contiguous()
    perm = torch.empty(k.numel(), dtype=torch.int64, device=k.device)
    dense = torch.empty(k.numel(), dtype=torch.int32, device=k.device)
    with torch.cuda.device(k.device):
        _check(lib().vrb_sortperm_f64(ctypes.c_void_p(k.data_ptr()), k.numel(), ctypes.c_void_p(perm.data_ptr()),
                                      ctypes.c_void_p(dense.data_ptr()), _stream_ptr(None)))
    return perm, dense
