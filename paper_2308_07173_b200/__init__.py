"""paper_2308_07173_b200 -- thin Python binding of libgicp_b200.so (include/gicp.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels. torch provides device memory and the current stream. There is no CPU
fallback: if the shared library is missing this import fails loudly.

Names follow the C ABI: build_index, knn, knn_self, covariances, knn_cov_self,
linearize, align (§III-C1, l.377-435).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# GICP_LIB_VARIANT selects an alternative build of the SAME library (tools/ only,
# for A/B timing of compile options); the default is the in-tree build.
LIB_PATH = os.environ.get("GICP_LIB_VARIANT") or os.path.join(_HERE, "libgicp_b200.so")

OK, EINVAL, EK, ERANGE, ENOMEM, ECUDA, EDEGENERATE = 0, -1, -2, -3, -4, -5, -6
LIN_REUSE_CORR, LIN_ERROR_ONLY = 1, 2
KMAX = 32

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                      "There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)


class IndexInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_cells", ctypes.c_int64), ("cell_size", ctypes.c_float),
                ("origin", ctypes.c_float * 3), ("dims", ctypes.c_int32 * 3), ("device_bytes", ctypes.c_int64),
                ("n_levels", ctypes.c_int32)]


class AlignParams(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int), ("lm", ctypes.c_int), ("rot_eps", ctypes.c_double),
                ("trans_eps", ctypes.c_double), ("max_corr_dist", ctypes.c_float)]


class AlignResult(ctypes.Structure):
    _fields_ = [("T", ctypes.c_double * 16), ("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("error", ctypes.c_double), ("inliers", ctypes.c_int64)]


_P = ctypes.c_void_p
_i64, _i32, _f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_float
_lib.gicp_last_error.restype = ctypes.c_char_p
_lib.gicp_version.restype = _i32
_lib.gicp_build_index.argtypes = [_P, _i64, _f32, _P, ctypes.POINTER(_P)]
_lib.gicp_index_free.argtypes = [_P]
_lib.gicp_index_free.restype = None
_lib.gicp_get_index_info.argtypes = [_P, ctypes.POINTER(IndexInfo)]
_lib.gicp_index_attach_cov.argtypes = [_P, _P, _P]
_lib.gicp_knn.argtypes = [_P, _P, _i64, _i32, _P, _P, _P]
_lib.gicp_knn_self.argtypes = [_P, _i32, _P, _P, _P]
_lib.gicp_covariances.argtypes = [_P, _i64, _P, _i64, _i32, _f32, _P, _P]
_lib.gicp_knn_cov_self.argtypes = [_P, _i32, _f32, _P, _P, _P, _P]


class CovParams(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int), ("sigma", ctypes.c_float), ("alpha", ctypes.c_float),
                ("c", ctypes.c_float), ("degree", ctypes.c_int), ("origin", ctypes.c_float * 3),
                ("reg", ctypes.c_int), ("eps", ctypes.c_float)]


_lib.gicp_index_attach_voxels.argtypes = [_P, _P, _P]
_lib.gicp_linearize_vgicp.argtypes = [_P, _P, _i64, _P, _P, _P, _i32, _i32, _P, _P, _P]
_lib.gicp_align_vgicp.argtypes = [_P, _P, _i64, _P, _i32, _P, ctypes.POINTER(AlignParams), ctypes.POINTER(AlignResult),
                                  _P]
_lib.gicp_ground_filter.argtypes = [_P, _i64, _f32, _i32, _P, _P, _P]
_lib.gicp_submap_build.argtypes = [_P, _i64, _i32, ctypes.POINTER(_P), _P]
_lib.gicp_submap_query.argtypes = [_P, _i32, _i32, _P, ctypes.POINTER(ctypes.c_int64), _P]
_lib.gicp_submap_free.argtypes = [_P]
_lib.gicp_submap_free.restype = None
_lib.gicp_align_timing.argtypes = [_i32, _P, _P, _P]
_lib.gicp_cluster.argtypes = [_P, _i64, _f32, _i32, _P, ctypes.POINTER(ctypes.c_int64), _P]
_lib.gicp_covariances_kd.argtypes = [_P, _i64, _P, _P, _i64, _i32, ctypes.POINTER(CovParams), _P, _P]
KERNELS = {"uniform": 0, "rbf": 1, "gaussian": 2, "polynomial": 3, "hi": 4, "laplacian": 5}
REGS = {"plane": 0, "min_eig": 1, "normalized_min_eig": 2}
_lib.gicp_linearize.argtypes = [_P, _P, _i64, _P, _P, _P, _P, _f32, _i32, _P, _P, _P]
_lib.gicp_align.argtypes = [_P, _P, _i64, _P, _P, _P, ctypes.POINTER(AlignParams), ctypes.POINTER(AlignResult),
                            _P]
_lib.gicp_linearize_batched.argtypes = [_P, _P, _P, _i32, _P, _P, _P, _P, _f32, _i32, _P, _P, _P]
_lib.gicp_align_batched.argtypes = [_P, _P, _P, _i32, _P, _P, _P, ctypes.POINTER(AlignParams), _P, _P]
REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                             ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_void_p)
_lib.gicp_align_batched_ex.argtypes = [_P, _P, _P, _i32, _P, _i32, _P, _P, _P, ctypes.POINTER(AlignParams), _P,
                                       REDUCE_FN, _P, _P]
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)
_lib.gicp_align_batched_sharded.argtypes = [_P, _P, _P, _i32, _P, _i32, _i32, _P, _P, _P, ctypes.POINTER(AlignParams),
                                            _P, _P, ALLREDUCE_FN, _P, _P]
_lib.gicp_combine_chunks.argtypes = [_P, _i32, _i32, _i32, _P, _P]
_lib.gicp_knn_query_order.argtypes = [_P, _P, _i64, _P, _P]
_lib.gicp_knn_subset.argtypes = [_P, _P, _i64, _P, _i64, _i32, _P, _P, _P]
_lib.gicp_index_export.argtypes = [_P, _P, _P, _P, ctypes.POINTER(ctypes.c_int)]
_lib.gicp_index_import.argtypes = [_P, _P, _P, ctypes.POINTER(_P)]
INDEX_HEADER_BYTES, INDEX_MAX_BUFFERS = 4096, 16

EXPORTS = ["gicp_last_error", "gicp_version", "gicp_build_index", "gicp_index_free", "gicp_get_index_info",
           "gicp_index_attach_cov",
           "gicp_knn", "gicp_knn_self", "gicp_covariances", "gicp_knn_cov_self", "gicp_linearize", "gicp_align",
           "gicp_linearize_batched", "gicp_align_batched", "gicp_align_batched_ex", "gicp_align_batched_sharded",
           "gicp_combine_chunks", "gicp_knn_query_order", "gicp_knn_subset", "gicp_index_export",
           "gicp_index_import", "gicp_covariances_kd",
           "gicp_index_attach_voxels", "gicp_linearize_vgicp", "gicp_align_vgicp", "gicp_ground_filter",
           "gicp_cluster", "gicp_submap_build", "gicp_submap_query", "gicp_submap_free", "gicp_align_timing"]


class GicpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int):
    if rc != OK:
        raise GicpError(rc, _lib.gicp_last_error().decode())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _pts(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dtype != torch.float32 or t.dim() != 2 or t.shape[1] != 3:
        raise ValueError(f"{name} must be float32 [n, 3]")
    return t.contiguous()


class Index:
    """An index owned by the library (gicp_build_index). Keeps a device copy."""

    def __init__(self, handle: ctypes.c_void_p, device: torch.device):
        self._h = handle
        self.device = device
        info = IndexInfo()
        _check(_lib.gicp_get_index_info(self._h, ctypes.byref(info)))
        self.n = int(info.n)
        self.n_cells = int(info.n_cells)
        self.cell_size = float(info.cell_size)
        self.origin = tuple(info.origin)
        self.dims = tuple(info.dims)
        self.device_bytes = int(info.device_bytes)
        self.n_levels = int(info.n_levels)

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            _lib.gicp_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def build_index(xyz: torch.Tensor, cell_size: float = 0.0) -> Index:
    xyz = _pts(xyz, "xyz")
    h = ctypes.c_void_p()
    _check(_lib.gicp_build_index(_dptr(xyz), xyz.shape[0], float(cell_size), _stream(), ctypes.byref(h)))
    return Index(h, xyz.device)


def attach_cov(index: Index, cov: torch.Tensor) -> None:
    """gicp_index_attach_cov: keep a sorted-order copy of `cov` ([n, 6], original
    order) in the index; linearize/align use it when passed this same tensor."""
    if cov.dtype != torch.float32 or cov.shape != (index.n, 6) or not cov.is_contiguous():
        raise ValueError("cov must be a contiguous float32 [n, 6] tensor")
    _check(_lib.gicp_index_attach_cov(index.handle, _dptr(cov), _stream()))
    index._attached = cov  # keep the tensor alive while attached


def knn(index: Index, q: torch.Tensor, k: int, out=None):
    q = _pts(q, "q")
    m = q.shape[0]
    nbr, d2 = out if out is not None else (torch.empty((m, k), dtype=torch.int32, device=q.device),
                                           torch.empty((m, k), dtype=torch.float32, device=q.device))
    _check(_lib.gicp_knn(index.handle, _dptr(q), m, k, _dptr(nbr), _dptr(d2), _stream()))
    return nbr, d2


def knn_self(index: Index, k: int, out=None):
    nbr, d2 = out if out is not None else (torch.empty((index.n, k), dtype=torch.int32, device=index.device),
                                           torch.empty((index.n, k), dtype=torch.float32, device=index.device))
    _check(_lib.gicp_knn_self(index.handle, k, _dptr(nbr), _dptr(d2), _stream()))
    return nbr, d2


def covariances(xyz: torch.Tensor, nbr: torch.Tensor, eps: float = 1e-3, out=None):
    xyz = _pts(xyz, "xyz")
    if nbr.dtype != torch.int32 or nbr.dim() != 2:
        raise ValueError("nbr must be int32 [m, k]")
    nbr = nbr.contiguous()
    m, k = nbr.shape
    cov = out if out is not None else torch.empty((m, 6), dtype=torch.float32, device=xyz.device)
    _check(_lib.gicp_covariances(_dptr(xyz), xyz.shape[0], _dptr(nbr), m, k, float(eps), _dptr(cov), _stream()))
    return cov


def covariances_kd(xyz: torch.Tensor, nbr: torch.Tensor, kernel="laplacian", sigma=1.0, q=None, alpha=1.0, c=0.0,
                   degree=2, origin=(0.0, 0.0, 0.0), reg="plane", eps: float = 1e-3, out=None):
    """Kernel-descriptor weighted covariances (gicp_covariances_kd, Table I).
    q: queries [m,3] (default: row i's query is xyz[i]). Returns cov float32 [m,6]."""
    xyz = _pts(xyz, "xyz")
    if nbr.dtype != torch.int32 or nbr.dim() != 2:
        raise ValueError("nbr must be int32 [m, k]")
    nbr = nbr.contiguous()
    m, k = nbr.shape
    qq = None if q is None else _pts(q, "q")
    p = CovParams(KERNELS[kernel] if isinstance(kernel, str) else int(kernel), float(sigma), float(alpha), float(c),
                  int(degree), (ctypes.c_float * 3)(*[float(v) for v in origin]),
                  REGS[reg] if isinstance(reg, str) else int(reg), float(eps))
    cov = out if out is not None else torch.empty((m, 6), dtype=torch.float32, device=xyz.device)
    _check(_lib.gicp_covariances_kd(_dptr(xyz), xyz.shape[0], None if qq is None else _dptr(qq), _dptr(nbr), m, k,
                                    ctypes.byref(p), _dptr(cov), _stream()))
    return cov


def knn_cov_self(index: Index, k: int, eps: float = 1e-3, with_nbr: bool = True, out=None):
    n = index.n
    if out is not None:
        nbr, d2, cov = out
    else:
        cov = torch.empty((n, 6), dtype=torch.float32, device=index.device)
        nbr = torch.empty((n, k), dtype=torch.int32, device=index.device) if with_nbr else None
        d2 = torch.empty((n, k), dtype=torch.float32, device=index.device) if with_nbr else None
    _check(_lib.gicp_knn_cov_self(index.handle, k, float(eps), _dptr(nbr), _dptr(d2), _dptr(cov), _stream()))
    return nbr, d2, cov


def _T(T) -> np.ndarray:
    T = np.ascontiguousarray(np.asarray(T, dtype=np.float64).reshape(4, 4))
    return T


def linearize(src: torch.Tensor, src_cov: torch.Tensor, tgt: Index, tgt_cov: torch.Tensor, T, max_corr_dist=1.0,
              corr: torch.Tensor | None = None, reuse_corr: bool = False, error_only: bool = False, out=None,
              pivot=None):
    """Returns (out29 float64 device tensor [29], corr int32 device tensor [ns]).
    pivot: rotation pivot (3,) of the perturbation, default the origin."""
    src = _pts(src, "src")
    ns = src.shape[0]
    Th = _T(T)
    out29 = out if out is not None else torch.empty(29, dtype=torch.float64, device=src.device)
    if corr is None:
        if reuse_corr:
            raise ValueError("reuse_corr needs corr")
        corr = torch.empty(ns, dtype=torch.int32, device=src.device)
    flags = (LIN_REUSE_CORR if reuse_corr else 0) | (LIN_ERROR_ONLY if error_only else 0)
    piv = None if pivot is None else np.ascontiguousarray(np.asarray(pivot, dtype=np.float64).reshape(3))
    _check(_lib.gicp_linearize(_dptr(src), _dptr(src_cov.contiguous()), ns, tgt.handle, _dptr(tgt_cov.contiguous()),
                               Th.ctypes.data_as(_P), None if piv is None else piv.ctypes.data_as(_P),
                               float(max_corr_dist), flags, _dptr(out29), _dptr(corr), _stream()))
    return out29, corr


@dataclass
class AlignInfo:
    iterations: int
    converged: bool
    error: float
    inliers: int


def align(src: torch.Tensor, src_cov: torch.Tensor, tgt: Index, tgt_cov: torch.Tensor, T0, max_iter=64, lm=True,
          rot_eps=1e-6, trans_eps=1e-5, max_corr_dist=1.0):
    src = _pts(src, "src")
    T0h = _T(T0)
    p = AlignParams(int(max_iter), int(bool(lm)), float(rot_eps), float(trans_eps), float(max_corr_dist))
    r = AlignResult()
    _check(_lib.gicp_align(_dptr(src), _dptr(src_cov.contiguous()), src.shape[0], tgt.handle,
                           _dptr(tgt_cov.contiguous()), T0h.ctypes.data_as(_P), ctypes.byref(p), ctypes.byref(r),
                           _stream()))
    T = np.array(r.T[:], dtype=np.float64).reshape(4, 4)
    return T, AlignInfo(int(r.iterations), bool(r.converged), float(r.error), int(r.inliers))


def _offsets(offsets, total, allow_empty=False):
    o = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64).reshape(-1))
    if o.size < (1 if allow_empty else 2) or o[0] != 0 or o[-1] != total:
        raise ValueError("offsets must be [0, ..., n_points] with B+1 entries")
    return o


def linearize_batched(src: torch.Tensor, src_cov: torch.Tensor, offsets, tgt: Index, tgt_cov: torch.Tensor, Ts,
                      max_corr_dist=1.0, pivots=None, corr: torch.Tensor | None = None, reuse_corr: bool = False,
                      error_only: bool = False, out=None):
    """B registrations in one launch: registration b owns src[offsets[b]:offsets[b+1]].
    Returns (out float64 device [B, 29], corr int32 device [n])."""
    src = _pts(src, "src")
    ns = src.shape[0]
    o = _offsets(offsets, ns)
    B = o.size - 1
    Th = np.ascontiguousarray(np.asarray(Ts, dtype=np.float64).reshape(B, 16))
    piv = None if pivots is None else np.ascontiguousarray(np.asarray(pivots, dtype=np.float64).reshape(B, 3))
    out = out if out is not None else torch.empty((B, 29), dtype=torch.float64, device=src.device)
    if corr is None:
        if reuse_corr:
            raise ValueError("reuse_corr needs corr")
        corr = torch.empty(ns, dtype=torch.int32, device=src.device)
    flags = (LIN_REUSE_CORR if reuse_corr else 0) | (LIN_ERROR_ONLY if error_only else 0)
    _check(_lib.gicp_linearize_batched(_dptr(src), _dptr(src_cov.contiguous()), o.ctypes.data_as(_P), B, tgt.handle,
                                       _dptr(tgt_cov.contiguous()), Th.ctypes.data_as(_P),
                                       None if piv is None else piv.ctypes.data_as(_P), float(max_corr_dist), flags,
                                       _dptr(out), _dptr(corr), _stream()))
    return out, corr


def align_batched(src: torch.Tensor, src_cov: torch.Tensor, offsets, tgt: Index, tgt_cov: torch.Tensor, T0s,
                  max_iter=64, lm=True, rot_eps=1e-6, trans_eps=1e-5, max_corr_dist=1.0, allow_degenerate=False):
    """Lockstep LM for B registrations. Returns (T [B,4,4] float64 numpy, [AlignInfo] * B).
    With allow_degenerate, registrations with < 6 correspondences are reported
    (inliers < 6) instead of raising."""
    src = _pts(src, "src")
    o = _offsets(offsets, src.shape[0])
    B = o.size - 1
    T0h = np.ascontiguousarray(np.asarray(T0s, dtype=np.float64).reshape(B, 16))
    p = AlignParams(int(max_iter), int(bool(lm)), float(rot_eps), float(trans_eps), float(max_corr_dist))
    res = (AlignResult * B)()
    rc = _lib.gicp_align_batched(_dptr(src), _dptr(src_cov.contiguous()), o.ctypes.data_as(_P), B, tgt.handle,
                                 _dptr(tgt_cov.contiguous()), T0h.ctypes.data_as(_P), ctypes.byref(p),
                                 ctypes.cast(res, _P), _stream())
    if not (allow_degenerate and rc == EDEGENERATE):
        _check(rc)
    Ts = np.array([np.array(r.T[:], dtype=np.float64).reshape(4, 4) for r in res])
    return Ts, [AlignInfo(int(r.iterations), bool(r.converged), float(r.error), int(r.inliers)) for r in res]


def align_batched_ex(src: torch.Tensor, src_cov: torch.Tensor, offsets, entry_reg, B: int, tgt: Index,
                     tgt_cov: torch.Tensor, T0s, reduce, max_iter=64, lm=True, rot_eps=1e-6, trans_eps=1e-5,
                     max_corr_dist=1.0, allow_degenerate=False):
    """Sharded batched align (gicp_align_batched_ex): E local entries (offsets [E+1]),
    entry e of registration entry_reg[e]; reduce(entry_rows [E,32] float64 numpy) ->
    registration rows [B,32] (the cross-rank combine, sharding.make_chunk_reducer)."""
    src = _pts(src, "src")
    o = _offsets(offsets, src.shape[0], allow_empty=True)  # a rank may hold no entry at all
    E = o.size - 1
    er = np.ascontiguousarray(np.asarray(entry_reg, dtype=np.int32).reshape(E))
    T0h = np.ascontiguousarray(np.asarray(T0s, dtype=np.float64).reshape(B, 16))
    p = AlignParams(int(max_iter), int(bool(lm)), float(rot_eps), float(trans_eps), float(max_corr_dist))
    res = (AlignResult * B)()
    err = []

    def cb(erows, ne, rrows, nb, user):
        try:
            rows = np.ctypeslib.as_array(erows, shape=(ne, 32)).copy() if ne > 0 else np.zeros((0, 32))
            out = np.asarray(reduce(rows), dtype=np.float64).reshape(nb, 32)
            np.ctypeslib.as_array(rrows, shape=(nb, 32))[:] = out
            return 0
        except Exception as e:  # reported after the call returns
            err.append(e)
            return 1
    cfn = REDUCE_FN(cb)
    rc = _lib.gicp_align_batched_ex(_dptr(src) if src.shape[0] else None,
                                    _dptr(src_cov.contiguous()) if src.shape[0] else None, o.ctypes.data_as(_P), E,
                                    er.ctypes.data_as(_P) if E else None, B, tgt.handle, _dptr(tgt_cov.contiguous()),
                                    T0h.ctypes.data_as(_P), ctypes.byref(p), ctypes.cast(res, _P), cfn, None,
                                    _stream())
    if err:
        raise err[0]
    if not (allow_degenerate and rc == EDEGENERATE):
        _check(rc)
    Ts = np.array([np.array(r.T[:], dtype=np.float64).reshape(4, 4) for r in res])
    return Ts, [AlignInfo(int(r.iterations), bool(r.converged), float(r.error), int(r.inliers)) for r in res]


def align_batched_sharded(src: torch.Tensor, src_cov: torch.Tensor, offsets, entry_chunk, num_chunks: int, B: int,
                          tgt: Index, tgt_cov: torch.Tensor, T0s, allreduce=None, max_iter=64, lm=True, rot_eps=1e-6,
                          trans_eps=1e-5, max_corr_dist=1.0, allow_degenerate=False):
    """Sharded batched align with the reduction on the device
    (gicp_align_batched_sharded): E local entries (offsets [E+1]), entry e = chunk
    row entry_chunk[e] = b * num_chunks + c. allreduce(table) must sum the float64
    device tensor `table` [B * num_chunks * 32] over the ranks in place on the
    current stream (torch.distributed.all_reduce; sharding.make_allreduce), or None
    for a single process."""
    src = _pts(src, "src")
    o = _offsets(offsets, src.shape[0], allow_empty=True)
    E = o.size - 1
    ec = np.ascontiguousarray(np.asarray(entry_chunk, dtype=np.int32).reshape(E))
    T0h = np.ascontiguousarray(np.asarray(T0s, dtype=np.float64).reshape(B, 16))
    p = AlignParams(int(max_iter), int(bool(lm)), float(rot_eps), float(trans_eps), float(max_corr_dist))
    res = (AlignResult * B)()
    table = torch.zeros(B * int(num_chunks) * 32, dtype=torch.float64, device=tgt.device)
    err = []

    def cb(ptr, count, user, stream):
        try:
            allreduce(table)
            return 0
        except Exception as e:  # reported after the call returns
            err.append(e)
            return 1
    cfn = ALLREDUCE_FN(cb) if allreduce is not None else ALLREDUCE_FN()
    rc = _lib.gicp_align_batched_sharded(_dptr(src) if src.shape[0] else None,
                                         _dptr(src_cov.contiguous()) if src.shape[0] else None, o.ctypes.data_as(_P),
                                         E, ec.ctypes.data_as(_P) if E else None, int(num_chunks), B, tgt.handle,
                                         _dptr(tgt_cov.contiguous()), T0h.ctypes.data_as(_P), ctypes.byref(p),
                                         ctypes.cast(res, _P), _dptr(table), cfn, None, _stream())
    if err:
        raise err[0]
    if not (allow_degenerate and rc == EDEGENERATE):
        _check(rc)
    Ts = np.array([np.array(r.T[:], dtype=np.float64).reshape(4, 4) for r in res])
    return Ts, [AlignInfo(int(r.iterations), bool(r.converged), float(r.error), int(r.inliers)) for r in res]


def combine_chunks(table: torch.Tensor, B: int, num_chunks: int, width: int, out=None) -> torch.Tensor:
    """gicp_combine_chunks: [B][num_chunks][width] float64 device -> [B][width], summed
    over the chunks in chunk order."""
    table = table.contiguous()
    out = out if out is not None else torch.empty((B, width), dtype=torch.float64, device=table.device)
    _check(_lib.gicp_combine_chunks(_dptr(table), int(B), int(num_chunks), int(width), _dptr(out), _stream()))
    return out


def knn_query_order(index: Index, q: torch.Tensor) -> torch.Tensor:
    """gicp_knn_query_order: the queries' cell-sorted order (int32 device [m])."""
    q = _pts(q, "q")
    perm = torch.empty(q.shape[0], dtype=torch.int32, device=q.device)
    _check(_lib.gicp_knn_query_order(index.handle, _dptr(q), q.shape[0], _dptr(perm), _stream()))
    return perm


def knn_subset(index: Index, q: torch.Tensor, ids: torch.Tensor, k: int, out):
    """gicp_knn_subset: rows ids of out = (nbr int32 [m, k], d2 float32 [m, k])."""
    q = _pts(q, "q")
    ids = ids.to(torch.int32).contiguous()
    nbr, d2 = out
    _check(_lib.gicp_knn_subset(index.handle, _dptr(q), q.shape[0], _dptr(ids) if ids.numel() else None, ids.numel(),
                                int(k), _dptr(nbr), _dptr(d2), _stream()))
    return nbr, d2


def index_export(index: Index):
    """gicp_index_export: (header bytes, [(device pointer or 0, bytes)] * n)."""
    hdr = (ctypes.c_ubyte * INDEX_HEADER_BYTES)()
    ptrs = (ctypes.c_void_p * INDEX_MAX_BUFFERS)()
    nbytes = (ctypes.c_int64 * INDEX_MAX_BUFFERS)()
    nb = ctypes.c_int(0)
    _check(_lib.gicp_index_export(index.handle, ctypes.cast(hdr, _P), ctypes.cast(ptrs, _P), ctypes.cast(nbytes, _P),
                                  ctypes.byref(nb)))
    return bytes(hdr), [(int(ptrs[i] or 0), int(nbytes[i])) for i in range(nb.value)]


def index_import(header: bytes, buffers, device) -> Index:
    """gicp_index_import from a header and device tensors (uint8) laid out as exported."""
    hdr = (ctypes.c_ubyte * INDEX_HEADER_BYTES).from_buffer_copy(header)
    ptrs = (ctypes.c_void_p * INDEX_MAX_BUFFERS)(*[(b.data_ptr() if b is not None and b.numel() else None)
                                                   for b in buffers])
    h = ctypes.c_void_p()
    _check(_lib.gicp_index_import(ctypes.cast(hdr, _P), ctypes.cast(ptrs, _P), _stream(), ctypes.byref(h)))
    return Index(h, torch.device(device))


def attach_voxels(index: Index, cov: torch.Tensor):
    """VGICP voxel Gaussians (N, mean, mean covariance) of the index's level-0 voxels;
    the index must be built with cell_size = the VGICP resolution."""
    index._voxcov = cov.contiguous()
    _check(_lib.gicp_index_attach_voxels(index.handle, _dptr(index._voxcov), _stream()))


def linearize_vgicp(src: torch.Tensor, src_cov: torch.Tensor, tgt: Index, T, mode: int = 7, pivot=None,
                    error_only: bool = False, base: torch.Tensor | None = None, reuse: bool = False, out=None):
    """Voxelized GICP linearisation -> (out29 float64 device [29] (28 = number of
    pairs), base int32 device [ns, 3] (each point's base voxel; reused when reuse))."""
    src = _pts(src, "src")
    Th = _T(T)
    out29 = out if out is not None else torch.empty(29, dtype=torch.float64, device=src.device)
    if base is None:
        if reuse:
            raise ValueError("reuse needs base")
        base = torch.empty((src.shape[0], 3), dtype=torch.int32, device=src.device)
    piv = None if pivot is None else np.ascontiguousarray(np.asarray(pivot, dtype=np.float64).reshape(3))
    flags = (LIN_ERROR_ONLY if error_only else 0) | (LIN_REUSE_CORR if reuse else 0)
    _check(_lib.gicp_linearize_vgicp(_dptr(src), _dptr(src_cov.contiguous()), src.shape[0], tgt.handle,
                                     Th.ctypes.data_as(_P), None if piv is None else piv.ctypes.data_as(_P), int(mode),
                                     flags, _dptr(base), _dptr(out29), _stream()))
    return out29, base


def align_vgicp(src: torch.Tensor, src_cov: torch.Tensor, tgt: Index, T0, mode: int = 7, max_iter=64,
                rot_eps=1e-6, trans_eps=1e-5):
    src = _pts(src, "src")
    T0h = _T(T0)
    p = AlignParams(int(max_iter), 1, float(rot_eps), float(trans_eps), 1.0)
    r = AlignResult()
    _check(_lib.gicp_align_vgicp(_dptr(src), _dptr(src_cov.contiguous()), src.shape[0], tgt.handle, int(mode),
                                 T0h.ctypes.data_as(_P), ctypes.byref(p), ctypes.byref(r), _stream()))
    T = np.array(r.T[:], dtype=np.float64).reshape(4, 4)
    return T, AlignInfo(int(r.iterations), bool(r.converged), float(r.error), int(r.inliers))


def ground_filter(xyz: torch.Tensor, cell: float, min_count: int, with_count: bool = False):
    """z-vote ground filter: keep (bool device [n]) = the point's 2-D cell holds
    >= min_count points (vertical features); optionally the counts (int32 [n])."""
    xyz = _pts(xyz, "xyz")
    n = xyz.shape[0]
    keep = torch.empty(n, dtype=torch.uint8, device=xyz.device)
    count = torch.empty(n, dtype=torch.int32, device=xyz.device) if with_count else None
    _check(_lib.gicp_ground_filter(_dptr(xyz) if n else None, n, float(cell), int(min_count),
                                   _dptr(keep) if n else None, None if count is None or not n else _dptr(count),
                                   _stream()))
    return (keep.bool(), count) if with_count else keep.bool()


def cluster(xyz: torch.Tensor, tol: float, min_size: int = 1):
    """Euclidean clusters: (labels int32 device [n] -- 0.. by descending size, -1
    below min_size --, number of clusters)."""
    xyz = _pts(xyz, "xyz")
    n = xyz.shape[0]
    lab = torch.empty(n, dtype=torch.int32, device=xyz.device)
    nc = ctypes.c_int64(0)
    _check(_lib.gicp_cluster(_dptr(xyz) if n else None, n, float(tol), int(min_size), _dptr(lab) if n else None,
                             ctypes.byref(nc), _stream()))
    return lab, int(nc.value)


class Submap:
    """Arc-length bucketed map (gicp_submap_*): query(center, radius) -> the point
    indices (int32 device) of the window of buckets around a race-line position."""

    def __init__(self, bucket: torch.Tensor, n_buckets: int):
        if bucket.dtype != torch.int32 or bucket.dim() != 1:
            raise ValueError("bucket must be int32 [n]")
        self._bucket = bucket.contiguous()
        self.n = bucket.shape[0]
        self.n_buckets = int(n_buckets)
        self.device = bucket.device
        h = _P()
        _check(_lib.gicp_submap_build(_dptr(self._bucket) if self.n else None, self.n, self.n_buckets,
                                      ctypes.byref(h), _stream()))
        self._h = h

    def query(self, center: int, radius: int) -> torch.Tensor:
        out = torch.empty(max(self.n, 1), dtype=torch.int32, device=self.device)
        cnt = ctypes.c_int64(0)
        _check(_lib.gicp_submap_query(self._h, int(center), int(radius), _dptr(out), ctypes.byref(cnt), _stream()))
        return out[:cnt.value]

    def free(self):
        if self._h:
            _lib.gicp_submap_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def align_timing(enable: bool = True):
    """Per-launch device timing of the aligns' linearisations on this thread: returns
    (ms, launches, points), each [dual, full, trial], accumulated since the previous
    call (points: source points linearised, summed over the launches), resets them
    and sets the enable flag."""
    ms = (ctypes.c_double * 3)()
    n = (ctypes.c_int64 * 3)()
    pts = (ctypes.c_int64 * 3)()
    _check(_lib.gicp_align_timing(int(bool(enable)), ctypes.cast(ms, _P), ctypes.cast(n, _P), ctypes.cast(pts, _P)))
    return list(ms), list(n), list(pts)


def version() -> int:
    return int(_lib.gicp_version())
