"""The CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package. The product path (paper_2308_07173_b200) never does.

Python side: ctypes marshalling of numpy arrays into oracle/oracle.c (plain C,
fp64, brute force), which holds every piece of the method's arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, EK, EDEGENERATE = 0, -1, -2, -6
LIN_REUSE_CORR = 1


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


class AlignParams(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int), ("lm", ctypes.c_int), ("rot_eps", ctypes.c_double),
                ("trans_eps", ctypes.c_double), ("max_corr_dist", ctypes.c_float)]


class AlignResult(ctypes.Structure):
    _fields_ = [("T", ctypes.c_double * 16), ("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("error", ctypes.c_double), ("inliers", ctypes.c_int64)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, f32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_double
        L.oracle_knn.argtypes = [P, i64, P, i64, i32, P, P, i32]
        L.oracle_d2.argtypes = [P, P]
        L.oracle_d2.restype = f32
        L.oracle_jacobi3.argtypes = [P, P, P]
        L.oracle_covariance.argtypes = [P, i64, P, i64, i32, f64, P, P, P, i32]
        L.oracle_linearize.argtypes = [P, P, i64, P, P, i64, P, P, f32, i32, P, P, P, i32]
        L.oracle_pivoted_exp.argtypes = [P, P, P]
        L.oracle_pivoted_exp.restype = None
        L.oracle_se3_exp.argtypes = [P, P]
        L.oracle_se3_exp.restype = None
        L.oracle_ldlt_solve6.argtypes = [P, P, P]
        L.oracle_kernel_eval.argtypes = [i32, f64, f64, f64, i32, P, P]
        L.oracle_kernel_eval.restype = f64
        L.oracle_covariance_kd.argtypes = [P, i64, P, P, i64, i32, i32, f64, f64, f64, i32, P, i32, f64, P, P, i32]
        L.oracle_ground_filter.argtypes = [P, i64, f32, i32, P, P]
        L.oracle_cluster.argtypes = [P, i64, f32, i32, P]
        L.oracle_submap_query.argtypes = [P, i64, i32, i32, i32, P]
        L.oracle_submap_query.restype = i64
        L.oracle_cluster.restype = i64
        L.oracle_linearize_vgicp.argtypes = [P, P, i64, P, P, i64, f32, P, P, i32, i32, P, P, P]
        L.oracle_align_vgicp.argtypes = [P, P, i64, P, P, i64, f32, i32, P, ctypes.POINTER(AlignParams),
                                         ctypes.POINTER(AlignResult)]
        L.oracle_align.argtypes = [P, P, i64, P, P, i64, P, ctypes.POINTER(AlignParams),
                                   ctypes.POINTER(AlignResult), i32]
        L.oracle_align_ex.argtypes = [P, P, i64, P, P, i64, P, ctypes.POINTER(AlignParams),
                                      ctypes.POINTER(AlignResult), i32, P, i32, ctypes.POINTER(ctypes.c_int)]
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what} failed with code {code}")
        self.code = code


def knn(tgt, q, k, nthreads=0):
    """O1: (nbr int32 [m,k], d2 float32 [m,k]) -- brute force over all targets."""
    tgt, q = _f32(tgt), _f32(q)
    m = q.shape[0]
    nbr = np.empty((m, k), np.int32)
    d2 = np.empty((m, k), np.float32)
    rc = lib().oracle_knn(_ptr(tgt), tgt.shape[0], _ptr(q), m, k, _ptr(nbr), _ptr(d2), nthreads)
    if rc != OK:
        raise OracleError(rc, "oracle_knn")
    return nbr, d2


def d2(q, p):
    q, p = _f32(q), _f32(p)
    return float(lib().oracle_d2(_ptr(q), _ptr(p)))


def jacobi3(S):
    S = np.ascontiguousarray(S, dtype=np.float64).reshape(3, 3)
    lam = np.empty(3)
    V = np.empty((3, 3))
    lib().oracle_jacobi3(_ptr(S), _ptr(lam), _ptr(V))
    return lam, V


def covariance(xyz, nbr, eps=1e-3, nthreads=0):
    """O2: (cov fp64 [m,6], gap [m], S6 [m,6])."""
    xyz = _f32(xyz)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    m, k = nbr.shape
    cov = np.empty((m, 6))
    gap = np.empty(m)
    S6 = np.empty((m, 6))
    rc = lib().oracle_covariance(_ptr(xyz), xyz.shape[0], _ptr(nbr), m, k, eps, _ptr(cov), _ptr(gap),
                                 _ptr(S6), nthreads)
    if rc != OK:
        raise OracleError(rc, "oracle_covariance")
    return cov, gap, S6


def linearize(src, src_cov, tgt, tgt_cov, T, max_corr_dist=1.0, corr=None, nthreads=0, pivot=None):
    """O3: (out29, absum29, corr). With corr given: REUSE_CORR (no search).
    pivot: the point the rotation of the perturbation is about (default origin)."""
    src, tgt = _f32(src), _f32(tgt)
    src_cov, tgt_cov = _f32(src_cov), _f32(tgt_cov)
    T = np.ascontiguousarray(T, dtype=np.float64)
    out = np.empty(29)
    ab = np.empty(29)
    flags = 0
    if corr is not None:
        corr = np.ascontiguousarray(corr, dtype=np.int32).copy()
        flags = LIN_REUSE_CORR
    else:
        corr = np.empty(src.shape[0], np.int32)
    piv = None if pivot is None else np.ascontiguousarray(pivot, dtype=np.float64)
    rc = lib().oracle_linearize(_ptr(src), _ptr(src_cov), src.shape[0], _ptr(tgt), _ptr(tgt_cov), tgt.shape[0],
                                _ptr(T), None if piv is None else _ptr(piv), max_corr_dist, flags, _ptr(out),
                                _ptr(ab), _ptr(corr), nthreads)
    if rc != OK:
        raise OracleError(rc, "oracle_linearize")
    return out, ab, corr


KD_UNIFORM, KD_RBF, KD_GAUSSIAN, KD_POLYNOMIAL, KD_HI, KD_LAPLACIAN = range(6)
REG_PLANE, REG_MIN_EIG, REG_NORMALIZED_MIN_EIG = range(3)


def kernel_eval(kind, x, y, sigma=1.0, alpha=1.0, c=0.0, d=2):
    """O5: one Table I kernel value K(x, y) (x = query, y = neighbour)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return float(lib().oracle_kernel_eval(int(kind), float(sigma), float(alpha), float(c), int(d), _ptr(x), _ptr(y)))


def covariance_kd(xyz, nbr, kind, q=None, sigma=1.0, alpha=1.0, c=0.0, d=2, origin=(0.0, 0.0, 0.0),
                  reg=REG_PLANE, eps=1e-3, nthreads=0):
    """O6: kernel-weighted covariance, (cov fp64 [m,6], gap [m])."""
    xyz = _f32(xyz)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    m, k = nbr.shape
    qq = None if q is None else _f32(q)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    cov = np.empty((m, 6))
    gap = np.empty(m)
    rc = lib().oracle_covariance_kd(_ptr(xyz), xyz.shape[0], None if qq is None else _ptr(qq), _ptr(nbr), m, k,
                                    int(kind), float(sigma), float(alpha), float(c), int(d), _ptr(o), int(reg),
                                    float(eps), _ptr(cov), _ptr(gap), nthreads)
    if rc != OK:
        raise OracleError(rc, "oracle_covariance_kd")
    return cov, gap


def linearize_vgicp(src, src_cov, tgt, tgt_cov, T, res=1.0, mode=7, pivot=None, base=None):
    """O7: voxelized GICP linearisation -> (out29, absum29, base). With base given
    (int32 [ns,3]) the pairs are those base voxels (REUSE); otherwise they are
    computed at T and returned."""
    src, tgt = _f32(src), _f32(tgt)
    src_cov, tgt_cov = _f32(src_cov), _f32(tgt_cov)
    T = np.ascontiguousarray(T, dtype=np.float64)
    piv = None if pivot is None else np.ascontiguousarray(pivot, dtype=np.float64)
    out = np.empty(29)
    ab = np.empty(29)
    flags = 0
    if base is not None:
        base = np.ascontiguousarray(base, dtype=np.int32).copy()
        flags = LIN_REUSE_CORR
    else:
        base = np.empty((src.shape[0], 3), np.int32)
    rc = lib().oracle_linearize_vgicp(_ptr(src), _ptr(src_cov), src.shape[0], _ptr(tgt), _ptr(tgt_cov), tgt.shape[0],
                                      float(res), _ptr(T), None if piv is None else _ptr(piv), int(mode), flags,
                                      _ptr(base), _ptr(out), _ptr(ab))
    if rc != OK:
        raise OracleError(rc, "oracle_linearize_vgicp")
    return out, ab, base


def align_vgicp(src, src_cov, tgt, tgt_cov, T0, res=1.0, mode=7, max_iter=64, rot_eps=1e-6, trans_eps=1e-5):
    """O8: LM on O7 -> dict(T, iterations, converged, error, inliers)."""
    src, tgt = _f32(src), _f32(tgt)
    src_cov, tgt_cov = _f32(src_cov), _f32(tgt_cov)
    T0 = np.ascontiguousarray(T0, dtype=np.float64)
    p = AlignParams(max_iter, 1, rot_eps, trans_eps, 1.0)
    r = AlignResult()
    rc = lib().oracle_align_vgicp(_ptr(src), _ptr(src_cov), src.shape[0], _ptr(tgt), _ptr(tgt_cov), tgt.shape[0],
                                  float(res), int(mode), _ptr(T0), ctypes.byref(p), ctypes.byref(r))
    if rc != OK:
        raise OracleError(rc, "oracle_align_vgicp")
    return dict(T=np.array(r.T[:]).reshape(4, 4), iterations=r.iterations, converged=bool(r.converged),
                error=r.error, inliers=r.inliers)


def ground_filter(xyz, cell, min_count):
    """O9: (keep bool [n], count int32 [n]) of the z-vote filter."""
    xyz = _f32(xyz).reshape(-1, 3)
    n = xyz.shape[0]
    keep = np.zeros(n, np.uint8)
    count = np.zeros(n, np.int32)
    rc = lib().oracle_ground_filter(_ptr(xyz), n, float(cell), int(min_count), _ptr(count), _ptr(keep))
    if rc != OK:
        raise OracleError(rc, "oracle_ground_filter")
    return keep.astype(bool), count


def cluster(xyz, tol, min_size=1):
    """O10: (labels int32 [n] -- rank by descending size, -1 if dropped --, count)."""
    xyz = _f32(xyz).reshape(-1, 3)
    lab = np.empty(xyz.shape[0], np.int32)
    nc = lib().oracle_cluster(_ptr(xyz), xyz.shape[0], float(tol), int(min_size), _ptr(lab))
    if nc < 0:
        raise OracleError(int(nc), "oracle_cluster")
    return lab, int(nc)


def submap_query(bucket, n_buckets, center, radius):
    """O11: point indices of the window of buckets around `center` (int32 [m])."""
    b = np.ascontiguousarray(bucket, dtype=np.int32)
    out = np.empty(max(1, b.size), np.int32)
    m = lib().oracle_submap_query(_ptr(b), b.size, int(n_buckets), int(center), int(radius), _ptr(out))
    if m < 0:
        raise OracleError(int(m), "oracle_submap_query")
    return out[:m].copy()


def se3_exp(delta):
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    T = np.empty((4, 4))
    lib().oracle_se3_exp(_ptr(delta), _ptr(T))
    return T


def pivoted_exp(delta, pivot):
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    c = np.ascontiguousarray(pivot, dtype=np.float64)
    T = np.empty((4, 4))
    lib().oracle_pivoted_exp(_ptr(delta), _ptr(c), _ptr(T))
    return T


def ldlt_solve6(A, y):
    A = np.ascontiguousarray(A, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = np.empty(6)
    rc = lib().oracle_ldlt_solve6(_ptr(A), _ptr(y), _ptr(x))
    if rc != 0:
        raise OracleError(rc, "oracle_ldlt_solve6")
    return x


TRACE_W = 40


def align(src, src_cov, tgt, tgt_cov, T0, max_iter=64, lm=True, rot_eps=1e-6, trans_eps=1e-5,
          max_corr_dist=1.0, nthreads=0, trace=False):
    """O4: returns dict(T, iterations, converged, error, inliers) and, with trace=True,
    'trace': one row per LM trial [it, lambda, e, e', rho, accepted, delta(6), b(6), H(21), 0]."""
    src, tgt = _f32(src), _f32(tgt)
    src_cov, tgt_cov = _f32(src_cov), _f32(tgt_cov)
    T0 = np.ascontiguousarray(T0, dtype=np.float64)
    p = AlignParams(max_iter, int(lm), rot_eps, trans_eps, max_corr_dist)
    r = AlignResult()
    cap = 10 * max_iter if trace else 0
    tr = np.zeros((max(cap, 1), TRACE_W))
    ntr = ctypes.c_int(0)
    rc = lib().oracle_align_ex(_ptr(src), _ptr(src_cov), src.shape[0], _ptr(tgt), _ptr(tgt_cov), tgt.shape[0],
                               _ptr(T0), ctypes.byref(p), ctypes.byref(r), nthreads,
                               _ptr(tr) if trace else None, cap, ctypes.byref(ntr))
    if rc != OK:
        raise OracleError(rc, "oracle_align")
    out = dict(T=np.array(r.T[:]).reshape(4, 4), iterations=r.iterations, converged=bool(r.converged),
               error=r.error, inliers=r.inliers)
    if trace:
        out["trace"] = tr[:ntr.value].copy()
    return out


def pack_cov(cov6):
    """fp64 [m,6] -> fp32 [m,6] (the library's covariance storage)."""
    return np.ascontiguousarray(np.asarray(cov6, dtype=np.float64).astype(np.float32))
