"""Independent numpy emulation of the O1 fp32 squared distance (test helper).

d2 = fmaf(dz, dz, fmaf(dy, dy, dx*dx)) with dx = fl32(qx - px) etc. Written from
the IEEE-754 definition, not from oracle/: a fused multiply-add is the exact
a*b + c rounded once to fp32. a*b of two fp32 values is exact in fp64 (48-bit
significand); a TwoSum gives the exact residual of the fp64 addition, which
decides the one case where rounding the fp64 sum to fp32 can differ from rounding
the exact value (the fp64 sum lands exactly on an fp32 rounding midpoint).
"""
import numpy as np


def _two_sum(a, b):
    s = a + b
    bb = s - a
    e = (a - (s - bb)) + (b - bb)
    return s, e


def fma32(a, b, c):
    a = np.asarray(a, np.float32).astype(np.float64)
    b = np.asarray(b, np.float32).astype(np.float64)
    c = np.asarray(c, np.float32).astype(np.float64)
    p = a * b                      # exact
    s, e = _two_sum(p, c)          # s + e == p + c exactly
    r = s.astype(np.float32)       # round-to-nearest-even of s
    # Is s exactly halfway between two fp32 neighbours? Then the sign of e decides.
    lo = np.where(r.astype(np.float64) <= s, r, np.nextafter(r, np.float32(-np.inf)))
    hi = np.where(r.astype(np.float64) >= s, r, np.nextafter(r, np.float32(np.inf)))
    mid = (lo.astype(np.float64) + hi.astype(np.float64)) * 0.5
    is_mid = (mid == s) & (lo != hi) & (e != 0)
    fix = np.where(e > 0, hi, lo)
    return np.where(is_mid, fix, r).astype(np.float32)


def d2_fp32(q, p):
    """q: [..., 3], p: [..., 3] float32 -> float32 d2 in the O1 order (broadcasting)."""
    q = np.asarray(q, np.float32)
    p = np.asarray(p, np.float32)
    dx = (q[..., 0] - p[..., 0]).astype(np.float32)
    dy = (q[..., 1] - p[..., 1]).astype(np.float32)
    dz = (q[..., 2] - p[..., 2]).astype(np.float32)
    xx = (dx * dx).astype(np.float32)
    return fma32(dz, dz, fma32(dy, dy, xx))


def knn_lexsort(tgt, q, k):
    """Independent brute force: lexsort by (d2 fp32, index) per query."""
    tgt = np.asarray(tgt, np.float32)
    q = np.asarray(q, np.float32)
    n = tgt.shape[0]
    idx = np.arange(n)
    nbr = np.empty((q.shape[0], k), np.int32)
    dd = np.empty((q.shape[0], k), np.float32)
    for i in range(q.shape[0]):
        d = d2_fp32(q[i][None, :], tgt)
        order = np.lexsort((idx, d))[:k]
        nbr[i] = order
        dd[i] = d[order]
    return nbr, dd
