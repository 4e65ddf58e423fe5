"""Pins for the parts of O3/O4 that a plausible mistake would otherwise slip through.

1. The rotated source covariance R C^p R^T in the compound covariance (PAPER.md
   eq_trans_err_dist l.388-395 / eq_trans_likelihood l.396-402, printed there as
   C^q - T^T C^p T; readings R1/R2). The expected values below are built
   from geometry only — a plane covariance I - (1-eps) n n^T carried by a rotation R
   has normal R n — and never from the matrix product the oracle evaluates, so a
   transposed rotation (R^T C R), a dropped rotation (C) or a sign error fails.
2. The strict gate d2 < fl32(r*r) (reading R3): fixtures with a nearest target at
   exactly r (exact dyadic arithmetic) must be outliers.
3. O4's LM gain ratio rho = (e - e') / (e - q(delta)) with the GN model
   q(delta) = e + 2 b^T delta + delta^T H delta (b = 1/2 de/ddelta, H the GN
   quadratic form — both pinned in test_oracle_linearize.py); the oracle computes the
   denominator as delta^T (lambda delta - b), equal to e - q(delta) only when delta
   solves (H + lambda I) delta = -b.
4. Recovery of a 10 degree rotation (|rot| <= 10 deg, error <= 0.05 m
   / 0.5 deg on structured clouds).
"""
import math

import numpy as np
import pytest

import gen

EPS = 2.0 ** -10            # exactly representable in fp32: covariances store it exactly


def _cov6(C):
    return np.array([C[0, 0], C[0, 1], C[0, 2], C[1, 1], C[1, 2], C[2, 2]], np.float32)


def _plane(n, eps=EPS):
    n = np.asarray(n, np.float64)
    n = n / np.linalg.norm(n)
    return np.eye(3) - (1 - eps) * np.outer(n, n)


def _H(o29):
    H = np.zeros((6, 6))
    k = 0
    for a in range(6):
        for b in range(a, 6):
            H[a, b] = H[b, a] = o29[k]
            k += 1
    return H


def _rz(deg):
    c, s = math.cos(math.radians(deg)), math.sin(math.radians(deg))
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def test_rotated_anisotropic_single_correspondence(orc):
    # T = Rz(30 deg), C^p = diag(1, eps, 1) (source plane normal e_y), C^q = diag(1, 1, eps).
    # The source plane seen in the target frame has normal u = R e_y = (-1/2, sqrt3/2, 0),
    # so A = C^q + R C^p R^T has eigenvectors u (1 + eps), w = (sqrt3/2, 1/2, 0) (2) and
    # e_z (1 + eps); in particular A_xy = +(1 - eps) sin30 cos30 (the literal T^T C^p T of
    # l.391 would give the opposite sign).
    R = _rz(30.0)
    T = np.eye(4)
    T[:3, :3] = R
    p = np.array([[2.0, 1.0, 0.5]], np.float32)
    pp = R @ p[0].astype(np.float64)
    q = (pp + np.array([0.125, -0.25, 0.0625])).astype(np.float32)[None]
    cs = np.diag([1.0, EPS, 1.0])
    cq = np.diag([1.0, 1.0, EPS])
    out, ab, corr = orc.linearize(p, _cov6(cs)[None], q, _cov6(cq)[None], T, 2.0)
    assert corr[0] == 0 and out[28] == 1
    # the fp64 transform in the oracle's FMA order differs from R @ p by rounding only
    d = q[0].astype(np.float64) - pp
    u = np.array([-0.5, math.sqrt(3) / 2, 0.0])
    w = np.array([math.sqrt(3) / 2, 0.5, 0.0])
    z = np.array([0.0, 0.0, 1.0])
    al, be, ga = d @ u, d @ w, d @ z
    e_ref = al * al / (1 + EPS) + be * be / 2 + ga * ga / (1 + EPS)
    assert math.isclose(out[27], e_ref, rel_tol=1e-12)
    Md = al / (1 + EPS) * u + be / 2 * w + ga / (1 + EPS) * z
    assert np.allclose(out[24:27], -Md, rtol=1e-10, atol=1e-14)          # v-block: -M d
    assert np.allclose(out[21:24], -np.cross(pp, Md), rtol=1e-10, atol=1e-13)
    M = np.outer(u, u) / (1 + EPS) + np.outer(w, w) / 2 + np.outer(z, z) / (1 + EPS)
    assert np.allclose(_H(out)[3:, 3:], M, rtol=1e-10, atol=1e-14)
    # what the plausible mistakes would have produced, for the record: they differ
    for wrong in (R.T @ cs @ R, cs):
        Mw = np.linalg.inv(cq + wrong)
        assert abs(d @ Mw @ d - e_ref) > 1e-2 * e_ref


def _orthonormal_pairs(rng, n):
    a = rng.normal(size=(n, 3))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    b = np.cross(a, rng.normal(size=(n, 3)))
    b /= np.linalg.norm(b, axis=1, keepdims=True)
    return a, b


def test_rotated_perpendicular_planes_many_points(orc):
    # Each correspondence: target normal n, source normal n_p chosen so that R n_p = m is
    # perpendicular to n. Then A = 2I - (1-eps)(m m^T + n n^T) has eigenpairs
    # (m, 1+eps), (n, 1+eps), (m x n, 2): e_i = ((d.m)^2 + (d.n)^2)/(1+eps) + (d.(m x n))^2/2.
    rng = np.random.default_rng(7)
    N = 64
    R = gen.euler_to_R(0.3, -0.2, 1.1)
    t = np.array([1.5, -2.0, 0.25])
    T = gen.make_T(R, t)
    src = (rng.uniform(-20, 20, size=(N, 3))).astype(np.float32)
    pp = src.astype(np.float64) @ R.T + t
    # targets spread far apart so the 1-NN of each transformed source is its own target
    dd = rng.uniform(-0.2, 0.2, size=(N, 3))
    tgt = (pp + dd).astype(np.float32)
    n, m = _orthonormal_pairs(rng, N)
    cq = np.stack([_cov6(_plane(n[i])) for i in range(N)])
    cp = np.stack([_cov6(_plane(R.T @ m[i])) for i in range(N)])
    out, ab, corr = orc.linearize(src, cp, tgt, cq, T, 1.0)
    assert np.array_equal(corr, np.arange(N))
    d = tgt.astype(np.float64) - pp
    x = np.cross(m, n)
    e_i = ((d * m).sum(1) ** 2 + (d * n).sum(1) ** 2) / (1 + EPS) + (d * x).sum(1) ** 2 / 2
    # fp32 storage of the covariances perturbs A by ~6e-8 relative, kappa <= 1/eps
    assert math.isclose(out[27], e_i.sum(), rel_tol=2e-4)
    Md = ((d * m).sum(1)[:, None] * m + (d * n).sum(1)[:, None] * n) / (1 + EPS) + (d * x).sum(1)[:, None] * x / 2
    assert np.allclose(out[24:27], -Md.sum(0), rtol=2e-4, atol=2e-4 * ab[24:27])
    assert np.allclose(out[21:24], -np.cross(pp, Md).sum(0), rtol=2e-4, atol=2e-4 * ab[21:24])


def test_global_rotation_invariance(orc):
    # Rotating the whole target frame by G (points, covariances G C^q G^T) and the pose to
    # G T leaves every residual's Mahalanobis length unchanged (e invariant; b's v-block
    # rotates by G). Holds for R C^p R^T only, not for R^T C^p R or C^p.
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    nt, _ = orc.knn(tgt, tgt, 10)
    ns, _ = orc.knn(src, src, 10)
    ct = orc.covariance(tgt, nt)[0]
    cs = orc.covariance(src, ns)[0].astype(np.float32)
    T = T_true @ gen.make_T(gen.euler_to_R(0.01, 0.02, -0.03), [0.02, 0.01, -0.01])
    out, ab, corr = orc.linearize(src, cs, tgt, ct.astype(np.float32), T, 1.0)
    assert out[28] > 100
    G = gen.euler_to_R(0.4, 0.7, -1.3)
    Gt = gen.make_T(G, [0.0, 0.0, 0.0])
    tgt_g = (tgt.astype(np.float64) @ G.T).astype(np.float32)
    full = np.array([[[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]] for c in ct])
    ct_g = np.stack([_cov6(G @ C @ G.T) for C in full])
    out_g, ab_g, _ = orc.linearize(src, cs, tgt_g, ct_g, Gt @ T, 1.0, corr=corr)
    # fp32 re-storage of rotated targets (~1e-7 m on a 10 m scene vs ~1 cm residuals)
    assert math.isclose(out_g[27], out[27], rel_tol=2e-3)


@pytest.mark.parametrize("r", [0.5, 0.75])
def test_gate_is_strict_at_exactly_r(orc, r):
    # targets on a 4 m lattice; sources offset from a target by exact dyadic vectors so
    # every fp32 d2 is exact: |offset| = r exactly -> outlier; 0.5 r -> inlier
    g = np.arange(0, 12, 4.0)
    tgt = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3).astype(np.float32)
    offs = np.array([[r, 0, 0], [0, -r, 0], [0, 0, r], [r / 2, 0, 0], [0, r / 2, r / 4],
                     [-r, 0, 0], [0, 0, -r / 2]], np.float32)
    src = (tgt[13] + offs).astype(np.float32)
    r2 = np.float32(r) * np.float32(r)
    d2 = (offs.astype(np.float64) ** 2).sum(1)
    assert np.all(d2.astype(np.float32) == d2)                 # exact
    expect_in = d2 < r2
    assert expect_in.sum() == 3 and (d2 == r2).sum() == 4
    cov = np.tile(_cov6(np.eye(3)), (len(tgt), 1))
    out, ab, corr = orc.linearize(src, cov[:len(src)], tgt, cov, np.eye(4), r)
    assert np.array_equal(corr >= 0, expect_in)
    assert np.all(corr[expect_in] == 13)
    assert out[28] == expect_in.sum()
    # with identity covariances M = I/2: e = sum of d2/2 over inliers
    assert math.isclose(out[27], d2[expect_in].sum() / 2, rel_tol=1e-15)


def test_lm_gain_ratio_uses_the_gauss_newton_model(orc):
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    nt, _ = orc.knn(tgt, tgt, 10)
    ns, _ = orc.knn(src, src, 10)
    ct = orc.covariance(tgt, nt)[0].astype(np.float32)
    cs = orc.covariance(src, ns)[0].astype(np.float32)
    r = orc.align(src, cs, tgt, ct, T0, trace=True)
    tr = r["trace"]
    assert len(tr) >= r["iterations"] - 1 and len(tr) > 2
    checked = 0
    for row in tr:
        lam, e, en, rho, acc = row[1], row[2], row[3], row[4], row[5]
        delta, b, H = row[6:12], row[12:18], _H(row[18:39])
        # delta solves (H + lambda I) delta = -b (LDL^T), independently re-solved
        assert np.allclose((H + lam * np.eye(6)) @ delta, -b, rtol=1e-8, atol=1e-10 * np.abs(b).max())
        pred = e - (e + 2 * b @ delta + delta @ H @ delta)     # e - q(delta), q the GN model
        assert pred > 0
        # the denominator the oracle divided by, against the model's predicted decrease
        # (near the optimum both are differences of ~equal terms: compare at their scale)
        den = (e - en) / rho
        assert abs(den - pred) <= 1e-4 * (abs(2 * b @ delta) + abs(delta @ H @ delta))
        assert bool(acc) == (rho > 0)
        if acc:
            assert en < e                                       # accepted steps decrease the cost
        checked += 1
    assert checked == len(tr)
    # far from the optimum the GN model predicts the first step's decrease closely (near
    # it, the dependence of M on R — not differentiated, reading R4 — dominates rho)
    assert abs(tr[0][4] - 1.0) < 0.01


def test_lm_rho_is_one_on_a_translation_only_quadratic(orc):
    # exact copy shifted by a pure translation, identical isotropic covariances: at every
    # trial the optimal delta has omega ~ 0 and the cost is quadratic in v, so rho ~ 1.
    tgt = gen.corner_scene(11, 0.0)
    src = (tgt - np.array([0.1, -0.05, 0.02], np.float32)).astype(np.float32)
    cov = np.tile(_cov6(np.eye(3) * 0.01), (len(tgt), 1))
    r = orc.align(src, cov, tgt, cov, np.eye(4), trace=True, max_corr_dist=0.5)
    tr = r["trace"]
    first = tr[0]
    assert first[5] == 1.0
    assert abs(first[4] - 1.0) < 1e-3


def test_ten_degree_rotation_recovered(orc):
    # |rot| <= 10 deg (with |t| <= 2 m) recovered within 0.05 m / 0.5 deg
    tgt = gen.corner_scene(11, 0.002)
    src = gen.corner_scene(12, 0.002)
    c = np.array([2.5, 2.5, 0.5])
    Tt = gen.make_T(_rz(10.0), c - _rz(10.0) @ c + np.array([0.3, -0.2, 0.05]))
    src_t = gen.apply_T(gen.inv_T(Tt), src).astype(np.float32)
    nt, _ = orc.knn(tgt, tgt, 10)
    ns, _ = orc.knn(src_t, src_t, 10)
    ct = orc.covariance(tgt, nt)[0].astype(np.float32)
    cs = orc.covariance(src_t, ns)[0].astype(np.float32)
    r = orc.align(src_t, cs, tgt, ct, np.eye(4), max_corr_dist=3.0)
    dt = np.linalg.norm(r["T"][:3, 3] - Tt[:3, 3])
    ang = math.acos(max(-1.0, min(1.0, (np.trace(r["T"][:3, :3] @ Tt[:3, :3].T) - 1) / 2)))
    assert dt < 0.05 and ang < math.radians(0.5)
