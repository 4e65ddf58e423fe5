"""Pins for oracle O3 (linearize) and the O4 building blocks (SE(3) exp, LDL^T).

Definition (readings R1-R4, R12): d_i = q_j* - T p_i
(PAPER.md eq_trans_err l.382-387), cost d^T (C^q + R C^p R^T)^-1 d (eq_trans_err_dist
l.388-395 / eq_trans_likelihood l.396-402, read with '+' and the inverse),
J = [skew(p') | -I] for T <- Exp(delta) T, H = sum J^T M J, b = sum J^T M d,
e = sum d^T M d, j* = gated brute-force 1-NN of fl32(T p).
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import gen
from tests.fp32emu import d2_fp32


def _H(o29):
    H = np.zeros((6, 6))
    k = 0
    for a in range(6):
        for b in range(a, 6):
            H[a, b] = H[b, a] = o29[k]
            k += 1
    return H


def _eye_cov(n):
    return np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (n, 1))


def _plane_cov(n, normal, eps=1e-3):
    C = np.eye(3) - (1 - eps) * np.outer(normal, normal)
    return np.tile(np.array([C[0, 0], C[0, 1], C[0, 2], C[1, 1], C[1, 2], C[2, 2]], np.float32), (n, 1))


def test_se3_exp_vs_scipy_rodrigues(orc):
    rng = np.random.default_rng(0)
    for t in range(50):
        w = rng.normal(size=3) * 10 ** rng.uniform(-12, 0.3)
        v = rng.normal(size=3)
        T = orc.se3_exp(np.concatenate([w, v]))
        R = Rotation.from_rotvec(w).as_matrix()
        assert np.allclose(T[:3, :3], R, atol=1e-12)
        assert np.allclose(T[3], [0, 0, 0, 1])
        # translation: V v with V the SO(3) left Jacobian; check via the
        # defining integral V = int_0^1 Exp(s w) ds (numerical quadrature)
        s = np.linspace(0, 1, 2001)
        Vq = np.trapezoid(np.stack([Rotation.from_rotvec(si * w).as_matrix() for si in s]), s, axis=0)
        assert np.allclose(T[:3, 3], Vq @ v, atol=1e-6)


def test_ldlt_vs_numpy_solve(orc):
    rng = np.random.default_rng(1)
    for _ in range(50):
        A = rng.normal(size=(6, 6))
        A = A @ A.T + 1e-3 * np.eye(6)
        y = rng.normal(size=6)
        assert np.allclose(orc.ldlt_solve6(A, y), np.linalg.solve(A, y), rtol=1e-8, atol=1e-10)


def test_correspondences_are_gated_bruteforce_nn(orc):
    tgt = gen.uniform_cloud(3000, 1, -5, 5)
    src = gen.uniform_cloud(400, 2, -6, 6)
    T = gen.make_T(gen.euler_to_R(0.1, -0.05, 0.3), [0.2, 0.1, -0.3])
    out, ab, corr = orc.linearize(src, _eye_cov(400), tgt, _eye_cov(3000), T, max_corr_dist=0.3)
    # independent: fp64 transform in the spec'd FMA order == numpy matmul up to
    # rounding; recompute with numpy fp64 and round to fp32, then lexsort-1NN
    p = src.astype(np.float64)
    pp = p @ T[:3, :3].T + T[:3, 3]
    s = pp.astype(np.float32)
    r2 = np.float32(0.3) * np.float32(0.3)
    mism = 0
    for i in range(400):
        d = d2_fp32(s[i][None], tgt)
        j = int(np.lexsort((np.arange(3000), d))[0])
        ref = j if d[j] < r2 else -1
        mism += int(corr[i] != ref)
    # the only admissible differences come from fp64 rounding of T p (1 ulp)
    assert mism == 0
    assert out[28] == np.count_nonzero(corr >= 0)


def test_exact_copy_identity_gives_zero(orc):
    tgt = gen.corner_scene(11)
    cov = _plane_cov(len(tgt), np.array([0, 0, 1.0]))
    out, ab, corr = orc.linearize(tgt, cov, tgt, cov, np.eye(4), 1.0)
    assert np.array_equal(corr, np.arange(len(tgt)))
    assert np.all(out[21:28] == 0.0)
    assert out[28] == len(tgt)
    H = _H(out)
    assert np.all(np.linalg.eigvalsh(H) > 0)


def test_single_correspondence_closed_form(orc):
    # C = diag(1,1,eps) on both sides, R = I: M = diag(1/2, 1/2, 1/(2 eps));
    # e = (dx^2 + dy^2)/2 + dz^2/(2 eps); b = J^T M d with J = [skew(p) | -I].
    eps = 1e-3
    tgt = np.array([[1.0, 2.0, 3.0]], np.float32)
    src = np.array([[1.25, 1.5, 3.125]], np.float32)
    cov = _plane_cov(1, np.array([0, 0, 1.0]), eps)
    out, ab, corr = orc.linearize(src, cov, tgt, cov, np.eye(4), 2.0)
    d = tgt[0].astype(np.float64) - src[0]
    # A = C + C (fp32 storage of eps rounds), M = A^-1
    c = np.float32(1 - (1 - eps))
    m = np.array([0.5, 0.5, 1 / (2 * float(c))])
    assert math.isclose(out[27], (m * d * d).sum(), rel_tol=1e-12)
    assert np.allclose(out[24:27], -(m * d), rtol=1e-12)                 # v-block: -M d
    p = src[0].astype(np.float64)
    # omega-block: skew(p)^T M d = -skew(p) M d = -(p x M d)
    assert np.allclose(out[21:24], -np.cross(p, m * d), rtol=1e-12)
    H = _H(out)
    assert np.allclose(H[3:, 3:], np.diag(m), rtol=1e-12)


def test_b_is_half_gradient_of_e(orc):
    # With isotropic source covariances M does not depend on R, so with corr held
    # fixed e(Exp(t u) T) has derivative 2 b^T u at t = 0 (central differences).
    tgt = gen.corner_scene(11, 0.002)
    src = gen.corner_scene(12, 0.002)
    nbr, _ = orc.knn(tgt, tgt, 10)
    ct, _, _ = orc.covariance(tgt, nbr)
    ct = ct.astype(np.float32)
    cs = _eye_cov(len(src)) * np.float32(0.01)
    T = gen.make_T(gen.euler_to_R(0.01, -0.02, 0.03), [0.05, -0.04, 0.02])
    out, ab, corr = orc.linearize(src, cs, tgt, ct, T, 1.0)
    b = out[21:27]
    h = 1e-6
    for a in range(6):
        u = np.zeros(6)
        u[a] = h
        ep = orc.linearize(src, cs, tgt, ct, orc.se3_exp(u) @ T, 1.0, corr=corr)[0][27]
        em = orc.linearize(src, cs, tgt, ct, orc.se3_exp(-u) @ T, 1.0, corr=corr)[0][27]
        g = (ep - em) / (2 * h)
        assert math.isclose(g, 2 * b[a], rel_tol=1e-5, abs_tol=1e-6 * ab[21 + a])


def test_H_is_gauss_newton_quadratic_form(orc):
    # At d = 0 (exact copy, T = I) e(Exp(t u)) = t^2 u^T H u + O(t^3) for any
    # covariances: check the diagonal and, by polarisation, off-diagonals.
    tgt = gen.corner_scene(11, 0.002)
    nbr, _ = orc.knn(tgt, tgt, 10)
    ct, _, _ = orc.covariance(tgt, nbr)
    ct = ct.astype(np.float32)
    out, ab, corr = orc.linearize(tgt, ct, tgt, ct, np.eye(4), 1.0)
    H = _H(out)
    t = 1e-5

    def Q(u):
        ep = orc.linearize(tgt, ct, tgt, ct, orc.se3_exp(t * u), 1.0, corr=corr)[0][27]
        em = orc.linearize(tgt, ct, tgt, ct, orc.se3_exp(-t * u), 1.0, corr=corr)[0][27]
        return (ep + em) / (2 * t * t)

    E = np.eye(6)
    for a in range(6):
        assert math.isclose(Q(E[a]), H[a, a], rel_tol=1e-4)
    for a, c in [(0, 3), (1, 5), (2, 4), (0, 1), (3, 4)]:
        pol = (Q(E[a] + E[c]) - Q(E[a] - E[c])) / 4
        assert math.isclose(pol, H[a, c], rel_tol=1e-3, abs_tol=1e-4 * math.sqrt(H[a, a] * H[c, c]))


def test_sum_is_order_exact_sum_of_point_terms(orc):
    # the reduction equals the exactly-rounded sum (math.fsum) of the per-point
    # terms obtained by linearising each point alone
    tgt = gen.corner_scene(11, 0.002)
    src = gen.corner_scene(12, 0.002)[:200]
    nbr, _ = orc.knn(tgt, tgt, 10)
    ct = orc.covariance(tgt, nbr)[0].astype(np.float32)
    cs = _eye_cov(len(src)) * np.float32(0.02)
    T = gen.make_T(gen.euler_to_R(0.0, 0.0, 0.02), [0.1, 0.0, 0.0])
    out, ab, corr = orc.linearize(src, cs, tgt, ct, T, 1.0)
    terms = np.array([orc.linearize(src[i:i + 1], cs[i:i + 1], tgt, ct, T, 1.0)[0] for i in range(len(src))])
    for c in range(28):
        ref = math.fsum(terms[:, c])
        assert math.isclose(out[c], ref, rel_tol=1e-14, abs_tol=1e-14 * ab[c])
    assert out[28] == terms[:, 28].sum()


def test_H_symmetric_psd_and_condition_bound(orc):
    src, tgt, T, T0 = gen.config_c1(sigma=0.002)
    nt, _ = orc.knn(tgt, tgt, 10)
    ns, _ = orc.knn(src, src, 10)
    ct = orc.covariance(tgt, nt)[0].astype(np.float32)
    cs = orc.covariance(src, ns)[0].astype(np.float32)
    out, ab, corr = orc.linearize(src, cs, tgt, ct, T, 1.0)
    w = np.linalg.eigvalsh(_H(out))
    assert w.min() > -1e-9 * w.max()
    # per correspondence, cond(C^q + R C^p R^T) <= 1/eps
    for i in np.nonzero(corr >= 0)[0][:50]:
        Cq = ct[corr[i]]
        Cp = cs[i]
        f = lambda c: np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]], np.float64)
        A = f(Cq) + T[:3, :3] @ f(Cp) @ T[:3, :3].T
        assert np.linalg.cond(A) <= 1 / 1e-3 * (1 + 1e-4)


def test_errors(orc):
    p = gen.uniform_cloud(10, 1)
    with pytest.raises(orc.OracleError):
        orc.linearize(p, _eye_cov(10), p, _eye_cov(10), np.eye(4), 0.0)


def test_pivoted_exp_fixes_the_pivot(orc):
    rng = np.random.default_rng(5)
    for _ in range(10):
        c = rng.normal(size=3) * 300
        w = rng.normal(size=3) * 0.1
        E = orc.pivoted_exp(np.concatenate([w, np.zeros(3)]), c)
        assert np.allclose(E[:3, :3] @ c + E[:3, 3], c, atol=1e-9)       # rotation about c
        v = rng.normal(size=3)
        E2 = orc.pivoted_exp(np.concatenate([np.zeros(3), v]), c)
        assert np.allclose(E2[:3, :3], np.eye(3)) and np.allclose(E2[:3, 3], v)


def test_pivoted_jacobian_finite_differences(orc):
    # with a pivot c, J = [skew(p' - c) | -I] for T <- Tr(c) Exp(delta) Tr(-c) T:
    # b = 1/2 de/ddelta (isotropic source covariances) and H the GN quadratic form
    tgt = (gen.corner_scene(11, 0.002) + np.array([480.0, -250.0, 3.0], np.float32)).astype(np.float32)
    src = (gen.corner_scene(12, 0.002) + np.array([480.0, -250.0, 3.0], np.float32)).astype(np.float32)
    nbr, _ = orc.knn(tgt, tgt, 10)
    ct = orc.covariance(tgt, nbr)[0].astype(np.float32)
    cs = _eye_cov(len(src)) * np.float32(0.01)
    c = np.array([478.0, -251.0, 2.0])
    T = gen.make_T(gen.euler_to_R(0.001, -0.002, 0.003), [0.05, -0.04, 0.02])
    out, ab, corr = orc.linearize(src, cs, tgt, ct, T, 1.0, pivot=c)
    b = out[21:27]
    h = 1e-6
    for a in range(6):
        u = np.zeros(6)
        u[a] = h
        ep = orc.linearize(src, cs, tgt, ct, orc.pivoted_exp(u, c) @ T, 1.0, corr=corr, pivot=c)[0][27]
        em = orc.linearize(src, cs, tgt, ct, orc.pivoted_exp(-u, c) @ T, 1.0, corr=corr, pivot=c)[0][27]
        assert math.isclose((ep - em) / (2 * h), 2 * b[a], rel_tol=1e-5, abs_tol=1e-6 * ab[21 + a])
    # exact copy at T = I: quadratic form of H
    out, ab, corr = orc.linearize(tgt, ct, tgt, ct, np.eye(4), 1.0, pivot=c)
    Hm = _H(out)
    t = 1e-5
    for a in range(6):
        E = np.zeros(6)
        E[a] = 1.0
        ep = orc.linearize(tgt, ct, tgt, ct, orc.pivoted_exp(t * E, c), 1.0, corr=corr, pivot=c)[0][27]
        em = orc.linearize(tgt, ct, tgt, ct, orc.pivoted_exp(-t * E, c), 1.0, corr=corr, pivot=c)[0][27]
        assert math.isclose((ep + em) / (2 * t * t), Hm[a, a], rel_tol=1e-4)
