"""Pins for oracle O2 (fp64 covariance, Jacobi eigen, GICP plane regularisation).

Definition (readings R6, R7, R11): mu = (1/k) sum X_j,
S = (1/k) sum (X_j - mu)(X_j - mu)^T, eigenvalues replaced by (eps, 1, 1) in
ascending order, C = V diag(eps,1,1) V^T. Paper: the Gaussian model
p_i ~ N(p_i, C^p_i) and "computing covariance when estimate the
C^p_i and C^q_i" (l.404, l.413). SPEC examples S:284-286.
"""
import math

import numpy as np
import pytest

import gen

EPS = 1e-3


def _full(c6):
    c6 = np.asarray(c6)
    return np.array([[c6[0], c6[1], c6[2]], [c6[1], c6[3], c6[4]], [c6[2], c6[4], c6[5]]])


def _rot(seed):
    rng = np.random.default_rng(seed)
    Q, R = np.linalg.qr(rng.normal(size=(3, 3)))
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def test_jacobi_vs_lapack_eigh(orc):
    rng = np.random.default_rng(0)
    for t in range(300):
        A = rng.normal(size=(3, 3)) * 10 ** rng.uniform(-3, 3)
        S = A @ A.T
        if t % 3 == 0:  # near-degenerate spectra
            V = _rot(t)
            S = V @ np.diag([1e-6, 1.0, 1.0 + 10 ** -rng.uniform(1, 6)]) @ V.T
        lam, V = orc.jacobi3(S)
        ref = np.linalg.eigvalsh(S)
        assert np.allclose(lam, ref, rtol=1e-12, atol=1e-14 * np.abs(ref).max())
        assert np.allclose(V.T @ V, np.eye(3), atol=1e-13)
        assert np.allclose(S @ V, V * lam, atol=1e-12 * np.abs(ref).max())


def test_planar_grid_gives_exact_diag(orc):
    g = np.arange(-3, 4, dtype=np.float32) * 0.25
    x, y = np.meshgrid(g, g)
    P = np.stack([x.ravel(), y.ravel(), np.zeros(x.size)], -1).astype(np.float32)
    nbr = np.arange(len(P), dtype=np.int32)[None, :32]
    cov, gap, S6 = orc.covariance(P, nbr)
    assert np.allclose(_full(cov[0]), np.diag([1.0, 1.0, EPS]), atol=1e-14)


def test_tilted_plane_closed_form_and_spectrum(orc):
    rng = np.random.default_rng(1)
    for t in range(20):
        R = _rot(100 + t)
        uv = rng.uniform(-1, 1, (20, 2))
        local = np.concatenate([uv, np.zeros((20, 1))], 1)
        P = (local @ R.T + np.array([500.0, -300.0, 2.0])).astype(np.float32)
        nbr = np.arange(20, dtype=np.int32)[None]
        cov, gap, _ = orc.covariance(P, nbr)
        n = R[:, 2]
        C = _full(cov[0])
        # fp32 input rounding tilts the plane by ~1e-7 rad
        assert np.allclose(C, np.eye(3) - (1 - EPS) * np.outer(n, n), atol=1e-5)
        assert np.allclose(np.linalg.eigvalsh(C), [EPS, 1, 1], atol=1e-9)


def test_scatter_matches_numpy_cov_and_gap(orc):
    rng = np.random.default_rng(2)
    P = (rng.normal(size=(400, 3)) * [1.0, 0.5, 0.02] + [100, 200, 3]).astype(np.float32)
    nbr = rng.integers(0, 400, (50, 20)).astype(np.int32)
    cov, gap, S6 = orc.covariance(P, nbr)
    for i in range(50):
        X = P[nbr[i]].astype(np.float64)
        S = np.cov(X.T, bias=True)
        assert np.allclose(_full(S6[i]), S, rtol=1e-10, atol=1e-14)
        lam, V = np.linalg.eigh(S)
        assert math.isclose(gap[i], (lam[1] - lam[0]) / lam[2], rel_tol=1e-8, abs_tol=1e-12)
        Cref = V @ np.diag([EPS, 1, 1]) @ V.T
        if gap[i] > 1e-6:
            assert np.allclose(_full(cov[i]), Cref, atol=1e-8)


def test_rotation_equivariance(orc):
    rng = np.random.default_rng(3)
    P = (rng.normal(size=(300, 3)) * [2.0, 1.0, 0.05]).astype(np.float64)
    nbr = rng.integers(0, 300, (40, 16)).astype(np.int32)
    R = _rot(7)
    c1, g1, _ = orc.covariance(P.astype(np.float32), nbr)
    # rotate in fp64 then round: equivariance holds to fp32 input rounding
    c2, g2, _ = orc.covariance((P @ R.T).astype(np.float32), nbr)
    for i in range(40):
        if g1[i] > 1e-2:
            assert np.allclose(_full(c2[i]), R @ _full(c1[i]) @ R.T, atol=1e-4)


def test_noisy_plane_normal_within_one_degree(orc):
    # plane -> smallest regularised eigen-direction within 1 deg of the normal
    rng = np.random.default_rng(4)
    R = _rot(11)
    local = np.concatenate([rng.uniform(-2, 2, (2000, 2)), rng.normal(0, 0.001, (2000, 1))], 1)
    P = (local @ R.T).astype(np.float32)
    nbr, _ = orc.knn(P, P[:200], 20)
    cov, gap, _ = orc.covariance(P, nbr)
    n = R[:, 2]
    for i in range(200):
        w, V = np.linalg.eigh(_full(cov[i]))
        ang = math.degrees(math.acos(min(1.0, abs(V[:, 0] @ n))))
        assert ang < 1.0
        assert abs(w[0] - EPS) < 1e-9


def test_degenerate_duplicates_give_diag(orc):
    P = np.repeat(np.array([[812.5, -3.25, 1.0]], np.float32), 12, 0)
    nbr = np.arange(10, dtype=np.int32)[None]
    cov, gap, S6 = orc.covariance(P, nbr)
    assert np.allclose(_full(cov[0]), np.diag([1.0, 1.0, EPS]), rtol=0, atol=1e-15)
    assert gap[0] == 0.0 and np.all(S6[0] == 0)


def test_k1_and_errors(orc):
    P = gen.uniform_cloud(20, 1)
    cov, gap, _ = orc.covariance(P, np.arange(20, dtype=np.int32)[:, None])  # k = 1: single point
    assert np.allclose(cov, np.tile([1, 0, 0, 1, 0, EPS], (20, 1)))
    with pytest.raises(orc.OracleError):
        orc.covariance(P, np.full((2, 3), 99, np.int32))
