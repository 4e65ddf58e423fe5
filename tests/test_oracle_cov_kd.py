"""Pins of the kernel-descriptor oracle (O5 kernel_eval, O6 covariance_kd;
PAPER.md Table I l.420-435, readings R19-R21).
Each check is against something other than the oracle's own formula: SPEC's
worked kernel values, closed forms, LAPACK (numpy eigh / weighted
np.cov), exact reductions to the unweighted oracle, invariances."""
import math

import numpy as np
import pytest

import gen

orc = pytest.importorskip("oracle")
K = orc


def test_kernel_values_worked_examples():
    # SPEC S:275-277
    assert K.kernel_eval(K.KD_LAPLACIAN, [1.5, -2.0, 3.0], [1.5, -2.0, 3.0], sigma=0.7) == 1.0
    assert K.kernel_eval(K.KD_RBF, [0, 0, 0], [1, 0, 0], sigma=1.0) == pytest.approx(math.exp(-1.0), rel=1e-15)
    assert K.kernel_eval(K.KD_POLYNOMIAL, [1, 1, 1], [1, 1, 1], alpha=1.0, c=0.0, d=2) == 9.0
    # closed forms of the other rows of Table I
    s = 0.5
    x, y = np.array([0.0, 0.0, 0.0]), np.array([0.0, 2 * s, 0.0])   # ||x-y||^2 = 4 s^2
    assert K.kernel_eval(K.KD_GAUSSIAN, x, y, sigma=s) == pytest.approx(math.exp(-2.0), rel=1e-15)
    assert K.kernel_eval(K.KD_LAPLACIAN, x, y, sigma=s) == pytest.approx(math.exp(-2.0), rel=1e-15)
    assert K.kernel_eval(K.KD_RBF, x, y, sigma=3.0) == pytest.approx(math.exp(-3.0), rel=1e-15)  # times sigma
    assert K.kernel_eval(K.KD_HI, [1, 2, 3], [3, 2, 1]) == pytest.approx(4.0 / 6.0, rel=1e-15)
    assert K.kernel_eval(K.KD_POLYNOMIAL, [1, 2, 0], [3, 1, 5], alpha=0.5, c=1.0, d=3) == pytest.approx(3.5 ** 3)
    assert K.kernel_eval(K.KD_UNIFORM, [1, 2, 3], [9, 9, 9]) == 1.0


@pytest.fixture(scope="module")
def cloud():
    xyz = gen.uniform_cloud(3000, 5, lo=-4.0, hi=4.0)
    nbr, _ = K.knn(xyz, xyz, 16)
    return xyz, nbr


def test_uniform_kernel_is_the_unweighted_oracle_bitwise(cloud):
    xyz, nbr = cloud
    c0, g0, _ = K.covariance(xyz, nbr)
    c1, g1 = K.covariance_kd(xyz, nbr, K.KD_UNIFORM)
    assert np.array_equal(c0, c1) and np.array_equal(g0, g1)
    # an infinitely wide Gaussian weights every neighbour exactly 1.0
    c2, _ = K.covariance_kd(xyz, nbr, K.KD_GAUSSIAN, sigma=1e12)
    assert np.array_equal(c0, c2)
    # a polynomial kernel that is negative everywhere is clamped to 0 -> uniform
    c3, _ = K.covariance_kd(xyz, nbr, K.KD_POLYNOMIAL, alpha=0.0, c=-1.0, d=1)
    assert np.array_equal(c0, c3)


@pytest.mark.parametrize("kind,sigma", [(1, 2.0), (2, 0.5), (3, 1.0), (4, 1.0), (5, 0.5)])
@pytest.mark.parametrize("reg", [1, 2])
def test_weighted_scatter_and_clamps_vs_lapack(cloud, kind, sigma, reg):
    """MIN_EIG / NORMALIZED_MIN_EIG: C = V diag(clamp(lam)) V^T with (lam, V) from
    numpy eigh of the weighted scatter np.cov(aweights=w, bias=True), the weights
    from the (separately pinned) kernel_eval."""
    xyz, nbr = cloud
    o = xyz.min(axis=0).astype(np.float64)
    rows = np.arange(0, 3000, 97)
    cov, _ = K.covariance_kd(xyz, nbr[rows], kind, q=xyz[rows], sigma=sigma, alpha=0.01, c=1.0, d=2, origin=o,
                             reg=reg)
    for t, i in enumerate(rows):
        X = xyz[nbr[i]].astype(np.float64)
        qx = xyz[i].astype(np.float64) - o
        Y = X - o
        if kind == K.KD_HI:
            qx, Y = np.maximum(qx, 0), np.maximum(Y, 0)
        w = np.array([max(0.0, K.kernel_eval(kind, qx, y, sigma=sigma, alpha=0.01, c=1.0, d=2)) for y in Y])
        S = np.cov(X.T, aweights=w, bias=True)
        lam, V = np.linalg.eigh(S)
        lw = np.maximum(lam, 1e-3) if reg == 1 else np.maximum(lam / lam[2], 1e-3)
        C = (V * lw) @ V.T
        got = cov[t]
        ref = np.array([C[0, 0], C[0, 1], C[0, 2], C[1, 1], C[1, 2], C[2, 2]])
        assert np.abs(got - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max()), (kind, reg, i)


@pytest.mark.parametrize("kind", range(6))
def test_plane_any_kernel_gives_the_plane_model(kind):
    """points on a plane, any kernel -> the regularised normal is the
    plane normal; noise-free: C = I - (1 - eps) n n^T to rounding."""
    rng = np.random.default_rng(3)
    n = np.array([0.3, -0.4, 0.866])
    n /= np.linalg.norm(n)
    u = np.cross(n, [1.0, 0.0, 0.0])
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    uv = rng.uniform(-2, 2, (400, 2))
    pts = (np.array([5.0, 6.0, 7.0]) + uv[:, :1] * u + uv[:, 1:] * v).astype(np.float32)
    nbr, _ = K.knn(pts, pts, 12)
    cov, _ = K.covariance_kd(pts, nbr, kind, sigma=0.5, alpha=0.01, c=1.0, d=2, origin=pts.min(0).astype(np.float64))
    ref = np.eye(3) - (1 - 1e-3) * np.outer(n, n)
    r6 = np.array([ref[0, 0], ref[0, 1], ref[0, 2], ref[1, 1], ref[1, 2], ref[2, 2]])
    assert np.abs(cov - r6).max() < 2e-5  # fp32 coordinates of the plane


def test_distance_kernels_are_translation_invariant(cloud):
    xyz, nbr = cloud
    sh = np.array([1000.0, -500.0, 20.0])
    xyz2 = (xyz.astype(np.float64) + sh).astype(np.float32)
    for kind in (K.KD_RBF, K.KD_GAUSSIAN, K.KD_LAPLACIAN):
        a, gap = K.covariance_kd(xyz, nbr, kind, sigma=0.8)
        b, _ = K.covariance_kd(xyz2, nbr, kind, sigma=0.8, origin=sh)
        m = gap >= 1e-2  # the normal is well defined; fp32 rounding of the shifted coordinates
        assert m.mean() > 0.9 and np.abs(a[m] - b[m]).max() < 1e-3


def test_degenerate_neighbourhoods():
    pts = np.repeat(np.array([[1.0, 2.0, 3.0]], np.float32), 10, axis=0)
    nbr = np.tile(np.arange(10, dtype=np.int32), (10, 1))
    plane, _ = K.covariance_kd(pts, nbr, K.KD_LAPLACIAN, sigma=1.0)
    assert np.array_equal(plane[0], [1, 0, 0, 1, 0, 1e-3])
    for reg in (1, 2):
        c, _ = K.covariance_kd(pts, nbr, K.KD_LAPLACIAN, sigma=1.0, reg=reg)
        assert np.array_equal(c[0], [1e-3, 0, 0, 1e-3, 0, 1e-3])


def test_hi_weights_in_unit_interval():
    rng = np.random.default_rng(9)
    for _ in range(200):
        x, y = rng.uniform(0, 10, 3), rng.uniform(0, 10, 3)
        w = K.kernel_eval(K.KD_HI, x, y)
        assert 0.0 <= w <= 1.0
