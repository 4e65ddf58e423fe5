"""Pins for oracle O4 (host LM align) against known transforms.

Paper: "T = argmin_T sum_i d_i^T (...) d_i" (PAPER.md eq_trans_likelihood
l.396-402); the optimiser is DESIGN.md reading R13 (LM, left perturbation).
"""
import math

import numpy as np
import pytest

import gen


def _covs(orc, pts, k=10):
    nbr, _ = orc.knn(pts, pts, k)
    return orc.covariance(pts, nbr)[0].astype(np.float32)


def _pose_err(T, Tref):
    dt = np.linalg.norm(T[:3, 3] - Tref[:3, 3])
    c = (np.trace(T[:3, :3] @ Tref[:3, :3].T) - 1) / 2
    return dt, math.acos(max(-1.0, min(1.0, c)))


def test_identical_clouds_identity_guess(orc):
    # S:293 / S:300: register(A, A, I) = I (within 1e-9), cost ~ 0, 1-2 iterations
    p = gen.corner_scene(11, 0.002)
    c = _covs(orc, p)
    r = orc.align(p, c, p, c, np.eye(4))
    assert r["converged"] and r["iterations"] <= 2
    assert np.allclose(r["T"], np.eye(4), atol=1e-9)
    assert r["error"] == 0.0


def test_exact_copy_recovers_T_true(orc):
    src, tgt, T_true, T0 = gen.config_c1(exact_copy=True)
    r = orc.align(src, _covs(orc, src), tgt, _covs(orc, tgt), T0)
    dt, dr = _pose_err(r["T"], T_true)
    assert r["converged"]
    assert dt < 2e-6 and dr < 2e-6


def test_independent_resample_recovery(orc):
    for sigma in (0.0, 0.002):
        src, tgt, T_true, T0 = gen.config_c1(sigma=sigma)
        r = orc.align(src, _covs(orc, src), tgt, _covs(orc, tgt), T0)
        dt, dr = _pose_err(r["T"], T_true)
        assert r["converged"]
        assert dt < 0.02 and dr < math.radians(0.2)


def test_spec_shift_recovered(orc):
    # cloud vs copy shifted by (1, 0, 0), identity guess -> within 0.05 m
    tgt = gen.corner_scene(21, 0.002)
    src = (tgt - np.array([1.0, 0.0, 0.0], np.float32)).astype(np.float32)
    r = orc.align(src, _covs(orc, src), tgt, _covs(orc, tgt), np.eye(4), max_corr_dist=2.0)
    assert abs(r["T"][0, 3] - 1.0) < 0.05 and np.linalg.norm(r["T"][1:3, 3]) < 0.05


def test_gauss_newton_variant_agrees(orc):
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    cs, ct = _covs(orc, src), _covs(orc, tgt)
    a = orc.align(src, cs, tgt, ct, T0, lm=True)
    b = orc.align(src, cs, tgt, ct, T0, lm=False)
    dt, dr = _pose_err(a["T"], b["T"])
    assert dt < 1e-4 and dr < 1e-5


def test_degenerate_raises(orc):
    # fewer than 6 gated correspondences -> NotEnoughCorrespondences
    p = gen.corner_scene(11)
    c = _covs(orc, p)
    far = (p + np.array([100.0, 0, 0], np.float32)).astype(np.float32)
    with pytest.raises(orc.OracleError) as e:
        orc.align(far, c, p, c, np.eye(4))
    assert e.value.code == orc.EDEGENERATE
