"""Pins of the voxelized-GICP oracle (O7 linearize_vgicp, O8 align_vgicp;
PAPER.md l.419, readings R22-R23): a one-voxel
closed form (numpy solve), the reduction to the pinned GICP oracle O3 when every
voxel holds one point, the pair count, and recovery of a known transform."""
import numpy as np
import pytest

import gen

orc = pytest.importorskip("oracle")


def test_single_voxel_closed_form():
    rng = np.random.default_rng(4)
    tgt = (np.array([2.05, 3.05, 4.05]) + rng.uniform(0.0, 0.9, (7, 3))).astype(np.float32)  # one 1-m voxel
    tgt[0] = [2.01, 3.01, 4.01]  # the bbox minimum: voxel (0,0,0) holds all seven
    ct = gen.random_covariances(7, 5)
    src = np.array([[2.6, 3.5, 4.3]], np.float32)
    cs = gen.random_covariances(1, 6)
    T = np.eye(4)
    out, _, _ = orc.linearize_vgicp(src, cs, tgt, ct, T, res=1.0, mode=1)
    full = lambda c: np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]], np.float64)  # noqa: E731
    mu = tgt.astype(np.float64).mean(axis=0)
    S = np.mean([full(c.astype(np.float64)) for c in ct.astype(np.float32)], axis=0)
    A = S + full(cs[0].astype(np.float32).astype(np.float64))
    d = mu - src[0].astype(np.float64)
    e = 7.0 * d @ np.linalg.solve(A, d)
    assert out[28] == 1.0
    assert out[27] == pytest.approx(e, rel=1e-12)
    # b's translation block: J = [skew(p') | -I] -> b_v = -N M d
    assert np.allclose(out[24:27], -7.0 * np.linalg.solve(A, d), rtol=1e-12, atol=0)


def test_one_point_per_voxel_reduces_to_gicp():
    """Target on a lattice of spacing 2 x res: every voxel holds one point, its mean
    is the point and its covariance the point's, N = 1 -- so mode 1 is GICP with
    the correspondence 'the target point in my voxel' (O3 with REUSE_CORR)."""
    g = np.stack(np.meshgrid(np.arange(12), np.arange(12), np.arange(3), indexing="ij"), -1).reshape(-1, 3)
    tgt = (g * 2.0 + 0.25).astype(np.float32)
    ct = gen.random_covariances(len(tgt), 7)
    rng = np.random.default_rng(8)
    src = (tgt[rng.choice(len(tgt), 150, replace=False)] + rng.uniform(0.15, 0.6, (150, 3))).astype(np.float32)
    cs = gen.random_covariances(150, 9)
    T = gen.make_T(gen.euler_to_R(0.001, -0.002, 0.002), [0.05, -0.04, 0.02])
    out, _, _ = orc.linearize_vgicp(src, cs, tgt, ct, T, res=1.0, mode=1, pivot=[1.0, 2.0, 3.0])
    # the correspondence: the lattice point whose voxel holds fl32(T p)
    o = tgt.min(axis=0)
    pp = src.astype(np.float64) @ T[:3, :3].T + T[:3, 3]
    cs_ = np.floor(((pp.astype(np.float32) - o).astype(np.float32) * np.float32(1.0)).astype(np.float32))
    ct_ = np.floor(((tgt - o).astype(np.float32)).astype(np.float32))
    lut = {tuple(c): j for j, c in enumerate(ct_.astype(np.int64))}
    corr = np.array([lut.get(tuple(c), -1) for c in cs_.astype(np.int64)], np.int32)
    assert (corr >= 0).sum() == out[28] > 100
    ref, _, _ = orc.linearize(src, cs, tgt, ct, T, 1.0, corr=corr, pivot=[1.0, 2.0, 3.0])
    assert np.array_equal(out, ref)


def test_pair_counts_by_mode():
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    cs = gen.random_covariances(len(src), 1)
    ct = gen.random_covariances(len(tgt), 2)
    n = [orc.linearize_vgicp(src, cs, tgt, ct, T_true, res=1.0, mode=m)[0][28] for m in (1, 7, 27)]
    assert 0 < n[0] <= len(src) and n[0] < n[1] < n[2] <= 27 * len(src)
    # REUSE with the returned base voxels reproduces the evaluation exactly
    o1, _, base = orc.linearize_vgicp(src, cs, tgt, ct, T0, res=1.0, mode=7)
    o2, _, _ = orc.linearize_vgicp(src, cs, tgt, ct, T0, res=1.0, mode=7, base=base)
    assert np.array_equal(o1, o2)


def test_align_vgicp_recovers_the_corner():
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.0)
    ns, _ = orc.knn(src, src, 10)
    nt, _ = orc.knn(tgt, tgt, 10)
    cs = orc.covariance(src, ns)[0]
    ct = orc.covariance(tgt, nt)[0]
    r = orc.align_vgicp(src, cs, tgt, ct, T0, res=0.5, mode=27)
    assert r["converged"]
    assert np.linalg.norm(r["T"][:3, 3] - T_true[:3, 3]) < 0.02
