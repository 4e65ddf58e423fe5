"""GPU parity on the fixtures that pin the oracle's easily-mistaken parts
(tests/test_oracle_pins_geometry.py), the bench's own alignment (C3) against O4,
and all rows of a 200k-point racetrack kNN.

Bars as in tests/test_gpu_parity.py.
"""
import math

import numpy as np
import pytest

import gen
from tests.conditioning import kappa_prime
from tests.test_oracle_pins_geometry import EPS, _cov6, _orthonormal_pairs, _plane, _rz

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2308_07173_b200 as g  # noqa: E402
from tests.test_gpu_parity import D, H, _pose_err, assert_cov_parity, assert_lin_parity  # noqa: E402


def test_linearize_rotated_anisotropic_gpu(orc):
    # the perpendicular-planes fixture: e against the geometric closed form and the oracle
    rng = np.random.default_rng(7)
    N = 64
    R = gen.euler_to_R(0.3, -0.2, 1.1)
    t = np.array([1.5, -2.0, 0.25])
    T = gen.make_T(R, t)
    src = (rng.uniform(-20, 20, size=(N, 3))).astype(np.float32)
    pp = src.astype(np.float64) @ R.T + t
    tgt = (pp + rng.uniform(-0.2, 0.2, size=(N, 3))).astype(np.float32)
    n, m = _orthonormal_pairs(rng, N)
    cq = np.stack([_cov6(_plane(n[i])) for i in range(N)])
    cp = np.stack([_cov6(_plane(R.T @ m[i])) for i in range(N)])
    idx = g.build_index(D(tgt), 1.0)
    for piv in (None, t + np.array([0.5, 0.25, -1.0])):
        out, corr = g.linearize(D(src), D(cp), idx, D(cq), T, 1.0, pivot=piv)
        o29, ab, ocorr = orc.linearize(src, cp, tgt, cq, T, 1.0, pivot=piv)
        assert np.array_equal(H(corr), ocorr) and np.array_equal(ocorr, np.arange(N))
        g29 = H(out)
        assert_lin_parity(g29, o29, ab)
    d = tgt.astype(np.float64) - pp
    x = np.cross(m, n)
    e_ref = (((d * m).sum(1) ** 2 + (d * n).sum(1) ** 2) / (1 + EPS) + (d * x).sum(1) ** 2 / 2).sum()
    assert math.isclose(g29[27], e_ref, rel_tol=2e-4)


def test_linearize_rotated_single_gpu(orc):
    R = _rz(30.0)
    T = np.eye(4)
    T[:3, :3] = R
    p = np.array([[2.0, 1.0, 0.5]], np.float32)
    pp = R @ p[0].astype(np.float64)
    q = (pp + np.array([0.125, -0.25, 0.0625])).astype(np.float32)[None]
    cs = _cov6(np.diag([1.0, EPS, 1.0]))[None]
    cq = _cov6(np.diag([1.0, 1.0, EPS]))[None]
    idx = g.build_index(D(q), 1.0)
    out, corr = g.linearize(D(p), D(cs), idx, D(cq), T, 2.0)
    o29, ab, _ = orc.linearize(p, cs, q, cq, T, 2.0)
    g29 = H(out)
    assert_lin_parity(g29, o29, ab)
    d = q[0].astype(np.float64) - pp
    u = np.array([-0.5, math.sqrt(3) / 2, 0.0])
    w = np.array([math.sqrt(3) / 2, 0.5, 0.0])
    e_ref = (d @ u) ** 2 / (1 + EPS) + (d @ w) ** 2 / 2 + d[2] ** 2 / (1 + EPS)
    assert math.isclose(g29[27], e_ref, rel_tol=1e-5)


@pytest.mark.parametrize("r", [0.5, 0.75])
@pytest.mark.parametrize("cell", [0.3, 1.0, 4.0])
def test_gate_is_strict_at_exactly_r_gpu(orc, r, cell):
    gr = np.arange(0, 12, 4.0)
    tgt = np.stack(np.meshgrid(gr, gr, gr, indexing="ij"), -1).reshape(-1, 3).astype(np.float32)
    offs = np.array([[r, 0, 0], [0, -r, 0], [0, 0, r], [r / 2, 0, 0], [0, r / 2, r / 4],
                     [-r, 0, 0], [0, 0, -r / 2]], np.float32)
    src = (tgt[13] + offs).astype(np.float32)
    cov = np.tile(_cov6(np.eye(3)), (len(tgt), 1))
    idx = g.build_index(D(tgt), cell)
    out, corr = g.linearize(D(src), D(cov[:len(src)]), idx, D(cov), np.eye(4), r)
    o29, ab, ocorr = orc.linearize(src, cov[:len(src)], tgt, cov, np.eye(4), r)
    assert np.array_equal(H(corr), ocorr)
    assert H(out)[28] == 3 == o29[28]
    assert_lin_parity(H(out), o29, ab)


# ---------------------------------------------------------------------------
# C3 (the bench's workload): align pose parity against O4
# ---------------------------------------------------------------------------

def _c3_cropped(n_sub=3000, seed=5, margin=4.0):
    """A seeded scan subsample of C3 and the map cropped EXACTLY to the subsample's
    bounding box at T0 plus `margin` (kept in original order, so index ties resolve
    alike): a map point outside the crop can be the 1-NN of a search point only if the
    point moved more than margin - r from its T0 position, which the test checks."""
    sc, mp, T_true, T0 = gen.config_c3()
    rng = np.random.default_rng(seed)
    sub = np.sort(rng.choice(len(sc), n_sub, replace=False))
    src = np.ascontiguousarray(sc[sub])
    pw = src.astype(np.float64) @ T0[:3, :3].T + T0[:3, 3]
    lo, hi = pw.min(0) - margin, pw.max(0) + margin
    inb = np.all((mp >= lo) & (mp <= hi), axis=1)
    lo2, hi2 = lo - 1.5, hi + 1.5
    inb2 = np.all((mp >= lo2) & (mp <= hi2), axis=1)
    return sc, mp, src, sub, inb, inb2, T_true, T0


def test_align_c3_vs_oracle_cropped(orc):
    sc, mp, src, sub, inb, inb2, T_true, T0 = _c3_cropped()
    crop, crop2 = np.ascontiguousarray(mp[inb]), np.ascontiguousarray(mp[inb2])
    # covariance INPUTS (both sides get the same): oracle kNN(k=20) + O2
    nb_c, _ = orc.knn(crop2, crop, 20)
    ct_crop = orc.covariance(crop2, nb_c)[0].astype(np.float32)
    nb_s, _ = orc.knn(sc, src, 20)
    cs = orc.covariance(sc, nb_s)[0].astype(np.float32)
    ct_full = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(mp), 1))
    ct_full[inb] = ct_crop
    imap = g.build_index(D(mp), 0.5)           # the bench's map index
    ctd = D(ct_full)
    g.attach_cov(imap, ctd)
    ref = orc.align(src, cs, crop, ct_crop, T0)
    T, info = g.align(D(src), D(cs), imap, ctd, T0)
    assert ref["converged"] and info.converged
    # the crop argument: no subsample point moved farther than margin - r from T0
    moved = np.linalg.norm((src.astype(np.float64) @ (ref["T"][:3, :3] - T0[:3, :3]).T
                            + (ref["T"][:3, 3] - T0[:3, 3])), axis=1).max()
    assert moved < 4.0 - 1.0 - 0.5
    o29, _, corr = orc.linearize(src, cs, crop, ct_crop, ref["T"], 1.0)     # J about the origin
    pw = src.astype(np.float64) @ ref["T"][:3, :3].T + ref["T"][:3, 3]
    kp = kappa_prime(o29, pw[corr >= 0])
    dt, dr = _pose_err(T, ref["T"])
    print(f"C3 cropped align: kappa'={kp:.3g} oracle it={ref['iterations']} gpu it={info.iterations} "
          f"dt={dt:.3g} m dr={dr:.3g} rad, |t - t_true|={np.linalg.norm(T[:3, 3] - T_true[:3, 3]):.3g}")
    # kappa' sits near the eps floor on C3 (the along-track slide, ~2.3e-3 here), where
    # SURVEY §8(c) only asks for equal costs; both runs take the same LM steps, so the
    # pose bar is asserted anyway (measured: 1.5e-8 m, 3.7e-8 rad)
    assert dt <= 1e-3 and dr <= 1e-4
    # the linearisation at the oracle's optimum, against the full map on the GPU
    out, gcorr = g.linearize(D(src), D(cs), imap, ctd, ref["T"], 1.0, pivot=ref["T"][:3, 3])
    hc = H(gcorr)
    crop_ids = np.nonzero(inb)[0]
    assert np.array_equal(hc >= 0, corr >= 0)
    assert np.array_equal(hc[hc >= 0], crop_ids[corr[corr >= 0]])


# ---------------------------------------------------------------------------
# every row of a 200k racetrack self-kNN + covariance
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("k", [10, 20])
def test_knn_cov_racetrack_all_rows(orc, k):
    mp = gen.racetrack_map(200_000, 5)
    idx = g.build_index(D(mp), 1.15 * math.sqrt(k / (math.pi * 3.1)))
    nbr, d2, cov = g.knn_cov_self(idx, k)
    on, od = orc.knn(mp, mp, k)
    hn, hd = H(nbr), H(d2)
    assert np.array_equal(hn, on)
    assert np.array_equal(hd.view(np.uint32), od.view(np.uint32))
    oc, gap, _ = orc.covariance(mp, on)
    masked = float((gap < 1e-2).mean())
    print(f"200k racetrack k={k}: masked (gap < 1e-2) fraction {masked:.4%}")
    assert_cov_parity(H(cov), oc, gap, masked_frac_max=0.01)
