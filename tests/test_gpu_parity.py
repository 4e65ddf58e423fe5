"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bars:
  kNN          nbr and d2 bitwise equal.
  covariance   |C_gpu - C_ref|max <= 1e-4 where the eigengap g >= 1e-2; elsewhere
               finite, symmetric, spectrum {eps, 1, 1} +- 1e-4.
  linearize    corr bitwise, inlier count equal, |dH|max <= 1e-4 |H|max,
               b/e: |d| <= 1e-4 |ref| or <= 1e-5 sum|term| (cancellation regime).
  align        |dt| <= 1e-3 m, angle <= 1e-4 rad on well-conditioned geometry.
"""
import math

import numpy as np
import pytest

import gen
from tests.conditioning import kappa_prime

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2308_07173_b200 as g  # noqa: E402

DEV = torch.device("cuda:0")


def D(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def H(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _full(c6):
    c6 = np.asarray(c6, np.float64)
    return np.stack([np.stack([c6[..., 0], c6[..., 1], c6[..., 2]], -1),
                     np.stack([c6[..., 1], c6[..., 3], c6[..., 4]], -1),
                     np.stack([c6[..., 2], c6[..., 4], c6[..., 5]], -1)], -2)


def assert_cov_parity(cov_gpu, cov_ref, gap, eps=1e-3, masked_frac_max=None):
    cov_gpu = np.asarray(cov_gpu, np.float64)
    assert np.all(np.isfinite(cov_gpu))
    m = gap >= 1e-2
    if m.any():
        err = np.abs(cov_gpu[m] - cov_ref[m]).max()
        assert err <= 1e-4, f"covariance parity {err}"
    if (~m).any():
        w = np.linalg.eigvalsh(_full(cov_gpu[~m]))
        assert np.abs(w - np.array([eps, 1, 1])).max() <= 1e-4
    if masked_frac_max is not None:
        # SURVEY §8 tolerances: report the masked fraction; < 1 % on the racetrack configs
        print(f"masked (gap < 1e-2) fraction {(~m).mean():.4%} of {m.size} rows")
        assert (~m).mean() <= masked_frac_max


# ---------------------------------------------------------------------------
# kNN
# ---------------------------------------------------------------------------

def test_lattice_worked_example(orc):
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lattice_knn.json")))
    L = gen.lattice(gold["side"])
    for cell in (0.7, 1.0, 2.5):
        idx = g.build_index(D(L), cell)
        nbr, d2 = g.knn(idx, D(np.array([gold["query"]], np.float32)), gold["k"])
        assert H(nbr)[0].tolist() == gold["nbr"]
        assert H(d2)[0].tolist() == gold["d2"]


@pytest.mark.parametrize("k", [1, 7, 20, 32])
@pytest.mark.parametrize("cell", [0.3, 1.0, 4.0])
def test_knn_uniform_external(orc, k, cell):
    tgt = gen.uniform_cloud(3000, 1, offset=(812.0, -377.0, 3.0))
    q = np.concatenate([gen.uniform_cloud(700, 2, -12, 12, offset=(812.0, -377.0, 3.0)),
                        np.array([[812.0 + 60, -377.0 - 45, 3.0 + 9]], np.float32)])  # one far query
    idx = g.build_index(D(tgt), cell)
    nbr, d2 = g.knn(idx, D(q), k)
    on, od = orc.knn(tgt, q, k)
    assert np.array_equal(H(nbr), on)
    assert np.array_equal(H(d2).view(np.uint32), od.view(np.uint32))


@pytest.mark.parametrize("k", [5, 16, 32])
def test_knn_self_quantised_ties(orc, k):
    # 1/8 m lattice: exact d2, frequent ties -> exercises the (d2, index) rule and
    # the tie re-search path
    p = gen.quantised_cloud(4000, 3, half=4.0)
    idx = g.build_index(D(p), 0.6)
    nbr, d2 = g.knn_self(idx, k)
    on, od = orc.knn(p, p, k)
    assert np.array_equal(H(nbr), on)
    assert np.array_equal(H(d2), od)
    nbr2, d22, cov = g.knn_cov_self(idx, k)
    assert np.array_equal(H(nbr2), on) and np.array_equal(H(d22), od)


def test_knn_duplicates_and_degenerate(orc):
    base = gen.uniform_cloud(300, 4, -2, 2)
    p = np.concatenate([base, np.repeat(base[:1], 40, 0), base[5:50]]).astype(np.float32)
    idx = g.build_index(D(p), 0.5)
    nbr, d2, cov = g.knn_cov_self(idx, 32)
    on, od = orc.knn(p, p, 32)
    assert np.array_equal(H(nbr), on) and np.array_equal(H(d2), od)
    oc, gap, _ = orc.covariance(p, on)
    assert_cov_parity(H(cov), oc, gap)
    # the duplicate block: all 32 neighbours identical -> diag(1, 1, eps)
    c = H(cov)[300]
    assert np.allclose(c, [1, 0, 0, 1, 0, 1e-3], atol=1e-7)


@pytest.mark.parametrize("k", [10, 20])
def test_knn_cov_racetrack_subset(orc, k):
    mp = gen.racetrack_map(200_000, 5)
    idx = g.build_index(D(mp), 1.15 * math.sqrt(k / (math.pi * 3.1)))
    nbr, d2, cov = g.knn_cov_self(idx, k)
    nbr2, d22 = g.knn_self(idx, k)
    rng = np.random.default_rng(0)
    rows = rng.choice(len(mp), 3000, replace=False)
    on, od = orc.knn(mp, mp[rows], k)
    hn, hd = H(nbr), H(d2)
    assert np.array_equal(hn[rows], on) and np.array_equal(hd[rows], od)
    assert np.array_equal(H(nbr2), hn) and np.array_equal(H(d22), hd)
    oc, gap, _ = orc.covariance(mp, on)
    assert_cov_parity(H(cov)[rows], oc, gap, masked_frac_max=0.01)
    # the standalone covariance kernel on the same neighbour table
    cov2 = g.covariances(D(mp), D(on))
    assert_cov_parity(H(cov2), oc, gap)


def test_knn_scan_external_and_auto_cell(orc):
    sc, T = gen.scan(30_000, 380.0, 500)
    idx = g.build_index(D(sc), 0.0)      # automatic cell size
    assert idx.cell_size > 0
    q = sc[::7]
    nbr, d2 = g.knn(idx, D(q), 20)
    on, od = orc.knn(sc, q, 20)
    assert np.array_equal(H(nbr), on) and np.array_equal(H(d2), od)


def test_knn_edge_cases(orc):
    p = gen.uniform_cloud(50, 9)
    idx = g.build_index(D(p), 1.0)
    with pytest.raises(g.GicpError) as e:
        g.knn(idx, D(p), 51)
    assert e.value.code == g.EK
    with pytest.raises(g.GicpError):
        g.knn(idx, D(p), 33)
    nbr, d2 = g.knn(idx, D(p[:0]), 3)
    assert nbr.shape == (0, 3)
    one = g.build_index(D(p[:1]), 1.0)
    nbr, d2 = g.knn(one, D(p), 1)
    assert np.all(H(nbr) == 0)
    # a query far outside the grid (overflow -> brute-force path) and a NaN query
    q = np.array([[5000.0, -3000.0, 40.0], [np.nan, 0, 0], [1.0, 2.0, 3.0]], np.float32)
    nbr, d2 = g.knn(idx, D(q), 4)
    on, od = orc.knn(p, q[[0, 2]], 4)
    hn, hd = H(nbr), H(d2)
    assert np.array_equal(hn[[0, 2]], on) and np.array_equal(hd[[0, 2]], od)
    assert np.all(hn[1] == -1) and np.all(np.isinf(hd[1]))
    bad = p.copy()
    bad[3, 2] = np.inf
    with pytest.raises(g.GicpError) as e:
        g.build_index(D(bad), 1.0)
    assert e.value.code == g.EINVAL
    with pytest.raises(g.GicpError) as e:
        g.build_index(D(np.array([[0, 0, 0], [1e6, 1e6, 0]], np.float32)), 1e-3)
    assert e.value.code == g.ERANGE


# ---------------------------------------------------------------------------
# linearize / align
# ---------------------------------------------------------------------------

def _covs_oracle(orc, pts, k):
    nbr, _ = orc.knn(pts, pts, k)
    c, gap, _ = orc.covariance(pts, nbr)
    return c.astype(np.float32)


def assert_lin_parity(g29, o29, ab):
    assert g29[28] == o29[28], "inlier count"
    Hs = np.abs(o29[:21]).max()
    assert np.abs(g29[:21] - o29[:21]).max() <= 1e-4 * Hs
    for c in range(21, 28):
        d = abs(g29[c] - o29[c])
        assert d <= 1e-4 * abs(o29[c]) or d <= 1e-5 * ab[c], (c, g29[c], o29[c], ab[c])


@pytest.mark.parametrize("variant", ["copy", "resample", "noisy"])
def test_linearize_c1(orc, variant):
    src, tgt, T_true, T0 = gen.config_c1(exact_copy=(variant == "copy"), sigma=0.002 if variant == "noisy" else 0.0)
    cs, ct = _covs_oracle(orc, src, 10), _covs_oracle(orc, tgt, 10)
    idx = g.build_index(D(tgt), 0.6)
    for T in (T0, T_true, T_true @ gen.perturbation(0.05, 0.5, 3)):
        out, corr = g.linearize(D(src), D(cs), idx, D(ct), T, 1.0)
        o29, ab, ocorr = orc.linearize(src, cs, tgt, ct, T, 1.0)
        assert np.array_equal(H(corr), ocorr)
        assert_lin_parity(H(out), o29, ab)
        # with a rotation pivot (gicp_align's parametrisation)
        c = T[:3, 3] + np.array([0.3, -0.2, 0.1])
        outp, _ = g.linearize(D(src), D(cs), idx, D(ct), T, 1.0, pivot=c)
        op29, abp, _ = orc.linearize(src, cs, tgt, ct, T, 1.0, pivot=c)
        assert_lin_parity(H(outp), op29, abp)
        # REUSE_CORR and ERROR_ONLY paths
        out2, _ = g.linearize(D(src), D(cs), idx, D(ct), T, 1.0, corr=corr, reuse_corr=True, error_only=True)
        h2 = H(out2)
        assert h2[28] == o29[28] and abs(h2[27] - o29[27]) <= 1e-4 * abs(o29[27]) + 1e-5 * ab[27]


def test_linearize_deterministic_and_empty(orc):
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    cs, ct = _covs_oracle(orc, src, 10), _covs_oracle(orc, tgt, 10)
    idx = g.build_index(D(tgt), 0.6)
    a, _ = g.linearize(D(src), D(cs), idx, D(ct), T0, 1.0)
    a = H(a).copy()
    for _ in range(3):
        b, _ = g.linearize(D(src), D(cs), idx, D(ct), T0, 1.0)
        assert np.array_equal(H(b), a)
    e, _ = g.linearize(D(src[:0]), D(cs[:0]), idx, D(ct), T0, 1.0)
    assert np.all(H(e) == 0)


def test_attached_covariances_give_identical_results(orc):
    # gicp_index_attach_cov is a layout optimisation only: bitwise identical output
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    cs, ct = _covs_oracle(orc, src, 10), _covs_oracle(orc, tgt, 10)
    idx = g.build_index(D(tgt), 0.6)
    ctd = D(ct)
    a, ca = g.linearize(D(src), D(cs), idx, ctd, T0, 1.0)
    a, ca = H(a).copy(), H(ca).copy()
    g.attach_cov(idx, ctd)
    b, cb = g.linearize(D(src), D(cs), idx, ctd, T0, 1.0)
    assert np.array_equal(H(b), a) and np.array_equal(H(cb), ca)
    T1, i1 = g.align(D(src), D(cs), idx, ctd, T0)
    ref = orc.align(src, cs, tgt, ct, T0)
    dt, dr = _pose_err(T1, ref["T"])
    assert dt <= 1e-3 and dr <= 1e-4


def test_linearize_c2_scan_to_scan(orc):
    src, tgt, T_rel, T0 = gen.config_c2(30_000)
    cs, ct = _covs_oracle(orc, src, 20), _covs_oracle(orc, tgt, 20)
    idx = g.build_index(D(tgt), 0.0)
    for T in (T0, T_rel):
        out, corr = g.linearize(D(src), D(cs), idx, D(ct), T, 1.0, pivot=T[:3, 3])
        o29, ab, ocorr = orc.linearize(src, cs, tgt, ct, T, 1.0, pivot=T[:3, 3])
        assert np.array_equal(H(corr), ocorr)
        assert_lin_parity(H(out), o29, ab)


def _pose_err(T, Tr):
    dt = np.linalg.norm(T[:3, 3] - Tr[:3, 3])
    c = (np.trace(T[:3, :3] @ Tr[:3, :3].T) - 1) / 2
    return dt, math.acos(max(-1.0, min(1.0, c)))


@pytest.mark.parametrize("variant", ["copy", "resample", "noisy"])
def test_align_c1(orc, variant):
    src, tgt, T_true, T0 = gen.config_c1(exact_copy=(variant == "copy"), sigma=0.002 if variant == "noisy" else 0.0)
    cs, ct = _covs_oracle(orc, src, 10), _covs_oracle(orc, tgt, 10)
    idx = g.build_index(D(tgt), 0.6)
    T, info = g.align(D(src), D(cs), idx, D(ct), T0)
    ref = orc.align(src, cs, tgt, ct, T0)
    dt, dr = _pose_err(T, ref["T"])
    assert info.converged and ref["converged"]
    assert dt <= 1e-3 and dr <= 1e-4
    dt2, _ = _pose_err(T, T_true)
    assert dt2 < 0.02


def test_align_c2(orc):
    src, tgt, T_rel, T0 = gen.config_c2(30_000)
    cs, ct = _covs_oracle(orc, src, 20), _covs_oracle(orc, tgt, 20)
    idx = g.build_index(D(tgt), 0.0)
    T, info = g.align(D(src), D(cs), idx, D(ct), T0)
    ref = orc.align(src, cs, tgt, ct, T0)
    assert info.converged and ref["converged"]
    o29, _, corr = orc.linearize(src, cs, tgt, ct, ref["T"], 1.0)
    pw = src.astype(np.float64) @ ref["T"][:3, :3].T + ref["T"][:3, 3]
    kp = kappa_prime(o29, pw[corr >= 0])
    if kp >= 5e-3:
        dt, dr = _pose_err(T, ref["T"])
        assert dt <= 1e-3 and dr <= 1e-4
    else:
        # Below the eps floor (SURVEY.md §8(c) tolerances, align) pose parity is not
        # asserted: both LM results must reach costs within 1e-4 relative of each other.
        # Gauss-Newton takes no accept/reject decisions: its poses must agree too.
        e_gpu = orc.linearize(src, cs, tgt, ct, T, 1.0)[0][27]
        e_ref = o29[27]
        print(f"C2 eps floor: kappa'={kp:.3g} e_gpu={e_gpu:.9g} e_ref={e_ref:.9g} rel={(e_gpu - e_ref) / e_ref:.3g}")
        assert abs(e_gpu - e_ref) <= 1e-4 * e_ref, (kp, e_gpu, e_ref)
        Tg, ig = g.align(D(src), D(cs), idx, D(ct), T0, lm=False)
        rg = orc.align(src, cs, tgt, ct, T0, lm=False)
        dt, dr = _pose_err(Tg, rg["T"])
        assert dt <= 1e-3 and dr <= 1e-4, (kp, dt, dr)


def test_align_degenerate(orc):
    p = gen.corner_scene(11)
    c = _covs_oracle(orc, p, 10)
    idx = g.build_index(D(p), 0.6)
    far = (p + np.array([100.0, 0, 0], np.float32)).astype(np.float32)
    with pytest.raises(g.GicpError) as e:
        g.align(D(far), D(c), idx, D(c), np.eye(4))
    assert e.value.code == g.EDEGENERATE


# ---------------------------------------------------------------------------
# full-size C3 in the bench's launch configuration (sampled rows)
# ---------------------------------------------------------------------------

def test_c3_fullsize_sampled(orc):
    sc, mp, T_true, T0 = gen.config_c3()
    idx = g.build_index(D(mp), 0.5)
    nbr, d2, cov = g.knn_cov_self(idx, 20)
    rng = np.random.default_rng(77)
    rows = rng.choice(len(mp), 1500, replace=False)
    on, od = orc.knn(mp, mp[rows], 20)
    hn, hd, hc = H(nbr), H(d2), H(cov)
    assert np.array_equal(hn[rows], on) and np.array_equal(hd[rows], od)
    oc, gap, _ = orc.covariance(mp, on)
    assert_cov_parity(hc[rows], oc, gap, masked_frac_max=0.01)
    # linearize of a source subsample against the full map; covariances are
    # generic SPD inputs from gen (no oracle input comes from the CUDA path)
    sub = rng.choice(len(sc), 1500, replace=False)
    src = np.ascontiguousarray(sc[sub])
    cs = gen.random_covariances(len(src), 1)
    ct = gen.random_covariances(len(mp), 2)
    out, corr = g.linearize(D(src), D(cs), idx, D(ct), T0, 1.0, pivot=T0[:3, 3])
    o29, ab, ocorr = orc.linearize(src, cs, mp, ct, T0, 1.0, pivot=T0[:3, 3])
    assert np.array_equal(H(corr), ocorr)
    assert_lin_parity(H(out), o29, ab)


def test_c5_stress_sampled(orc):
    """C5: 20M-point multi-lap map, 1M external queries (10 scans in the map
    frame), k=32 kNN + covariance of the neighbour sets; cell 0.2 m (~1.1 r_32 at
    10x the C3 density). Sampled rows against the oracle (brute force over the
    full 20M), every row checked for the properties that hold at any size."""
    mp, q = gen.config_c5()
    mpd = D(mp)
    idx = g.build_index(mpd, 0.2)
    nbr, d2 = g.knn(idx, D(q), 32)
    cov = g.covariances(mpd, nbr, 1e-3)
    hn, hd, hc = H(nbr), H(d2), H(cov)
    # properties, all 1M rows: indices in range, rows ascending by (d2, idx)
    assert hn.min() >= 0 and hn.max() < len(mp)
    assert np.all(np.isfinite(hd))
    dd = np.diff(hd, axis=1)
    assert np.all((dd > 0) | ((dd == 0) & (np.diff(hn, axis=1) > 0)))
    rng = np.random.default_rng(78)
    rows = np.concatenate([[0, len(q) - 1], rng.choice(len(q), 254, replace=False)])
    on, od = orc.knn(mp, q[rows], 32)
    assert np.array_equal(hn[rows], on) and np.array_equal(hd[rows], od)
    oc, gap, _ = orc.covariance(mp, on)
    assert_cov_parity(hc[rows], oc, gap, masked_frac_max=0.01)
    idx.free()


# ---------------------------------------------------------------------------
# kernel-descriptor covariances: every Table I kernel x every
# regularisation against the oracle on a racetrack section (oracle neighbours)
@pytest.mark.parametrize("kernel,sigma", [("uniform", 1.0), ("rbf", 4.0), ("gaussian", 0.3), ("polynomial", 1.0),
                                          ("hi", 1.0), ("laplacian", 0.5)])
@pytest.mark.parametrize("reg", ["plane", "min_eig", "normalized_min_eig"])
def test_covariances_kd_vs_oracle(orc, kernel, sigma, reg):
    mp = gen.racetrack_map(2_000_000, 1)
    sel = np.nonzero((np.abs(mp[:, 0] - 150.0) < 25.0) & (mp[:, 1] > 0))[0][:20000]
    xyz = np.ascontiguousarray(mp[sel])
    nbr, _ = orc.knn(xyz, xyz, 20)
    o = xyz.min(axis=0).astype(np.float64)
    kinds = dict(uniform=0, rbf=1, gaussian=2, polynomial=3, hi=4, laplacian=5)
    regs = dict(plane=0, min_eig=1, normalized_min_eig=2)
    ref, gap = orc.covariance_kd(xyz, nbr, kinds[kernel], sigma=sigma, alpha=0.01, c=1.0, d=2, origin=o,
                                 reg=regs[reg])
    got = H(g.covariances_kd(D(xyz), D(nbr), kernel, sigma=sigma, alpha=0.01, c=1.0, degree=2, origin=o, reg=reg))
    assert np.all(np.isfinite(got))
    m = gap >= 1e-2
    assert m.mean() > 0.95
    scale = np.abs(ref[m]).max(axis=1, keepdims=True)
    assert (np.abs(got[m] - ref[m]) / np.maximum(scale, 1e-12)).max() <= 1e-4


def test_covariances_kd_external_queries_and_errors(orc):
    xyz = gen.uniform_cloud(5000, 11, lo=-3.0, hi=3.0)
    q = gen.uniform_cloud(700, 12, lo=-3.0, hi=3.0)
    nbr, _ = orc.knn(xyz, q, 16)
    ref, gap = orc.covariance_kd(xyz, nbr, 5, q=q, sigma=0.7)
    got = H(g.covariances_kd(D(xyz), D(nbr), "laplacian", sigma=0.7, q=D(q)))
    m = gap >= 1e-2
    assert np.abs(got[m] - ref[m]).max() <= 1e-4
    with pytest.raises(g.GicpError):
        g.covariances_kd(D(xyz), D(nbr), "laplacian", sigma=0.0, q=D(q))
    with pytest.raises(g.GicpError):
        g.covariances_kd(D(xyz), D(nbr), "polynomial", degree=0, q=D(q))


# ---------------------------------------------------------------------------
# correspondence certificates (reading R27): gicp_align skips the NN
# search for a point whose search point moved less than the certified radius of
# its previous search. The search is exact, so the alignment must be BITWISE the
# one that searches every point every time (GICP_ALIGN_NOCACHE=1).
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", ["c3", "c2"])
def test_align_certificates_bitwise(monkeypatch, cfg):
    if cfg == "c3":  # the bench's workload and launch configuration
        sc, mp, _, T0 = gen.config_c3()
        imap = g.build_index(D(mp), 0.5)
        k = 20
    else:
        sc, mp, _, T0 = gen.config_c2(30_000)
        imap = g.build_index(D(mp), 0.0)
        k = 20
    _, _, cov_map = g.knn_cov_self(imap, k, 1e-3, with_nbr=True)
    g.attach_cov(imap, cov_map)
    iscan = g.build_index(D(sc), 0.0)
    _, _, cov_scan = g.knn_cov_self(iscan, k, 1e-3, with_nbr=True)
    res = {}
    for mode in ("cache", "nocache"):
        if mode == "nocache":
            monkeypatch.setenv("GICP_ALIGN_NOCACHE", "1")
        else:
            monkeypatch.delenv("GICP_ALIGN_NOCACHE", raising=False)
        for lm in (True, False):
            T, info = g.align(D(sc), cov_scan, imap, cov_map, T0, lm=lm)
            res[(mode, lm)] = (T, info)
    for lm in (True, False):
        Ta, ia = res[("cache", lm)]
        Tb, ib = res[("nocache", lm)]
        assert np.array_equal(Ta, Tb), (lm, Ta, Tb)
        assert ia == ib, (lm, ia, ib)
