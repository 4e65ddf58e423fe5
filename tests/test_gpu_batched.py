"""Batched registration through the C ABI.

gicp_linearize_batched / gicp_align_batched partition every registration exactly
like the single calls, so each row / result must be BITWISE the single-call
result (which tests/test_gpu_parity.py pins to the oracle); one small
registration is also checked against the oracle directly. Registrations are
ragged (20000, 7777, 0 and 300 points) at different places on the track."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2308_07173_b200 as g  # noqa: E402

DEV = torch.device("cuda:0")
SIZES = [(0, 20000), (64, 7777), (128, 0), (200, 300)]


def D(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.fixture(scope="module")
def problem():
    mp = gen.racetrack_map(2_000_000, 1)
    im = g.build_index(D(mp), 0.5)
    _, _, cm = g.knn_cov_self(im, 20, 1e-3)
    g.attach_cov(im, cm)
    srcs, covs, Tt, T0 = [], [], [], []
    for i, n in SIZES:
        if n:
            sc, T, Tp = gen.config_c4_scan(i, n)
            sd = D(sc)
            isc = g.build_index(sd, 0.0)
            _, _, cs = g.knn_cov_self(isc, 20, 1e-3)
            isc.free()
        else:
            sc = np.zeros((0, 3), np.float32)
            cs = torch.zeros((0, 6), dtype=torch.float32, device=DEV)
            T, Tp = np.eye(4), np.eye(4)
        srcs.append(sc)
        covs.append(cs)
        Tt.append(T)
        T0.append(Tp)
    offs = np.concatenate([[0], np.cumsum([len(s) for s in srcs])]).astype(np.int64)
    src = D(np.concatenate(srcs).astype(np.float32))
    cov = torch.cat(covs).contiguous()
    yield dict(mp=mp, im=im, cm=cm, srcs=srcs, covs=covs, src=src, cov=cov, offs=offs, Tt=np.array(Tt),
               T0=np.array(T0))
    im.free()


@pytest.mark.parametrize("which", ["T0", "Tt"])
def test_linearize_batched_is_bitwise_the_single_calls(problem, which):
    p = problem
    Ts = p[which]
    piv = Ts[:, :3, 3]
    out, corr = g.linearize_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], Ts, 1.0, pivots=piv)
    out = out.cpu().numpy()
    corr = corr.cpu().numpy()
    for b in range(len(SIZES)):
        lo, hi = p["offs"][b], p["offs"][b + 1]
        if hi == lo:
            assert np.all(out[b] == 0.0)
            continue
        o1, c1 = g.linearize(p["src"][lo:hi], p["covs"][b], p["im"], p["cm"], Ts[b], 1.0, pivot=piv[b])
        assert np.array_equal(out[b], o1.cpu().numpy()), f"registration {b}"
        assert np.array_equal(corr[lo:hi], c1.cpu().numpy())
    # REUSE + ERROR_ONLY on the same correspondences
    c = torch.from_numpy(corr).to(DEV)
    oe, _ = g.linearize_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], Ts, 1.0, pivots=piv, corr=c,
                                reuse_corr=True, error_only=True)
    oe = oe.cpu().numpy()
    for b in range(len(SIZES)):
        lo, hi = p["offs"][b], p["offs"][b + 1]
        if hi == lo:
            continue
        o1, _ = g.linearize(p["src"][lo:hi], p["covs"][b], p["im"], p["cm"], Ts[b], 1.0, pivot=piv[b],
                            corr=c[lo:hi].clone(), reuse_corr=True, error_only=True)
        assert np.array_equal(oe[b], o1.cpu().numpy())


def test_linearize_batched_small_registration_vs_oracle(problem, orc):
    p = problem
    b = 3  # 300 points, brute force over the full 2M map in the oracle
    lo, hi = p["offs"][b], p["offs"][b + 1]
    Ts = p["T0"]
    out, corr = g.linearize_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], Ts, 1.0, pivots=Ts[:, :3, 3])
    o29, ab, ocorr = orc.linearize(p["srcs"][b], p["covs"][b].cpu().numpy(), p["mp"], p["cm"].cpu().numpy(), Ts[b],
                                   1.0, pivot=Ts[b, :3, 3])
    assert np.array_equal(corr.cpu().numpy()[lo:hi], ocorr)
    g29 = out.cpu().numpy()[b]
    assert g29[28] == o29[28]
    assert np.abs(g29[:21] - o29[:21]).max() <= 1e-4 * np.abs(o29[:21]).max()
    d = np.abs(g29[21:28] - o29[21:28])
    assert np.all((d <= 1e-4 * np.abs(o29[21:28])) | (d <= 1e-5 * ab[21:28]))


def test_align_batched_is_bitwise_the_single_aligns(problem):
    p = problem
    Ts, infos = g.align_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], p["T0"], allow_degenerate=True)
    for b in range(len(SIZES)):
        lo, hi = p["offs"][b], p["offs"][b + 1]
        if hi == lo:
            assert infos[b].inliers == 0 and not infos[b].converged
            continue
        T1, i1 = g.align(p["src"][lo:hi], p["covs"][b], p["im"], p["cm"], p["T0"][b])
        assert np.array_equal(Ts[b], T1), f"registration {b}"
        assert (infos[b].iterations, infos[b].converged, infos[b].error, infos[b].inliers) == \
            (i1.iterations, i1.converged, i1.error, i1.inliers)
        # moves toward the true pose (the along-track slide of a straight is weakly
        # constrained, so no tight recovery bar here; test_gpu_parity pins align)
        t_err = np.linalg.norm(T1[:3, 3] - p["Tt"][b][:3, 3])
        assert t_err < np.linalg.norm(p["T0"][b][:3, 3] - p["Tt"][b][:3, 3])
    with pytest.raises(g.GicpError):
        g.align_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], p["T0"])


def test_batched_argument_errors(problem):
    p = problem
    with pytest.raises(ValueError):
        g.linearize_batched(p["src"], p["cov"], [0, 5], p["im"], p["cm"], p["T0"][:1])
    bad = p["offs"].copy()
    bad[1], bad[2] = bad[2], bad[1]
    with pytest.raises(g.GicpError):
        g.linearize_batched(p["src"], p["cov"], bad, p["im"], p["cm"], p["T0"])


def test_align_batched_certificates_bitwise(problem, monkeypatch):
    """Correspondence certificates (R27) in the batched align: every
    registration bitwise the same with and without them (GICP_ALIGN_NOCACHE=1)."""
    p = problem
    Ta, ia = g.align_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], p["T0"], allow_degenerate=True)
    monkeypatch.setenv("GICP_ALIGN_NOCACHE", "1")
    Tb, ib = g.align_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], p["T0"], allow_degenerate=True)
    assert np.array_equal(np.asarray(Ta), np.asarray(Tb))
    assert [(i.iterations, i.converged, i.error, i.inliers) for i in ia] == \
        [(i.iterations, i.converged, i.error, i.inliers) for i in ib]


@pytest.mark.parametrize("single,coop", [(False, True), (False, False), (True, True)])
def test_split_evaluation_bitwise(problem, monkeypatch, single, coop):
    """The split evaluation (k_lin_cert -> k_lin_search -> k_lin_terms, used for
    launches of >= 1M points) and the fused k_linearize give bitwise the same
    aligns: forced on (GICP_LIN_SPLIT_MIN=0) against forced off; the unsettled
    points searched a warp per point (k_lin_search_coop) or per lane
    (GICP_LIN_COOP_MAX=0: k_lin_search<false>)."""
    p = problem
    monkeypatch.setenv("GICP_LIN_COOP_MAX", "16384" if coop else "0")
    def run():
        if single:
            b = int(np.argmax(np.diff(p["offs"])))
            lo, hi = p["offs"][b], p["offs"][b + 1]
            T, i = g.align(p["src"][lo:hi], p["covs"][b], p["im"], p["cm"], p["T0"][b])
            return [T], [i]
        return g.align_batched(p["src"], p["cov"], p["offs"], p["im"], p["cm"], p["T0"], allow_degenerate=True)
    monkeypatch.setenv("GICP_LIN_SPLIT_MIN", "0")
    Ta, ia = run()
    monkeypatch.setenv("GICP_LIN_SPLIT_MIN", str(1 << 40))
    Tb, ib = run()
    assert np.array_equal(np.asarray(Ta), np.asarray(Tb))
    assert [(i.iterations, i.converged, i.error, i.inliers) for i in ia] == \
        [(i.iterations, i.converged, i.error, i.inliers) for i in ib]
