"""Voxelized GICP through the C ABI against the oracle (O7/O8).
Bars as gicp_linearize: pair count equal, |dH|max <= 1e-4 |H|max, b/e within 1e-4
relative or 1e-5 sum|term|; align pose within 1e-3 m / 1e-4 rad."""
import math

import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2308_07173_b200 as g  # noqa: E402

DEV = torch.device("cuda:0")


def D(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def check(g29, o29, ab):
    assert g29[28] == o29[28]
    assert np.abs(g29[:21] - o29[:21]).max() <= 1e-4 * np.abs(o29[:21]).max()
    d = np.abs(g29[21:28] - o29[21:28])
    assert np.all((d <= 1e-4 * np.abs(o29[21:28])) | (d <= 1e-5 * ab[21:28]))


@pytest.mark.parametrize("mode", [1, 7, 27])
@pytest.mark.parametrize("res", [0.5, 1.0])
def test_linearize_vgicp_c1(orc, mode, res):
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    cs = gen.random_covariances(len(src), 1)
    ct = gen.random_covariances(len(tgt), 2)
    idx = g.build_index(D(tgt), res)
    g.attach_voxels(idx, D(ct))
    for T in (T0, T_true):
        out, base = g.linearize_vgicp(D(src), D(cs), idx, T, mode, pivot=T[:3, 3])
        out = out.cpu().numpy()
        o29, ab, obase = orc.linearize_vgicp(src, cs, tgt, ct, T, res, mode, pivot=T[:3, 3])
        check(out, o29, ab)
        assert np.array_equal(base.cpu().numpy(), obase)
        eo, _ = g.linearize_vgicp(D(src), D(cs), idx, T, mode, pivot=T[:3, 3], error_only=True)
        eo = eo.cpu().numpy()
        assert eo[28] == out[28] and eo[27] == out[27] and np.all(eo[:27] == 0)
        # REUSE: the pairs of T at T_true
        ro, _ = g.linearize_vgicp(D(src), D(cs), idx, T_true, mode, pivot=T[:3, 3], base=base, reuse=True)
        o29r, abr, _ = orc.linearize_vgicp(src, cs, tgt, ct, T_true, res, mode, pivot=T[:3, 3], base=obase)
        check(ro.cpu().numpy(), o29r, abr)
    idx.free()


def test_linearize_vgicp_c3_sample_and_align_c2(orc):
    # C3: a scan subsample against the 2M map at 1 m voxels
    sc, mp, T_true, T0 = gen.config_c3()
    rng = np.random.default_rng(5)
    src = np.ascontiguousarray(sc[rng.choice(len(sc), 3000, replace=False)])
    cs = gen.random_covariances(len(src), 3)
    ct = gen.random_covariances(len(mp), 4)
    idx = g.build_index(D(mp), 1.0)
    g.attach_voxels(idx, D(ct))
    out = g.linearize_vgicp(D(src), D(cs), idx, T0, 7, pivot=T0[:3, 3])[0].cpu().numpy()
    o29, ab, _ = orc.linearize_vgicp(src, cs, mp, ct, T0, 1.0, 7, pivot=T0[:3, 3])
    check(out, o29, ab)
    idx.free()
    # C1 align (well conditioned corner): GPU LM vs oracle LM
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.0)
    ns, _ = orc.knn(src, src, 10)
    nt, _ = orc.knn(tgt, tgt, 10)
    cs = orc.covariance(src, ns)[0].astype(np.float32)
    ct = orc.covariance(tgt, nt)[0].astype(np.float32)
    idx = g.build_index(D(tgt), 0.5)
    g.attach_voxels(idx, D(ct))
    T, info = g.align_vgicp(D(src), D(cs), idx, T0, 27)
    r = orc.align_vgicp(src, cs, tgt, ct, T0, 0.5, 27)
    assert info.converged and r["converged"]
    assert np.linalg.norm(T[:3, 3] - r["T"][:3, 3]) <= 1e-3
    c = (np.trace(T[:3, :3] @ r["T"][:3, :3].T) - 1) / 2
    assert math.acos(min(1.0, c)) <= 1e-4
    assert np.linalg.norm(T[:3, 3] - T_true[:3, 3]) < 0.02
    idx.free()


def test_vgicp_errors():
    src, tgt, T_true, T0 = gen.config_c1()
    idx = g.build_index(D(tgt), 0.5)
    with pytest.raises(g.GicpError):  # no voxels attached
        g.linearize_vgicp(D(src), D(gen.random_covariances(len(src), 1)), idx, T0)
    g.attach_voxels(idx, D(gen.random_covariances(len(tgt), 2)))
    with pytest.raises(g.GicpError):
        g.linearize_vgicp(D(src), D(gen.random_covariances(len(src), 1)), idx, T0, mode=5)
    idx.free()
