"""z-vote ground filter through the C ABI vs the oracle (O9):
keep mask and counts bit-exact (integer work on an fp32 decision taken the same
way on both sides)."""
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


@pytest.mark.parametrize("cell,mc", [(0.5, 10), (0.2, 3), (1.0, 1)])
def test_ground_filter_bitwise(orc, cell, mc):
    sc, _ = gen.scan(100_000, 150.0, 77)  # vehicle frame, banked ground + walls + posts
    keep, cnt = g.ground_filter(D(sc), cell, mc, with_count=True)
    ok, oc = orc.ground_filter(sc, cell, mc)
    assert np.array_equal(cnt.cpu().numpy(), oc)
    assert np.array_equal(keep.cpu().numpy(), ok)


def test_ground_filter_edges(orc):
    # points exactly on cell boundaries and negative coordinates
    ij = np.stack(np.meshgrid(np.arange(-20, 20), np.arange(-20, 20)), -1).reshape(-1, 2) * 0.5
    p = np.column_stack([np.repeat(ij, 3, axis=0), np.tile([0.0, 1.0, 2.0], len(ij))]).astype(np.float32)
    keep, cnt = g.ground_filter(D(p), 0.5, 3, with_count=True)
    ok, oc = orc.ground_filter(p, 0.5, 3)
    assert np.array_equal(cnt.cpu().numpy(), oc) and np.array_equal(keep.cpu().numpy(), ok)
    assert g.ground_filter(torch.zeros((0, 3), dtype=torch.float32, device=DEV), 0.5, 3).numel() == 0
    with pytest.raises(g.GicpError):
        g.ground_filter(D(p), 0.0, 3)


# --- Euclidean clustering (O10) ---------------------------------------------
def test_cluster_random_sets(orc):
    rng = np.random.default_rng(21)
    for t in range(20):
        p = rng.uniform(0, 10, (200, 3)).astype(np.float32)
        lab, nc = g.cluster(D(p), 1.0, 1 + t % 3)
        ol, onc = orc.cluster(p, 1.0, 1 + t % 3)
        assert nc == onc and np.array_equal(lab.cpu().numpy(), ol)


def test_cluster_km_offset_pairs_at_tol(orc):
    """Clouds ~2 km from the origin (the grid rounding grows with the extent): chains of
    points spaced just inside tol along random directions must stay one cluster."""
    rng = np.random.default_rng(22)
    tol = 0.3
    for t in range(10):
        base = np.array([2000.0, -1500.0, 30.0]) + rng.uniform(-5, 5, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        chain = base + np.outer(np.arange(12) * tol * (1 - 2e-6), d)
        other = base + rng.uniform(-3, 3, (150, 3))
        p = np.concatenate([chain, other, [[0.0, 0.0, 0.0]]]).astype(np.float32)
        lab, nc = g.cluster(D(p), tol, 1)
        ol, onc = orc.cluster(p, tol, 1)
        assert nc == onc and np.array_equal(lab.cpu().numpy(), ol)


def test_cluster_ground_filtered_scan(orc):
    """The paper's pipeline on a scan: ground filter, then clusters of the
    vertical features (walls, posts, boxes); labels bit-exact vs the oracle."""
    sc, _ = gen.scan(60_000, 300.0, 78)
    _, first = np.unique(np.floor(sc / 0.25).astype(np.int64), axis=0, return_index=True)  # voxel filter (SPEC pre)
    sc = np.ascontiguousarray(sc[np.sort(first)])
    keep = g.ground_filter(D(sc), 0.5, 6).cpu().numpy()
    feat = np.ascontiguousarray(sc[keep])
    assert 500 < len(feat) < 0.8 * len(sc)
    lab, nc = g.cluster(D(feat), 0.5, 10)
    ol, onc = orc.cluster(feat, 0.5, 10)
    assert nc == onc > 1 and np.array_equal(lab.cpu().numpy(), ol)


def test_cluster_edges():
    lab, nc = g.cluster(torch.zeros((0, 3), dtype=torch.float32, device=DEV), 1.0)
    assert nc == 0 and lab.numel() == 0
    same = torch.zeros((50, 3), dtype=torch.float32, device=DEV)  # coincident points: one cluster
    lab, nc = g.cluster(same, 0.1)
    assert nc == 1 and (lab == 0).all()
    with pytest.raises(g.GicpError):
        g.cluster(same, 0.0)


# --- sliding-window submap (O11) ----------------------------------------------
def test_submap_queries_match_the_oracle(orc):
    mp = gen.racetrack_map(2_000_000, 1)
    nb = 240  # ~10 m buckets of the 2408 m oval: bucket = the angle around the oval centre (a race-line proxy)
    b = (np.floor((np.arctan2(mp[:, 1], mp[:, 0]) + np.pi) / (2 * np.pi) * nb).astype(np.int64) % nb).astype(np.int32)
    sm = g.Submap(D(b), nb)
    for center, radius in ((0, 0), (0, 3), (17, 1), (239, 5), (120, 500)):
        got = sm.query(center, radius).cpu().numpy()
        assert np.array_equal(got, orc.submap_query(b, nb, center, radius)), (center, radius)
    sm.free()
    with pytest.raises(g.GicpError):
        g.Submap(D(np.array([0, 5, 240], np.int32)), 240)
