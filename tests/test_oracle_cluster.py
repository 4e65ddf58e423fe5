"""Pins of the Euclidean clustering oracle (O10, SPEC
S:549-556, reading R25): SPEC's worked examples and agreement with
scipy's connected components on 100 random 200-point sets (SPEC's own check),
plus the size filter and the label order."""
import numpy as np
import pytest

orc = pytest.importorskip("oracle")
csgraph = pytest.importorskip("scipy.sparse.csgraph")
sparse = pytest.importorskip("scipy.sparse")


def test_spec_examples():
    a = np.zeros((5, 3), np.float32)
    a[:, 0] = np.arange(5) * 0.5
    lab, nc = orc.cluster(np.concatenate([a, a + [10.0, 0.0, 0.0]]).astype(np.float32), 1.0)
    assert nc == 2 and len(set(lab[:5])) == 1 and len(set(lab[5:])) == 1 and lab[0] != lab[5]
    chain = np.zeros((30, 3), np.float32)
    chain[:, 1] = np.arange(30) * 0.9  # consecutive points within the tolerance
    lab, nc = orc.cluster(chain, 1.0)
    assert nc == 1 and (lab == 0).all()


def test_random_sets_vs_scipy_connected_components():
    rng = np.random.default_rng(11)
    done = 0
    while done < 100:
        p = rng.uniform(0, 10, (200, 3)).astype(np.float32)
        d = np.sqrt(((p[:, None, :].astype(np.float64) - p[None, :, :]) ** 2).sum(-1))
        if (np.abs(d - 1.0) < 1e-4).any():  # ambiguous in fp32: skip the set
            continue
        done += 1
        ncs, comp = csgraph.connected_components(sparse.csr_matrix(d <= 1.0), directed=False)
        lab, nc = orc.cluster(p, 1.0, 1)
        assert nc == ncs
        # same partition: a bijection between labels
        pairs = set(zip(lab.tolist(), comp.tolist()))
        assert len(pairs) == nc
        # order: descending size, ties by the smallest member index
        sizes = np.bincount(lab)
        firsts = np.array([np.nonzero(lab == c)[0][0] for c in range(nc)])
        key = list(zip(-sizes, firsts))
        assert key == sorted(key)


def test_min_size_drops_small_clusters():
    rng = np.random.default_rng(3)
    big = rng.uniform(0, 2, (50, 3))
    small = rng.uniform(0, 0.1, (3, 3)) + 20.0
    lone = np.array([[40.0, 0.0, 0.0]])
    lab, nc = orc.cluster(np.concatenate([small, big, lone]).astype(np.float32), 1.0, min_size=5)
    assert nc == 1 and (lab[:3] == -1).all() and (lab[3:53] == 0).all() and lab[53] == -1
