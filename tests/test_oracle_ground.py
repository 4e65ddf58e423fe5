"""Pins of the z-vote ground filter oracle (O9, SPEC S:543-548,
DESIGN.md reading R24): SPEC's worked examples, counts against numpy's unique on
clouds where the cell formula is exact, and SPEC's banked-straight-with-wall
property on a labelled synthetic scene."""
import numpy as np
import pytest

orc = pytest.importorskip("oracle")


def test_spec_examples():
    p = np.zeros((12, 3), np.float32)
    p[:, 0], p[:, 1], p[:, 2] = 0.3, 0.4, np.linspace(0.0, 2.5, 12)  # 12 stacked points, one cell
    keep, cnt = orc.ground_filter(p, 0.5, 5)
    assert keep.all() and (cnt == 12).all()
    q = np.array([[3.1, 3.2, 0.0], [3.3, 3.4, 0.01]], np.float32)      # 2 ground points in a cell
    keep, cnt = orc.ground_filter(np.concatenate([p, q]), 0.5, 5)
    assert keep[:12].all() and not keep[12:].any() and (cnt[12:] == 2).all()


def test_counts_vs_numpy_unique():
    rng = np.random.default_rng(2)
    cell = 0.25  # a power of two: fl32(x * 4) is exact, so floor(x / cell) is plain
    ij = rng.integers(-60, 60, (5000, 2))
    frac = rng.integers(0, 4, (5000, 2)) / 16.0  # stays inside the cell, exactly representable
    xy = (ij + frac) * cell
    p = np.column_stack([xy, rng.uniform(-1, 3, 5000)]).astype(np.float32)
    keep, cnt = orc.ground_filter(p, cell, 3)
    _, inv, counts = np.unique(ij, axis=0, return_inverse=True, return_counts=True)
    assert np.array_equal(cnt, counts[inv.ravel()])
    assert np.array_equal(keep, counts[inv.ravel()] >= 3)


def test_banked_straight_with_wall():
    """>= 99 % of ground removed, >= 95 % of wall kept (9 deg bank,
    1.2 m wall; voxel-filtered at leaf 0.25 <= cell 0.5; min_count 10)."""
    rng = np.random.default_rng(1)
    bank = np.tan(np.radians(9.0))
    g = np.column_stack([rng.uniform(0, 40, 400000), rng.uniform(-9, 9, 400000), np.zeros(400000)])
    g[:, 2] = bank * g[:, 1]
    w = np.column_stack([rng.uniform(0, 40, 200000), np.full(200000, 9.05), rng.uniform(0, 1.2, 200000)])
    w[:, 2] += bank * 9.0
    pts = np.concatenate([g, w]).astype(np.float32)
    lab = np.r_[np.zeros(len(g), bool), np.ones(len(w), bool)]
    _, first = np.unique(np.floor(pts / 0.25).astype(np.int64), axis=0, return_index=True)
    first.sort()
    p, lab = pts[first], lab[first]
    keep, _ = orc.ground_filter(p, 0.5, 10)
    assert 1.0 - keep[~lab].mean() >= 0.99 and keep[lab].mean() >= 0.95
