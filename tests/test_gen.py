"""Synthetic input generator: determinism and the recipe's structural facts."""
import math

import numpy as np

import gen


def test_map_deterministic_and_shaped():
    a = gen.racetrack_map(20_000, 3)
    b = gen.racetrack_map.__wrapped__(20_000, 3)
    assert a.dtype == np.float32 and a.shape == (20_000, 3) and a.flags.c_contiguous
    assert np.array_equal(a, b)
    assert np.abs(a[:, 0]).max() < 480 and np.abs(a[:, 1]).max() < 290
    assert a[:, 2].min() > -0.1 and a[:, 2].max() < 2 * 9 * math.tan(math.radians(20)) + 4.2


def test_bank_profile():
    u = np.linspace(0, gen.TRACK_LEN, 10_000)
    b = gen.bank(u)
    assert np.all(np.abs(b) < math.pi / 4)
    assert math.isclose(gen.bank(np.array([200.0]))[0], math.radians(9))
    assert math.isclose(gen.bank(np.array([gen.STRAIGHT + 100.0]))[0], math.radians(20))


def test_scan_frame_and_ranges():
    s, T = gen.scan(5000, 123.0, 77)
    r = np.linalg.norm(s, axis=1)
    assert s.shape == (5000, 3) and r.max() <= 100.0 + 1e-3 and r.min() >= 1.0 - 1e-3
    R = T[:3, :3]
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and math.isclose(np.linalg.det(R), 1.0)
    s2, T2 = gen.scan.__wrapped__(5000, 123.0, 77)
    assert np.array_equal(s, s2)


def test_c1_shapes():
    src, tgt, T, T0 = gen.config_c1()
    assert src.shape == tgt.shape == (1000, 3)
    src2, tgt2, _, _ = gen.config_c1(exact_copy=True)
    back = gen.apply_T(T, src2)
    assert np.abs(back - tgt2).max() < 1e-5
