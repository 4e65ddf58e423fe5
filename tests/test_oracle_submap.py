"""Pins of the sliding-window submap oracle (O11, SPEC
S:399-407 examples, reading R26)."""
import numpy as np
import pytest

orc = pytest.importorskip("oracle")


def test_spec_examples():
    rng = np.random.default_rng(0)
    nb = 40
    bucket = rng.integers(0, nb, 5000).astype(np.int32)
    # radius >= track length -> the whole map, each point once
    whole = orc.submap_query(bucket, nb, 7, nb)
    assert np.array_equal(np.sort(whole), np.arange(5000))
    # radius = 1 bucket -> the containing bucket and its two arc-length neighbours
    got = orc.submap_query(bucket, nb, 7, 1)
    want = np.concatenate([np.nonzero(bucket == b)[0] for b in (6, 7, 8)])
    assert np.array_equal(got, want)
    # the track is closed: the window wraps
    got = orc.submap_query(bucket, nb, 0, 2)
    want = np.concatenate([np.nonzero(bucket == b)[0] for b in (38, 39, 0, 1, 2)])
    assert np.array_equal(got, want)
    assert orc.submap_query(bucket, nb, 5, 0).size == (bucket == 5).sum()
    with pytest.raises(orc.OracleError):
        orc.submap_query(bucket, nb, nb, 1)
