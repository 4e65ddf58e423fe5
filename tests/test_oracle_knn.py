"""Pins for oracle O1 (brute-force kNN) against things other than itself.

Definition (readings R5, R9): the k smallest keys
(fp32 d2 in the fixed FMA order, target index) over ALL targets, ascending.
Paper: "finding corresponding points ... computationally expensive" (PAPER.md
l.403-405), "GPU-based nearest points search" (l.413, l.798).
"""
import ctypes
import json
import os

import numpy as np
import pytest

import gen
from tests.fp32emu import d2_fp32, fma32, knn_lexsort

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_fma_emulation_matches_libm_fmaf():
    libm = ctypes.CDLL("libm.so.6")
    libm.fmaf.argtypes = [ctypes.c_float] * 3
    libm.fmaf.restype = ctypes.c_float
    rng = np.random.default_rng(0)
    a = rng.normal(size=4000).astype(np.float32)
    b = rng.normal(size=4000).astype(np.float32)
    c = (rng.normal(size=4000) * 10).astype(np.float32)
    # include cases where fused and unfused differ
    a[:3] = np.float32(1 + 2 ** -12)
    b[:3] = np.float32(1 + 2 ** -12)
    c[:3] = np.float32(-1)
    ref = np.array([libm.fmaf(float(x), float(y), float(z)) for x, y, z in zip(a, b, c)], np.float32)
    assert np.array_equal(fma32(a, b, c), ref)
    assert fma32(a[:1], b[:1], c[:1])[0] == np.float32(2 ** -11 + 2 ** -24)


def test_lattice_worked_example(orc):
    g = json.load(open(os.path.join(GOLD, "lattice_knn.json")))
    L = gen.lattice(g["side"])
    nbr, d2 = orc.knn(L, np.array([g["query"]], np.float32), g["k"])
    assert nbr[0].tolist() == g["nbr"]
    assert d2[0].tolist() == g["d2"]


def test_exact_quantised_cloud_vs_integer_lexsort(orc):
    # On a 1/8 m lattice inside [-40, 40] every fp32 d2 is exact, so the order is
    # decided by exact integers; ties are frequent.
    tgt = gen.quantised_cloud(3000, 1, half=10.0)
    q = gen.quantised_cloud(300, 2, half=10.0)
    k = 16
    nbr, d2 = orc.knn(tgt, q, k)
    T8 = np.rint(tgt.astype(np.float64) * 8).astype(np.int64)
    Q8 = np.rint(q.astype(np.float64) * 8).astype(np.int64)
    idx = np.arange(len(tgt))
    ties = 0
    for i in range(len(q)):
        di = ((T8 - Q8[i]) ** 2).sum(1)
        order = np.lexsort((idx, di))[:k]
        assert nbr[i].tolist() == order.tolist()
        assert np.array_equal(d2[i].astype(np.float64) * 64, di[order].astype(np.float64))
        ties += int(np.any(np.diff(di[order]) == 0))
    assert ties > 0  # the fixture really exercises the tie rule


@pytest.mark.parametrize("k", [1, 7, 20, 32])
def test_random_float_cloud_vs_fma_emulation(orc, k):
    tgt = gen.uniform_cloud(2000, 3, offset=(812.0, -377.0, 3.0))
    q = gen.uniform_cloud(150, 4, offset=(812.0, -377.0, 3.0))
    nbr, d2 = orc.knn(tgt, q, k)
    rn, rd = knn_lexsort(tgt, q, k)
    assert np.array_equal(nbr, rn)
    assert np.array_equal(d2.view(np.uint32), rd.view(np.uint32))


def test_completeness_and_order_invariants(orc):
    tgt = gen.uniform_cloud(1500, 5)
    q = gen.uniform_cloud(100, 6)
    k = 12
    nbr, d2 = orc.knn(tgt, q, k)
    for i in range(len(q)):
        d_all = d2_fp32(q[i][None, :], tgt)
        keys = (d_all.view(np.uint32).astype(np.uint64) << np.uint64(32)) | np.arange(len(tgt), dtype=np.uint64)
        sel = keys[nbr[i]]
        assert np.all(np.diff(sel.astype(np.float64)) > 0) or np.all(sel[1:] > sel[:-1])
        rest = np.setdiff1d(np.arange(len(tgt)), nbr[i])
        assert keys[rest].min() > sel[-1]


def test_self_query_first_and_duplicates(orc):
    p = gen.uniform_cloud(500, 7)
    nbr, d2 = orc.knn(p, p, 5)
    assert np.array_equal(nbr[:, 0], np.arange(500))
    assert np.all(d2[:, 0] == 0)
    # >= k exact duplicates: ascending index among equal d2 = 0
    dup = np.concatenate([p[:10], np.repeat(p[10:11], 8, 0), p[11:50]])
    nbr, d2 = orc.knn(dup, dup[12:13], 6)
    assert nbr[0].tolist() == [10, 11, 12, 13, 14, 15]
    assert np.all(d2[0] == 0)


def test_edge_cases(orc):
    p = gen.uniform_cloud(10, 8)
    with pytest.raises(orc.OracleError) as e:
        orc.knn(p, p, 11)
    assert e.value.code == orc.EK
    with pytest.raises(orc.OracleError):
        orc.knn(p, p, 33)
    with pytest.raises(orc.OracleError):
        orc.knn(p, p, 0)
    nbr, d2 = orc.knn(p[:1], p, 1)          # n = 1
    assert np.all(nbr == 0)
    nbr, d2 = orc.knn(p, p[:0], 3)          # m = 0
    assert nbr.shape == (0, 3)
    bad = p.copy()
    bad[3, 1] = np.nan
    with pytest.raises(orc.OracleError):
        orc.knn(bad, p, 3)
    with pytest.raises(orc.OracleError):
        orc.knn(p, bad, 3)
    # a query far outside the cloud still gets the exact k nearest
    far = np.array([[2000.0, -2000.0, 50.0]], np.float32)
    nbr, d2 = orc.knn(p, far, 4)
    rn, rd = knn_lexsort(p, far, 4)
    assert np.array_equal(nbr, rn) and np.array_equal(d2, rd)


def test_d2_definition_order(orc):
    # operand order is part of the definition: unfused vs fused results differ here
    a, b = np.float32(0.7162393927574158), np.float32(1.1085484027862549)
    q = np.array([a, b, 0], np.float32)
    p = np.zeros(3, np.float32)
    unfused = np.float32(np.float32(b * b) + np.float32(a * a))
    fused = fma32(b, b, np.float32(a * a))[()]
    assert fused != unfused
    assert orc.d2(q, p) == fused
    q = np.array([0.1, 0.2, 0.3], np.float32)
    p = np.array([1.7, -2.3, 0.9], np.float32)
    assert orc.d2(q, p) == d2_fp32(q, p)
