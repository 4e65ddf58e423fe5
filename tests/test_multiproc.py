"""Multi-process host logic of the sharded linearisation (gloo, world_size 2, CPU).

The chunk partials come from the ORACLE here (no GPU in this test); the sharding,
all-gather and chunk-ordered combine are the product's (paper_2308_07173_b200/
sharding.py). H, b, e must be bitwise identical to the single-process combine of
the same chunks and agree with an unsharded linearisation to rounding.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load_sharding():
    import importlib.util
    spec = importlib.util.spec_from_file_location("gicp_sharding", os.path.join(ROOT, "paper_2308_07173_b200",
                                                                               "sharding.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _problem():
    sys.path.insert(0, ROOT)
    import gen
    import oracle
    src, tgt, T_true, T0 = gen.config_c1(sigma=0.002)
    cs = gen.random_covariances(len(src), 1)
    ct = gen.random_covariances(len(tgt), 2)
    return oracle, src, cs, tgt, ct, T0


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = _load_sharding()
    oracle, src, cs, tgt, ct, T0 = _problem()
    local = {}
    for c in sh.chunks_of_rank(rank, world):
        lo, hi = sh.chunk_bounds(len(src))[c]
        local[c] = oracle.linearize(src[lo:hi], cs[lo:hi], tgt, ct, T0, 1.0, pivot=T0[:3, 3])[0]
    full = sh.allgather_partials(local)
    q.put((rank, sh.combine(full)))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_chunking_is_world_size_independent():
    sh = _load_sharding()
    for n in (0, 1, 255, 256, 1000, 30_000, 100_000):
        b = sh.chunk_bounds(n)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(lo <= hi for lo, hi in b) and all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
        assert all(lo % sh.PPB == 0 or lo == n for lo, _ in b)
        for w in (1, 2, 4, 8):
            owned = sorted(c for r in range(w) for c in sh.chunks_of_rank(r, w))
            assert owned == list(range(sh.NUM_CHUNKS))


def test_gloo_world2_matches_single_process_bitwise():
    sh = _load_sharding()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    oracle, src, cs, tgt, ct, T0 = _problem()
    parts = np.stack([oracle.linearize(src[lo:hi], cs[lo:hi], tgt, ct, T0, 1.0, pivot=T0[:3, 3])[0]
                      for lo, hi in sh.chunk_bounds(len(src))])
    single = sh.combine(parts)
    assert np.array_equal(res[0], single) and np.array_equal(res[1], single)
    whole, ab, _ = oracle.linearize(src, cs, tgt, ct, T0, 1.0, pivot=T0[:3, 3])
    assert single[28] == whole[28]
    assert np.all(np.abs(single[:28] - whole[:28]) <= 1e-12 * ab[:28] + 1e-300)
