"""Multi-process host logic of the sharded linearisation (gloo, world_size 2-3, CPU).

The chunk rows come from the ORACLE here (no GPU in this test); the chunking and the
allreduce of the chunk table are the product's (paper_2308_07173_b200/sharding.py).
The allreduced table must be bitwise the single-process table for every world size
(the chunk-ordered sum itself is the library's, tested on the GPU in
tests/test_gpu_sharded.py), and its chunk-ordered sum agrees with an unsharded
linearisation to rounding.
"""
import os
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
    import torch
    import torch.distributed as dist
    # file rendezvous: no TCP port to race for (a bind/close/reuse port probe is racy)
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    sh = _load_sharding()
    oracle, src, cs, tgt, ct, T0 = _problem()
    # this rank's chunk rows (the oracle stands in for the GPU linearisation) in the
    # chunk table, zeros elsewhere; the product's allreduce fills the whole table
    table = torch.zeros((1, sh.NUM_CHUNKS, 29), dtype=torch.float64)
    for c in sh.chunks_of_rank(rank, world):
        lo, hi = sh.chunk_bounds(len(src))[c]
        table[0, c] = torch.from_numpy(oracle.linearize(src[lo:hi], cs[lo:hi], tgt, ct, T0, 1.0, pivot=T0[:3, 3])[0])
    sh.make_allreduce()(table)
    q.put((rank, table.numpy().copy()))
    dist.destroy_process_group()


def _free_port():
    """A fresh rendezvous file path for init_method='file://' (the name is kept so the
    callers read as before; nothing binds a port)."""
    import tempfile
    d = tempfile.mkdtemp(prefix="gicp_pg_")
    return os.path.join(d, "rendezvous")


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
    """The allreduced chunk table is bitwise the single-process table (every row has
    one non-zero contributor); its chunk-ordered sum (the library's combine, done
    here in the same order) agrees with an unsharded linearisation to rounding."""
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
    assert np.array_equal(res[0][0], parts) and np.array_equal(res[1][0], parts)
    single = np.zeros(29)
    for c in range(sh.NUM_CHUNKS):
        single = single + parts[c]
    whole, ab, _ = oracle.linearize(src, cs, tgt, ct, T0, 1.0, pivot=T0[:3, 3])
    assert single[28] == whole[28]
    assert np.all(np.abs(single[:28] - whole[:28]) <= 1e-12 * ab[:28] + 1e-300)


# --- point-sharded batched registration (C4): the reduce callback's host logic ---

SIZES = [20000, 0, 7777, 300, 256]


def _chunk_rows(b, c):
    """Deterministic stand-in for one chunk's 32-value row (what one GPU launch
    would produce for chunk c of registration b): wide dynamic range so any
    change of summation order shows in the bits."""
    rng = np.random.default_rng(1000 * b + c)
    return rng.standard_normal(32) * 10.0 ** rng.integers(-8, 8, 32)


def _table_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    sh = _load_sharding()
    table = torch.zeros((len(SIZES) * sh.NUM_CHUNKS, 32), dtype=torch.float64)
    for (b, c, _, _) in sh.registration_chunks(SIZES, rank, world):
        table[b * sh.NUM_CHUNKS + c] = torch.from_numpy(_chunk_rows(b, c))
    sh.make_allreduce()(table)
    q.put((rank, table.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_chunk_table_allreduce_is_world_size_independent(world):
    """Every rank gets the full chunk table of every registration, bitwise equal to
    the single-process table, for world sizes 2 and 3 (what the library then sums in
    chunk order on the device: gicp_align_batched_sharded)."""
    sh = _load_sharding()
    B = len(SIZES)
    single = np.zeros((B * sh.NUM_CHUNKS, 32))
    for (b, c, _, _) in sh.registration_chunks(SIZES, 0, 1):
        single[b * sh.NUM_CHUNKS + c] = _chunk_rows(b, c)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_table_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert np.array_equal(res[r], single)
    # chunks cover every point once; empty registrations have no entries
    for w in (1, 2, 4, 8):
        cov = {b: 0 for b in range(B)}
        for r in range(w):
            for (b, c, lo, hi) in sh.registration_chunks(SIZES, r, w):
                assert c % w == r and hi > lo
                cov[b] += hi - lo
        assert [cov[b] for b in range(B)] == SIZES
