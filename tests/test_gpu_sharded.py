"""Point-sharded batched registration (C4 across processes) on the
GPU: each process linearises its chunks of every registration through
gicp_align_batched_sharded and one all_reduce of the device chunk table per round
combines them, summed in chunk order on the device (gloo here:
there is one GPU, both processes use it; the host-side collective never makes
kernels wait on each other). World size 2 must reproduce world size 1 BITWISE
(fixed chunking, chunk-ordered combine), and both must agree with the unsharded
gicp_align_batched to rounding (different summation order)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCANS = [(0, 20000), (64, 7777), (200, 3000)]
TINY = [(10, 200), (90, 150)]  # one chunk each: rank 1 of 2 holds no entry at all


def _problem(scans=None):
    scans = scans or SCANS
    sys.path.insert(0, ROOT)
    import gen
    import paper_2308_07173_b200 as g
    dev = torch.device("cuda:0")
    D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    mp_ = gen.racetrack_map(2_000_000, 1)
    im = g.build_index(D(mp_), 0.5)
    _, _, cm = g.knn_cov_self(im, 20, 1e-3, with_nbr=False)
    g.attach_cov(im, cm)
    srcs, covs, T0 = [], [], []
    for i, n in scans:
        sc, T, Tp = gen.config_c4_scan(i, n)
        sd = D(sc)
        isc = g.build_index(sd, 0.0)
        _, _, cs = g.knn_cov_self(isc, 20, 1e-3, with_nbr=False)
        isc.free()
        srcs.append(sd)
        covs.append(cs)
        T0.append(Tp)
    offs = np.concatenate([[0], np.cumsum([s.shape[0] for s in srcs])]).astype(np.int64)
    return g, im, cm, torch.cat(srcs).contiguous(), torch.cat(covs).contiguous(), offs, np.array(T0)


def _worker(rank, world, port, q, tiny=False, groups=1):
    import torch.distributed as dist
    # file rendezvous: no TCP port to race for (a bind/close/reuse port probe is racy)
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2308_07173_b200 import sharding
    g, im, cm, src, cov, offs, T0 = _problem(TINY if tiny else None)
    if groups > 1:  # concurrent groups, their allreduces in round-robin order
        conc = sharding.ConcurrentAlign(offs, src.device, groups)
        Ts, infos = conc(g, src, cov, im, cm, T0)
    else:
        Ts, infos = sharding.align_batched_sharded(g, src, cov, offs, im, cm, T0)
    q.put((rank, Ts, [(i.iterations, i.converged, i.error, i.inliers) for i in infos]))
    dist.destroy_process_group()


def _free_port():
    """A fresh rendezvous file path for init_method='file://' (the name is kept so the
    callers read as before; nothing binds a port)."""
    import tempfile
    d = tempfile.mkdtemp(prefix="gicp_pg_")
    return os.path.join(d, "rendezvous")


def _run(world, tiny=False, groups=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, tiny, groups)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (T, inf)) for r, T, inf in (q.get(timeout=240) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_sharded_align_world2_is_bitwise_world1():
    r1 = _run(1)
    r2 = _run(2)
    T1, i1 = r1[0]
    for r in (0, 1):
        T2, i2 = r2[r]
        assert np.array_equal(T2, T1)
        assert i2 == i1
    # against the unsharded batched align (registration-wide summation order)
    g, im, cm, src, cov, offs, T0 = _problem()
    Tu, iu = g.align_batched(src, cov, offs, im, cm, T0)
    for b in range(len(SCANS)):
        assert np.linalg.norm(T1[b][:3, 3] - Tu[b][:3, 3]) <= 1e-3
        c = (np.trace(T1[b][:3, :3] @ Tu[b][:3, :3].T) - 1) / 2
        assert np.arccos(min(1.0, c)) <= 1e-4
        assert i1[b][3] > 0 and abs(i1[b][3] - iu[b].inliers) <= 0.001 * iu[b].inliers


@pytest.mark.parametrize("world", [1, 2])
def test_concurrent_groups_are_bitwise_the_single_call(world):
    """sharding.ConcurrentAlign (bench.py's timed steps): the batch split into
    concurrent groups, each its own host thread and stream, the groups' per-round
    allreduces ordered round-robin on the one process group; every pose and info
    bitwise the single batched call's."""
    r1 = _run(1)
    rg = _run(world, groups=2)
    for r in range(world):
        assert np.array_equal(rg[r][0], r1[0][0]) and rg[r][1] == r1[0][1]


def test_sharded_align_with_an_idle_rank():
    """Registrations smaller than one chunk: rank 1 has no entries but still takes
    part in every round's all_reduce; the result equals world size 1 bitwise."""
    r1 = _run(1, tiny=True)
    r2 = _run(2, tiny=True)
    for r in (0, 1):
        assert np.array_equal(r2[r][0], r1[0][0]) and r2[r][1] == r1[0][1]


def test_combine_chunks_is_the_chunk_ordered_sum():
    sys.path.insert(0, ROOT)
    import paper_2308_07173_b200 as g
    rng = np.random.default_rng(3)
    B, nc, w = 7, 8, 32
    t = rng.standard_normal((B, nc, w)) * 10.0 ** rng.integers(-8, 8, (B, nc, w))
    ref = np.zeros((B, w))
    for k in range(nc):
        ref = ref + t[:, k]
    out = g.combine_chunks(torch.from_numpy(t).cuda(), B, nc, w).cpu().numpy()
    assert np.array_equal(out, ref)


def test_sharded_linearize_world1():
    """sharded_linearize without a process group: the chunk-ordered device combine of
    the chunk linearisations, equal to the unsharded call to rounding."""
    sys.path.insert(0, ROOT)
    from paper_2308_07173_b200 import sharding
    g, im, cm, src, cov, offs, T0 = _problem(TINY + [(30, 5000)])
    s, c = src[offs[2]:offs[3]].contiguous(), cov[offs[2]:offs[3]].contiguous()
    T = T0[2]
    a = sharding.sharded_linearize(g, s, c, im, cm, T, 1.0, pivot=T[:3, 3]).cpu().numpy()
    b, _ = g.linearize(s, c, im, cm, T, 1.0, pivot=T[:3, 3])
    b = b.cpu().numpy()
    assert a[28] == b[28]
    assert np.allclose(a[:28], b[:28], rtol=1e-9, atol=1e-9 * np.abs(b[:28]).max())


# --- C5: query sharding over cell-sorted ranges, the index broadcast from rank 0 ---

def _c5_problem():
    sys.path.insert(0, ROOT)
    import gen
    mp = gen.racetrack_map(300_000, 3)
    sc, T = gen.scan(20_000, 700.0, 2001)
    q = gen.apply_T(T, sc).astype(np.float32)
    return mp, np.ascontiguousarray(q)


def _c5_worker(rank, world, port, q_out):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import paper_2308_07173_b200 as g
    from paper_2308_07173_b200 import sharding
    mp, q = _c5_problem()
    dev = torch.device("cuda:0")
    idx = g.build_index(torch.from_numpy(mp).to(dev), 0.4) if rank == 0 else None
    idx = sharding.broadcast_index(g, idx, src=0, device=dev)
    qd = torch.from_numpy(q).to(dev)
    nbr, d2, ids = sharding.knn_sharded(g, idx, qd, 32, gather=True)
    q_out.put((rank, nbr.cpu().numpy(), d2.cpu().numpy(), ids.cpu().numpy()))
    dist.destroy_process_group()


def test_c5_query_sharding_with_broadcast_index():
    """Rank 0 builds the map index and broadcasts it; each rank takes a contiguous
    range of the cell-sorted queries; the gathered rows are bitwise gicp_knn's."""
    sys.path.insert(0, ROOT)
    import paper_2308_07173_b200 as g
    mp, q = _c5_problem()
    dev = torch.device("cuda:0")
    idx = g.build_index(torch.from_numpy(mp).to(dev), 0.4)
    qd = torch.from_numpy(q).to(dev)
    ref_n, ref_d = g.knn(idx, qd, 32)
    ref_n, ref_d = ref_n.cpu().numpy(), ref_d.cpu().numpy()
    # export / import in one process: the copy answers identically
    hdr, bufs = g.index_export(idx)
    import paper_2308_07173_b200.sharding as sh
    ts = [None if nb == 0 else torch.as_tensor(sh._DevBytes(p, nb, dev), device=dev).clone() for p, nb in bufs]
    idx2 = g.index_import(hdr, ts, dev)
    n2, d22 = g.knn(idx2, qd, 32)
    assert np.array_equal(n2.cpu().numpy(), ref_n) and np.array_equal(d22.cpu().numpy(), ref_d)
    ctx = mp_ctx = torch.multiprocessing.get_context("spawn")
    qq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, 2, port, qq)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (n, d, i)) for r, n, d, i in (qq.get(timeout=240) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in (0, 1):
        assert np.array_equal(res[r][0], ref_n) and np.array_equal(res[r][1], ref_d)
    ids = np.sort(np.concatenate([res[0][2], res[1][2]]))
    assert np.array_equal(ids, np.arange(len(q)))
