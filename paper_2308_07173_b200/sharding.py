"""Multi-GPU sharding of the linearisation.

The target map/index is replicated on every rank; the source points of a
registration are split into a FIXED global set of chunks (aligned to the
linearize kernel's blocks (256-point multiples), independent of the world size).
Each rank linearises its chunks; the 32-value chunk rows are placed in a device
table [B * num_chunks][32] that is zero elsewhere, ONE in-place all_reduce(sum)
over NCCL (NVLink) fills every row from its single owner (exact), and the
library sums each registration's chunk rows in chunk order on the device
(gicp_combine_chunks). H, b and e are therefore bitwise identical for world sizes
1, 2, 4, 8, and every rank runs the identical host LM step (no broadcast of T).

This module is plumbing only (chunk bookkeeping, the collective): every sum of the
method's values happens in the library.
"""
from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch
import torch.distributed as dist

PPB = 256          # chunk alignment: a multiple of every linearize block size (kLinPPB = 256 / team)
NUM_CHUNKS = 8     # fixed global chunk count (= the largest world size served)


def chunk_bounds(n: int, num_chunks: int = NUM_CHUNKS):
    """[lo, hi) of every chunk: whole PPB blocks, as equal as possible."""
    nb = (n + PPB - 1) // PPB
    per = [nb // num_chunks + (1 if c < nb % num_chunks else 0) for c in range(num_chunks)]
    bounds, b = [], 0
    for c in range(num_chunks):
        lo = min(n, b * PPB)
        b += per[c]
        hi = min(n, b * PPB)
        bounds.append((lo, hi))
    return bounds


def chunks_of_rank(rank: int, world: int, num_chunks: int = NUM_CHUNKS):
    """Chunk ids owned by a rank (round robin)."""
    return [c for c in range(num_chunks) if c % world == rank]


def registration_chunks(sizes, rank: int, world: int, num_chunks: int = NUM_CHUNKS):
    """This rank's entries of a batch: (registration b, chunk c, lo, hi) with [lo, hi)
    relative to registration b, for every non-empty chunk c with c % world == rank."""
    out = []
    for b, n in enumerate(sizes):
        for c, (lo, hi) in enumerate(chunk_bounds(int(n), num_chunks)):
            if c % world == rank and hi > lo:
                out.append((b, c, lo, hi))
    return out


def make_allreduce(group=None):
    """In-place sum of a float64 device table over the group's ranks: NCCL reduces the
    device tensor on the current stream; gloo (CPU test runs) goes through host memory.
    None when there is nothing to reduce (no process group, or a single rank)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    if dist.get_backend(group) == "nccl":
        def ar(table: torch.Tensor):
            dist.all_reduce(table, op=dist.ReduceOp.SUM, group=group)
    else:
        def ar(table: torch.Tensor):
            h = table.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            table.copy_(h)
    return ar


def sharded_linearize(g, src, src_cov, index, tgt_cov, T, max_corr_dist=1.0, pivot=None, group=None,
                      num_chunks: int = NUM_CHUNKS):
    """gicp_linearize over this rank's chunks, the chunk table allreduced, the
    chunk-ordered sum on the device (gicp_combine_chunks). Returns float64 [29] (device)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n = src.shape[0]
    table = torch.zeros((1, num_chunks, 29), dtype=torch.float64, device=src.device)
    for c in chunks_of_rank(rank, world, num_chunks):
        lo, hi = chunk_bounds(n, num_chunks)[c]
        g.linearize(src[lo:hi].contiguous(), src_cov[lo:hi].contiguous(), index, tgt_cov, T, max_corr_dist,
                    pivot=pivot, out=table[0, c])
    ar = make_allreduce(group)
    if ar is not None:
        ar(table)
    return g.combine_chunks(table, 1, num_chunks, 29)[0]


class ShardPlan:
    """This rank's part of a batch (fixed global chunking): its entries (b, c, lo, hi),
    the device gather index of their rows in the batch arrays, the local entry
    offsets and the global chunk rows b * num_chunks + c. Reusable while the batch's
    layout is unchanged (bench.py builds it once)."""

    def __init__(self, offsets, device, group=None, num_chunks: int = NUM_CHUNKS, reg_base=None):
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        offsets = np.asarray(offsets, dtype=np.int64)
        self.B = len(offsets) - 1
        self.num_chunks = num_chunks
        base = offsets[:-1] if reg_base is None else np.asarray(reg_base, dtype=np.int64)
        self.entries = registration_chunks(np.diff(offsets), rank, world, num_chunks)
        lens = np.array([hi - lo for (_, _, lo, hi) in self.entries], dtype=np.int64)
        self.loffs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        starts = np.array([base[b] + lo for (b, _, lo, _) in self.entries], dtype=np.int64)
        n = int(self.loffs[-1])
        # row i of entry e: starts[e] + (i - loffs[e])
        idx = np.arange(n, dtype=np.int64) + np.repeat(starts - self.loffs[:-1], lens) if n else np.zeros(0, np.int64)
        self.idx = torch.from_numpy(idx).to(device)
        self.gid = np.array([b * num_chunks + c for (b, c, _, _) in self.entries], dtype=np.int32)
        self.group = group


def align_batched_sharded(g, src, src_cov, offsets, tgt, tgt_cov, T0s, group=None, num_chunks: int = NUM_CHUNKS,
                          reg_base=None, plan: ShardPlan | None = None, **params):
    """Batched LM alignment with the source points of every registration split into
    a fixed global chunking; this rank linearises its chunks (one batched launch
    per evaluation round), one NCCL all_reduce of the device chunk table per round
    combines them, and every rank runs the identical host LM. src / src_cov: the
    batch's points on this rank's GPU (only this rank's chunks are used);
    registration b has offsets[b+1] - offsets[b] points starting at row
    reg_base[b] (default offsets[b]; registrations may share rows). Returns
    (T [B,4,4], infos)."""
    if plan is None:
        plan = ShardPlan(offsets, src.device, group, num_chunks, reg_base)
    if plan.idx.numel():
        src_l, cov_l = src.index_select(0, plan.idx), src_cov.index_select(0, plan.idx)
    else:
        src_l = torch.zeros((0, 3), dtype=src.dtype, device=src.device)
        cov_l = torch.zeros((0, 6), dtype=src_cov.dtype, device=src_cov.device)
    return g.align_batched_sharded(src_l, cov_l, plan.loffs, plan.gid, plan.num_chunks, plan.B, tgt, tgt_cov, T0s,
                                   allreduce=make_allreduce(plan.group), **params)


class _RoundRobinGate:
    """Orders the per-round collectives of concurrently aligned groups: group k may
    enqueue its allreduce only on its turn; turns go round-robin over the groups
    still aligning. Every rank runs the same groups with the same round counts
    (their rows are bitwise equal), so every rank enqueues the same sequence of
    collectives on the one communicator."""

    def __init__(self, n):
        self.n, self.turn, self.done = n, 0, [False] * n
        self.cv = threading.Condition()

    def _advance(self):
        for step in range(1, self.n + 1):
            t = (self.turn + step) % self.n
            if not self.done[t]:
                self.turn = t
                break
        self.cv.notify_all()

    def run(self, k, fn):
        with self.cv:
            while self.turn != k:
                self.cv.wait()
            try:
                fn()
            finally:
                self._advance()

    def finish(self, k):
        with self.cv:
            self.done[k] = True
            if self.turn == k:
                self._advance()
            self.cv.notify_all()


class ConcurrentAlign:
    """The batch's registrations split into `n_groups` contiguous groups, each aligned
    by `align_batched_sharded` on its own host thread and CUDA stream, so one group's
    kernels run while another's host LM decides its next round (the GPU no longer
    idles at every round's host turn-around). Per registration the result is bitwise
    the single batched call's (every registration is evaluated exactly as alone).
    With a process group, the groups' chunk-table allreduces are issued in a fixed
    round-robin order (_RoundRobinGate) on the one communicator."""

    def __init__(self, offsets, device, n_groups: int, group=None, num_chunks: int = NUM_CHUNKS, reg_base=None):
        offsets = np.asarray(offsets, dtype=np.int64)
        B = len(offsets) - 1
        base = offsets[:-1] if reg_base is None else np.asarray(reg_base, dtype=np.int64)
        n_groups = max(1, min(int(n_groups), B))
        cuts = [round(k * B / n_groups) for k in range(n_groups + 1)]
        self.ranges = [(cuts[k], cuts[k + 1]) for k in range(n_groups) if cuts[k + 1] > cuts[k]]
        self.plans = []
        for lo, hi in self.ranges:
            sub = offsets[lo:hi + 1] - offsets[lo]
            self.plans.append(ShardPlan(sub, device, group, num_chunks, base[lo:hi]))
        self.streams = [torch.cuda.Stream(device=device) for _ in self.ranges]
        dev_index = torch.device(device).index
        self.pool = ThreadPoolExecutor(max_workers=len(self.ranges),
                                       initializer=lambda: torch.cuda.set_device(dev_index))
        self.group = group

    def __call__(self, g, src, src_cov, tgt, tgt_cov, T0s, **params):
        T0s = np.asarray(T0s, dtype=np.float64)
        caller = torch.cuda.current_stream(src.device)
        ready = torch.cuda.Event()
        ready.record(caller)
        collective = make_allreduce(self.group) is not None
        gate = _RoundRobinGate(len(self.ranges)) if collective else None

        def job(k):
            lo, hi = self.ranges[k]
            plan, st = self.plans[k], self.streams[k]
            try:
                st.wait_event(ready)
                with torch.cuda.stream(st):
                    ar = make_allreduce(plan.group)
                    if gate is not None and ar is not None:
                        inner = ar

                        def ar(table, _inner=inner, _k=k):
                            gate.run(_k, lambda: _inner(table))
                    if plan.idx.numel():
                        src_l, cov_l = src.index_select(0, plan.idx), src_cov.index_select(0, plan.idx)
                    else:
                        src_l = torch.zeros((0, 3), dtype=src.dtype, device=src.device)
                        cov_l = torch.zeros((0, 6), dtype=src_cov.dtype, device=src_cov.device)
                    T, infos = g.align_batched_sharded(src_l, cov_l, plan.loffs, plan.gid, plan.num_chunks, plan.B,
                                                       tgt, tgt_cov, T0s[lo:hi], allreduce=ar, **params)
                    done = torch.cuda.Event()
                    done.record(st)
                return np.asarray(T), infos, done
            finally:
                if gate is not None:
                    gate.finish(k)

        out = list(self.pool.map(job, range(len(self.ranges))))
        for _, _, done in out:
            caller.wait_event(done)
        T = np.concatenate([o[0] for o in out])
        infos = [i for o in out for i in o[1]]
        return T, infos


# ---------------------------------------------------------------------------
# Query sharding of the external kNN (config C5)
# ---------------------------------------------------------------------------

class _DevBytes:
    """A uint8 view of a device allocation the library owns (for the collective)."""

    def __init__(self, ptr: int, nbytes: int, device):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
        self.device = device


def broadcast_index(g, index, src: int = 0, group=None, device=None):
    """The index built once on rank `src` and broadcast to every rank (its header as a
    host object, its device buffers over NCCL); the other ranks import owning copies.
    `index` is the built index on `src` (ignored elsewhere). Returns this rank's index."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return index
    if rank == src:
        header, bufs = g.index_export(index)
        meta = [header, [nb for _, nb in bufs]]
    else:
        meta = [None, None]
    dist.broadcast_object_list(meta, src=src, group=group)
    header, sizes = meta
    dev = device if device is not None else (index.device if rank == src else torch.device("cuda"))
    tensors = []
    for i, nb in enumerate(sizes):
        if nb == 0:
            tensors.append(None)
            continue
        if rank == src:
            t = torch.as_tensor(_DevBytes(bufs[i][0], nb, dev), device=dev)
        else:
            t = torch.empty(nb, dtype=torch.uint8, device=dev)
        if dist.get_backend(group) == "nccl":
            dist.broadcast(t, src=src, group=group)
        else:  # gloo (CPU test runs): through host memory
            h = t.cpu()
            dist.broadcast(h, src=src, group=group)
            t.copy_(h)
        tensors.append(t)
    if rank == src:
        return index
    return g.index_import(header, tensors, dev)


def knn_sharded(g, index, q, k: int, group=None, gather: bool = False):
    """External kNN with the queries sharded by contiguous ranges of their cell-sorted
    order (gicp_knn_query_order; spatially coherent shards) over the ranks. Returns
    (nbr, d2, ids): this rank's rows are filled (the others zero) unless gather, which
    adds the shards together with one allreduce (exact: one contributor per row)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    m = q.shape[0]
    perm = g.knn_query_order(index, q)
    lo, hi = (m * rank) // world, (m * (rank + 1)) // world
    ids = perm[lo:hi].contiguous()
    nbr = torch.zeros((m, k), dtype=torch.int32, device=q.device)
    d2 = torch.zeros((m, k), dtype=torch.float32, device=q.device)
    g.knn_subset(index, q, ids, k, (nbr, d2))
    if gather and world > 1:
        ar = make_allreduce(group)
        ar_nbr = nbr.to(torch.float64)  # exact for indices < 2^53
        ar(ar_nbr)
        ar(d2)
        nbr = ar_nbr.to(torch.int32)
    return nbr, d2, ids
