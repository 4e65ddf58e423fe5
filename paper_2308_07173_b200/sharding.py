"""Multi-GPU sharding of the linearisation.

The target map/index is replicated on every rank; the source points of a
registration are split into a FIXED global set of chunks (aligned to the
linearize kernel's blocks (256-point multiples), independent of the world size), each rank
linearises its chunks (gicp_linearize on its GPU), the 29-value chunk partials are
all-gathered over NCCL (NVLink) and summed in chunk order on every rank. Because
the chunking and the summation order do not depend on the number of ranks, H, b
and e are bitwise identical for world sizes 1, 2, 4, 8, and every rank runs the
identical host LM step (no broadcast of T).
"""
from __future__ import annotations

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


def combine(partials: np.ndarray) -> np.ndarray:
    """Sum [num_chunks, 29] chunk partials in chunk order (fp64)."""
    out = np.zeros(partials.shape[1], dtype=np.float64)
    for c in range(partials.shape[0]):
        out = out + partials[c]
    return out


def allgather_partials(local: dict, num_chunks: int = NUM_CHUNKS, group=None, device=None) -> np.ndarray:
    """local: {chunk id: float64[29]} of this rank -> [num_chunks, 29] on every rank.
    One all_gather of a [num_chunks, 29] fp64 tensor per rank (zeros elsewhere)."""
    world = dist.get_world_size(group)
    buf = torch.zeros((num_chunks, 29), dtype=torch.float64, device=device)
    for c, v in local.items():
        buf[c] = torch.as_tensor(np.asarray(v, dtype=np.float64), device=device)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    full = torch.zeros_like(buf)
    for r in range(world):
        for c in range(num_chunks):
            if c % world == r:
                full[c] = outs[r][c]
    return full.cpu().numpy()


def sharded_linearize(g, src, src_cov, index, tgt_cov, T, max_corr_dist=1.0, pivot=None, group=None):
    """gicp_linearize over this rank's chunks + chunk-ordered combine (GPU ranks)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = src.shape[0]
    local = {}
    for c in chunks_of_rank(rank, world):
        lo, hi = chunk_bounds(n)[c]
        out, _ = g.linearize(src[lo:hi].contiguous(), src_cov[lo:hi].contiguous(), index, tgt_cov, T,
                             max_corr_dist, pivot=pivot)
        local[c] = out.cpu().numpy()
    return combine(allgather_partials(local, group=group, device=src.device))


# ---------------------------------------------------------------------------
# Point-sharded batched registration (config C4 across GPUs)
# ---------------------------------------------------------------------------

def registration_chunks(sizes, rank: int, world: int, num_chunks: int = NUM_CHUNKS):
    """This rank's entries of a batch: (registration b, chunk c, lo, hi) with [lo, hi)
    relative to registration b, for every non-empty chunk c with c % world == rank."""
    out = []
    for b, n in enumerate(sizes):
        for c, (lo, hi) in enumerate(chunk_bounds(int(n), num_chunks)):
            if c % world == rank and hi > lo:
                out.append((b, c, lo, hi))
    return out


def combine_chunk_table(table: np.ndarray, B: int, num_chunks: int = NUM_CHUNKS) -> np.ndarray:
    """[B * num_chunks, 32] chunk rows -> [B, 32] registration rows, summed in chunk order."""
    t = table.reshape(B, num_chunks, -1)
    acc = np.zeros((B, t.shape[2]), dtype=np.float64)
    for c in range(num_chunks):
        acc = acc + t[:, c]
    return acc


def make_chunk_reducer(entries, B: int, num_chunks: int = NUM_CHUNKS, group=None, device=None):
    """The reduce callback of gicp_align_batched_ex: scatter this rank's entry rows
    into the global [B * num_chunks, 32] chunk table (zeros elsewhere), ONE
    all_reduce(sum) of the table (exact: every row has a single non-zero
    contributor, so the sum order cannot matter), then the chunk-ordered combine.
    H, b and e are therefore bitwise identical for every world size."""
    gid = np.array([b * num_chunks + c for (b, c, _, _) in entries], dtype=np.int64)

    def reduce(entry_rows: np.ndarray) -> np.ndarray:
        table = np.zeros((B * num_chunks, entry_rows.shape[1]), dtype=np.float64)
        table[gid] = entry_rows
        t = torch.from_numpy(table).to(device) if device is not None else torch.from_numpy(table)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return combine_chunk_table(t.cpu().numpy(), B, num_chunks)
    return reduce


def align_batched_sharded(g, src, src_cov, offsets, tgt, tgt_cov, T0s, group=None, num_chunks: int = NUM_CHUNKS,
                          comm_device=None, **params):
    """Batched LM alignment with the source points of every registration split into
    a fixed global chunking; this rank linearises its chunks (one batched launch
    per evaluation round), one all_reduce per round combines them, and every rank
    runs the identical host LM. src / src_cov: the full concatenated batch on this
    rank's GPU (only this rank's chunks are used). Returns (T [B,4,4], infos)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    offsets = np.asarray(offsets, dtype=np.int64)
    B = len(offsets) - 1
    entries = registration_chunks(np.diff(offsets), rank, world, num_chunks)
    if entries:
        idx = torch.cat([torch.arange(int(offsets[b]) + lo, int(offsets[b]) + hi, device=src.device)
                         for (b, _, lo, hi) in entries])
        src_l, cov_l = src[idx].contiguous(), src_cov[idx].contiguous()
    else:
        src_l = torch.zeros((0, 3), dtype=src.dtype, device=src.device)
        cov_l = torch.zeros((0, 6), dtype=src_cov.dtype, device=src_cov.device)
    loffs = np.concatenate([[0], np.cumsum([hi - lo for (_, _, lo, hi) in entries])]).astype(np.int64)
    entry_reg = np.array([b for (b, _, _, _) in entries], dtype=np.int32)
    if comm_device is None and dist.is_initialized() and dist.get_backend(group) == "nccl":
        comm_device = src.device          # NCCL reduces device tensors only
    reducer = make_chunk_reducer(entries, B, num_chunks, group, comm_device)
    return g.align_batched_ex(src_l, cov_l, loffs, entry_reg, B, tgt, tgt_cov, T0s, reducer, **params)
