"""Multi-GPU sharding of the linearisation.

The target map/index is replicated on every rank; the source points of a
registration are split into a FIXED global set of chunks (aligned to the
linearize kernel's 256-point blocks, independent of the world size), each rank
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

PPB = 256          # points per linearize block (csrc/linearize.cu kPPB)
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
