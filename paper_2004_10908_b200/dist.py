"""Multi-GPU driver (SURVEY.md 8.5, row e): one process per GPU, torch.distributed
for the plumbing, NCCL over NVLink for the single collective.

The path shards exactly: row i of Y_{l+1} depends only on row i of Y_l
(invariant I4), so every rank runs the whole network on its own rows against a
replica of the weights (the paper's "up to 4 cudaFlows on 4 GPUs",
PAPER.md:2566, one per GPU) and the only exchange is the final gather of the
category bitmasks -- ceil(rows/32) 32-bit words per rank, 7.5 KB in total at
60,000 inputs.  The category list ("truth categories") is then
decoded identically on every rank.

Partitioning: contiguous slices of `chunk` rows, chunk = ceil(B / P) rounded up
to a multiple of 32, so that concatenating the per-rank bitmask words IS the
global bitmask (bit i%32 of word i//32 = row i) with no re-indexing.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np


def chunk_rows(batch: int, world: int) -> int:
    c = -(-batch // max(world, 1))
    return max(32, -(-c // 32) * 32)


def partition(batch: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) rows of `rank` (may be empty for trailing ranks)."""
    c = chunk_rows(batch, world)
    lo = min(batch, rank * c)
    return lo, min(batch, lo + c)


def slice_csr(rowptr: np.ndarray, idx: np.ndarray, val: Optional[np.ndarray], lo: int, hi: int):
    a, b = int(rowptr[lo]), int(rowptr[hi])
    return ((rowptr[lo:hi + 1] - a).astype(np.int64), idx[a:b],
            None if val is None else val[a:b])


def words_per_rank(batch: int, world: int) -> int:
    return chunk_rows(batch, world) // 32


def gather_bitmask(local_words, group=None):
    """all_gather_into_tensor of every rank's (equal-length, padded) bitmask
    words; returns the global word tensor on the same device."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    local_words = local_words.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty(local_words.numel() * ws, dtype=local_words.dtype,
                          device=local_words.device)
        dist.all_gather_into_tensor(out, local_words, group=group)
        return out
    host = local_words.cpu()                                        # gloo (CPU / single-GPU tests)
    parts = [torch.empty_like(host) for _ in range(ws)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(local_words.device)


def decode(words, batch: int) -> np.ndarray:
    """Global bitmask words -> ascending category ids (< batch)."""
    w = np.ascontiguousarray(np.asarray(words)).view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:batch]
    return np.flatnonzero(bits).astype(np.int32)


def infer_partitioned(net, rowptr: np.ndarray, idx: np.ndarray, val: Optional[np.ndarray],
                      group=None, device=None):
    """Strong-scaling inference of one global batch: this rank infers its
    contiguous slice on its GPU (sdnn_infer_device), then the bitmasks are
    all-gathered (NCCL) and decoded.  Every rank returns the same ascending
    global category ids."""
    import torch
    import torch.distributed as dist
    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    batch = rowptr.size - 1
    lo, hi = partition(batch, ws, rank)
    rp, ix, vv = slice_csr(rowptr, idx, val, lo, hi)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    words = torch.zeros(words_per_rank(batch, ws), dtype=torch.int32, device=dev)
    if hi > lo:
        rp_t = torch.from_numpy(rp).to(dev)
        ix_t = torch.from_numpy(np.ascontiguousarray(ix)).to(dev)
        vv_t = None if vv is None else torch.from_numpy(np.ascontiguousarray(vv)).to(dev)
        net.infer_torch(rp_t, ix_t, vv_t, alive_t=words[: (hi - lo + 31) // 32])
    allw = gather_bitmask(words, group)
    return decode(allw.cpu().numpy(), batch)
