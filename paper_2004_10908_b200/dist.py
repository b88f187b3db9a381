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


class NvlsGather:
    """f4: the category gather fused into the readout kernel over NVLink SHARP
    (sdnn_infer_device_nvls).  Two word buffers (alternating by call parity)
    and an arrival counter live in one torch symmetric-memory allocation whose
    multicast mapping the readout kernel stores through (multimem.st); the
    all_gather_into_tensor path (gather_bitmask) is the checked equivalent.
    Raises RuntimeError when the group has no multicast mapping (no NVLS)."""

    def __init__(self, total_words: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.group = group or dist.group.WORLD
        self.ws = dist.get_world_size(self.group)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.nw = int(total_words)
        self.stride = -(-self.nw // 32) * 32                    # words per buffer (128 B aligned)
        self.buf = symm.empty(2 * self.stride + 32, dtype=torch.int32, device=self.dev)
        self.buf.zero_()
        self.hdl = symm.rendezvous(self.buf, self.group.group_name)
        if not getattr(self.hdl, "multicast_ptr", 0):
            raise RuntimeError("no NVLS multicast mapping for this group")
        self.hdl.barrier()
        self.calls = 0
        # one checked round trip through the multicast counter before relying
        # on it (the wait gives up after ~4 s rather than hang)
        import ctypes
        from paper_2004_10908_b200 import lib, _check
        base, mc, flag = self.buf.data_ptr(), self.hdl.multicast_ptr, 4 * 2 * self.stride
        self.calls = 1
        _check(lib().sdnn_nvls_barrier(ctypes.c_void_p(base + flag), ctypes.c_void_p(mc + flag),
                                        self.ws, torch.cuda.current_stream(self.dev).cuda_stream))
        torch.cuda.synchronize(self.dev)
        ok = torch.tensor([int(self.timed_out() == 0)], dtype=torch.int32, device=self.dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if int(ok.item()) != 1:
            raise RuntimeError("NVLS multicast counter did not reach every rank")

    def timed_out(self) -> int:
        """1 if a wait on the arrival counter gave up (results invalid)."""
        return int(self.buf[2 * self.stride + 1].item())

    def params(self, word_offset: int):
        """sdnn_nvls for the next call; returns (struct, the local word tensor it fills)."""
        from paper_2004_10908_b200 import sdnn_nvls
        b = self.calls % 2
        self.calls += 1
        base, mc = self.buf.data_ptr(), self.hdl.multicast_ptr
        off, flag = 4 * b * self.stride, 4 * 2 * self.stride
        nv = sdnn_nvls(base + off, mc + off, base + flag, mc + flag, int(word_offset),
                       self.calls * self.ws)
        return nv, self.buf[b * self.stride: b * self.stride + self.nw]


def decode(words, batch: int) -> np.ndarray:
    """Host decode of global bitmask words -> ascending category ids (< batch);
    the CPU/gloo path (the GPU path decodes on the device, decode_device)."""
    w = np.ascontiguousarray(np.asarray(words)).view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:batch]
    return np.flatnonzero(bits).astype(np.int32)


def decode_device(words_t, batch: int, stream=None):
    """Device decode (sdnn_bitmask_to_ids kernel): (ids tensor, count tensor)."""
    from paper_2004_10908_b200 import bitmask_to_ids_torch
    return bitmask_to_ids_torch(words_t, batch, stream)


class Partitioned:
    """Strong-scaling inference of one global batch over the process group:
    this rank owns the contiguous word-aligned slice partition(B, P, rank) of
    the rows, infers it on its GPU against its replica of the weights
    (sdnn_infer_device), then the bitmask words are all-gathered over NCCL and
    decoded on the device into the ascending global category ids.  Inputs
    arrive from (pinned) host memory each call (the end-to-end path); the
    staging tensors are allocated once."""

    def __init__(self, net, batch: int, group=None, device=None, nvls: Optional[bool] = None):
        import torch
        import torch.distributed as dist
        self.net, self.batch, self.group = net, int(batch), group
        self.ws, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.lo, self.hi = partition(self.batch, self.ws, self.rank)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.words = torch.zeros(words_per_rank(self.batch, self.ws), dtype=torch.int32, device=self.dev)
        self._rp = self._ix = None
        # f4: fused NVLS gather when asked (nvls=True) or, by default, when the
        # group has a multicast mapping; otherwise the NCCL all-gather
        self.nvls = None
        if nvls is not False and dist.get_backend(group) == "nccl":
            try:
                self.nvls = NvlsGather(words_per_rank(self.batch, self.ws) * self.ws, group, self.dev)
            except Exception:
                if nvls:
                    raise

    def slice(self, rowptr, idx):
        return slice_csr(rowptr, idx, None, self.lo, self.hi)[:2]

    def __call__(self, rp_local, idx_local, stream=None):
        """rp_local/idx_local: this rank's slice (host numpy, ideally pinned).
        Returns the global ascending category ids (numpy) on every rank."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.dev)
        if self._rp is None or self._rp.numel() < rp_local.size or self._ix.numel() < max(1, idx_local.size):
            self._rp = torch.empty(rp_local.size, dtype=torch.int64, device=self.dev)
            self._ix = torch.empty(max(1, idx_local.size), dtype=torch.int32, device=self.dev)
        with torch.cuda.stream(s):
            rp_t = self._rp[:rp_local.size]
            ix_t = self._ix[:max(1, idx_local.size)]
            rp_t.copy_(torch.from_numpy(rp_local), non_blocking=True)
            if idx_local.size:
                ix_t[:idx_local.size].copy_(torch.from_numpy(idx_local), non_blocking=True)
            if self.nvls is not None:
                nv, allw = self.nvls.params(self.lo // 32)
                self.net.infer_torch_nvls(rp_t, ix_t, nv, stream=s)
            else:
                self.words.zero_()
                if self.hi > self.lo:
                    self.net.infer_torch(rp_t, ix_t, None, alive_t=self.words[: (self.hi - self.lo + 31) // 32],
                                         stream=s)
                allw = gather_bitmask(self.words, self.group)
            ids, cnt = decode_device(allw, self.batch, s)
            n = int(cnt.item())                                  # D2H: the count, then the ids
            if self.nvls is not None and self.nvls.timed_out():
                raise RuntimeError("NVLS gather: a rank never arrived (result invalid)")
            return ids[:n].cpu().numpy()


def infer_partitioned(net, rowptr: np.ndarray, idx: np.ndarray, val: Optional[np.ndarray],
                      group=None, device=None):
    """Strong-scaling inference of one global batch (see Partitioned); every
    rank returns the same ascending global category ids."""
    import torch
    ws, rank = dist_world(group)
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
    ids, cnt = decode_device(allw, batch)
    return ids[:int(cnt.item())].cpu().numpy()


def dist_world(group=None):
    import torch.distributed as dist
    return dist.get_world_size(group), dist.get_rank(group)
