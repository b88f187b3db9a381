"""Multi-process (world_size 2, gloo, CPU) checks of the multi-GPU host logic in
paper_2004_10908_b200/dist.py: contiguous partition, per-rank bitmask, gather,
decode.  The per-rank inference is stood in for by the CPU oracle (test
infrastructure) so the sharding logic is exercised end to end without a GPU;
on a GPU box the same functions wrap sdnn_infer_device (bench.py, N > 1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import sdnngen as g
from paper_2004_10908_b200 import dist as sdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, L, B, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = g.rn_spec(n, L)
        layers = list(g.iter_layers(spec))
        rp, idx = g.ms_inputs(n, B, seed=123)
        lo, hi = sdist.partition(B, world, rank)
        srp, sidx, _ = sdist.slice_csr(rp, idx, None, lo, hi)
        words = np.zeros(sdist.words_per_rank(B, world), np.uint32)
        if hi > lo:
            cats, _, _ = oracle.infer(n, layers, srp, sidx, None, nthreads=1)
            bits = np.packbits(cats.astype(np.uint8), bitorder="little")
            words.view(np.uint8)[:bits.size] = bits
        allw = sdist.gather_bitmask(torch.from_numpy(words.view(np.int32)))
        q.put((rank, sdist.decode(allw.numpy(), B).tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [333, 64, 31])
def test_partition_gather_decode_world2(B):
    n, L, world = 256, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, L, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = g.rn_spec(n, L)
    rp, idx = g.ms_inputs(n, B, seed=123)
    cats, _, _ = oracle.infer(n, g.iter_layers(spec), rp, idx, None)
    want = np.flatnonzero(cats).tolist()
    assert res[0] == want and res[1] == want


@pytest.mark.parametrize("B,world", [(60000, 8), (60000, 3), (31, 4), (0, 2), (65, 2)])
def test_partition_covers_rows_exactly(B, world):
    spans = [sdist.partition(B, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == B
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    c = sdist.chunk_rows(B, world)
    assert c % 32 == 0
    for r, (a, b) in enumerate(spans):
        assert a == min(B, r * c)               # word-aligned: concatenation == global mask


def test_decode_roundtrip():
    r = np.random.default_rng(0)
    ids = np.sort(r.choice(1000, 77, replace=False))
    bits = np.zeros(1024, np.uint8)
    bits[ids] = 1
    words = np.packbits(bits, bitorder="little").view(np.uint32)
    assert sdist.decode(words, 1000).tolist() == ids.tolist()
