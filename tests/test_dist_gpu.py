"""Multi-process GPU path with the real CUDA library: two ranks share cuda:0
(only one GPU is available in this environment, and NCCL refuses two ranks on
one device, so the collective runs over gloo), each infers its contiguous
slice with sdnn_infer_device, the bitmasks are all-gathered and decoded, and
every rank must return exactly the oracle's categories of the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2004_10908_b200 as sd
    import sdnngen as g
    from paper_2004_10908_b200 import dist as sdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, L, B = 1024, 40, 777
        spec = g.rn_spec(n, L)
        rp, idx = g.ms_inputs(n, B, seed=4242)
        with sd.Net.from_spec(spec, fmt="ell", threads=4, device=0) as net:
            ids = sdist.infer_partitioned(net, rp, idx, None, device=torch.device("cuda", 0))
        q.put((rank, ids.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_gpu_matches_oracle():
    import oracle
    import sdnngen as g
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    spec = g.rn_spec(1024, 40)
    rp, idx = g.ms_inputs(1024, 777, seed=4242)
    cats, _, _ = oracle.infer(1024, g.iter_layers(spec), rp, idx, None)
    want = np.flatnonzero(cats).tolist()
    assert res[0] == want and res[1] == want and 0 < len(want) < 777
