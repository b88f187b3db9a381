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


def _worker_e2e(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2004_10908_b200 as sd
    import sdnngen as g
    from paper_2004_10908_b200 import dist as sdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, L, B = 1024, 30, 1001
        spec = g.rn_spec(n, L)
        rp, idx = g.ms_inputs(n, B, seed=77)
        with sd.Net.from_spec(spec, fmt="ell", threads=4, device=0) as net:
            part = sdist.Partitioned(net, B, device=torch.device("cuda", 0))
            srp, sidx = part.slice(rp, idx)
            srp = torch.from_numpy(srp).pin_memory().numpy()
            sidx = torch.from_numpy(np.ascontiguousarray(sidx)).pin_memory().numpy()
            a = part(srp, sidx)
            b = part(srp, sidx)                       # staging reused
        q.put((rank, a.tolist(), b.tolist()))
    finally:
        dist.destroy_process_group()


def test_partitioned_e2e_device_decode():
    """The multi-GPU end-to-end call (dist.Partitioned: pinned host slice ->
    H2D -> sdnn_infer_device -> all-gather -> k_bitmask_ids on the device ->
    D2H of the ids) returns the oracle's global categories on every rank."""
    import oracle
    import sdnngen as g
    world = 3                                          # ragged: 1001 rows = 352 + 352 + 297
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_e2e, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, a, b = q.get(timeout=600)
        res[r] = (a, b)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cats, _, _ = oracle.infer(1024, g.iter_layers(g.rn_spec(1024, 30)), *g.ms_inputs(1024, 1001, seed=77), None)
    want = np.flatnonzero(cats).tolist()
    assert 0 < len(want) < 1001
    for r in range(world):
        assert res[r][0] == want and res[r][1] == want


def test_bitmask_to_ids_kernel():
    """k_bitmask_ids against a host decode: random words, bits past the batch
    ignored, empty batch."""
    import torch

    import paper_2004_10908_b200 as sd
    r = np.random.default_rng(3)
    for batch in (0, 1, 31, 32, 33, 1000, 60000, 65537):
        nw = max(1, (batch + 31) // 32)
        w = r.integers(0, 2 ** 32, size=nw, dtype=np.uint64).astype(np.uint32)
        w[r.random(nw) < 0.3] = 0
        t = torch.from_numpy(w.view(np.int32)).cuda()
        ids, cnt = sd.bitmask_to_ids_torch(t, batch)
        torch.cuda.synchronize()
        want = sd.bitmask_to_ids(w, batch)
        assert int(cnt.item()) == want.size
        assert ids[: want.size].cpu().numpy().tolist() == want.tolist()


def test_bench_two_ranks_strong_scaling(tmp_path):
    """bench.py under torchrun with 2 ranks (sharing the one GPU; gloo for the
    collective since NCCL refuses two ranks per device): one 1,000-input batch
    split across the ranks (strong scaling), per-rank times reported."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SDNN_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
                          "--config", "c1", "--steps", "3", "--warmup", "3", "--e2e-steps", "2"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["scaling"] == "strong" and line["n_gpus"] == 2
    assert line["config"]["global_batch"] == 1000
    m = line["multi_gpu"]
    assert len(m["per_rank_ms"]) == 2 and m["imbalance_max_over_mean"] >= 1.0
    assert m["rows_per_rank"] == [512, 488]
    assert line["e2e"]["value"] > 0


def _worker_nvls(port, q):
    import torch
    import torch.distributed as dist

    import paper_2004_10908_b200 as sd
    import sdnngen as g
    from paper_2004_10908_b200 import dist as sdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        n, L, B = 1024, 30, 999
        spec = g.rn_spec(n, L)
        rp, idx = g.ms_inputs(n, B, seed=5)
        rp_t, idx_t = torch.from_numpy(rp).to(dev), torch.from_numpy(idx).to(dev)
        try:
            nvg = sdist.NvlsGather((B + 31) // 32, device=dev)
        except Exception as e:                              # no multicast on this box
            q.put(("skip", repr(e)))
            return
        out = []
        with sd.Net.from_spec(spec, fmt="ell", threads=4, device=0) as net:
            ref = net.infer_torch(rp_t, idx_t).clone()
            for _ in range(3):                              # both buffers, counter epochs 1..3
                nv, allw = nvg.params(0)
                net.infer_torch_nvls(rp_t, idx_t, nv)
                ids, cnt = sdist.decode_device(allw, B)
                torch.cuda.synchronize()
                out.append(ids[: int(cnt.item())].cpu().numpy().tolist())
        want = sd.bitmask_to_ids(ref.cpu().numpy(), B).tolist()
        q.put(("ok", out, want))
    finally:
        dist.destroy_process_group()


def test_nvls_fused_readout_world1():
    """f4: the readout kernel that stores the category words through the NVLS
    multicast mapping (multimem.st) and waits on the arrival counter, with a
    one-rank NCCL group (the only topology available here): the gathered
    bitmask must equal the plain readout's, on three consecutive calls."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker_nvls, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    if res[0] == "skip":
        pytest.skip("no NVLS multicast mapping: " + res[1])
    assert p.exitcode == 0
    _, out, want = res
    assert 0 < len(want) < 999
    assert all(o == want for o in out)
