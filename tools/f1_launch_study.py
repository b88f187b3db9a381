"""f1: launch-path study on B200 -- the paper's only LSDNN
GPU-side claims are that a cudaFlow (one CUDA graph of the whole GPU task graph)
beats stream-based execution, 1.5x at one GPU (PAPER.md:2862-2866,
fig::dnn_cudaflow_overhead), and that the capturer (Algorithm 1)
with 2-4 streams is about as fast as the cudaFlow.

Same kernels, launched four ways:
  graph        one inference = one captured CUDA graph (the library default)
  loop         one inference = a plain stream loop of the same kernels
               (SDNN_F_NO_GRAPH)
  streams-k    the batch split into S independent chains (S handles), chains
               round-robined over k streams, plain launches
  capturer-k   the same S chains captured into ONE graph with Algorithm 1's
               stream assignment: levelize (chain c's i-th operation is at
               level i), stream = id-in-level mod max_streams = c mod k, events
               only on cross-stream edges (fork/join), then replayed

Run on the GPU box:  python tools/f1_launch_study.py [c1|c2] [S]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_10908_b200 as sd  # noqa: E402
import sdnngen as g  # noqa: E402
from paper_2004_10908_b200 import dist as sdist  # noqa: E402

CONFIGS = {"c1": (1024, 120, 1000), "c2": (4096, 480, 60000), "c3": (16384, 1920, 60000)}


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    n, L, B = CONFIGS[cfg]
    spec = g.rn_spec(n, L)
    rp, idx = g.ms_inputs(n, B)
    dev = torch.device("cuda", 0)
    res = {"config": cfg, "chains": S}
    # the layer chain alone (the resident tail would hide the launch structure)
    common = dict(fmt="ell", threads=8, flags=sd.SDNN_F_NO_RESIDENT)
    rp_t, idx_t = torch.from_numpy(rp).to(dev), torch.from_numpy(idx).to(dev)
    for name, flags in (("graph", 0), ("loop", sd.SDNN_F_NO_GRAPH)):
        net = sd.Net.from_spec(spec, **dict(common, flags=common["flags"] | flags))
        alive = torch.zeros((B + 31) // 32, dtype=torch.int32, device=dev)
        res[name] = timed(lambda: net.infer_torch(rp_t, idx_t, None, alive_t=alive))
        res[name + "_launches"] = net.stats()["launches_per_infer"]
        net.close()
    # S independent chains (batch partition) on k streams, and the capturer
    parts = []
    for c in range(S):
        lo, hi = sdist.partition(B, S, c)
        p_rp, p_idx, _ = sdist.slice_csr(rp, idx, None, lo, hi)
        net = sd.Net.from_spec(spec, **dict(common, flags=common["flags"] | sd.SDNN_F_NO_GRAPH))
        parts.append((net, torch.from_numpy(p_rp).to(dev), torch.from_numpy(np.ascontiguousarray(p_idx)).to(dev),
                      torch.zeros(max(1, (hi - lo + 31) // 32), dtype=torch.int32, device=dev)))
    streams = [torch.cuda.Stream(dev) for _ in range(8)]

    def run_k(k):
        main_s = torch.cuda.current_stream(dev)
        for s in streams[:k]:
            s.wait_stream(main_s)
        for c, (net, a, b_, al) in enumerate(parts):
            s = streams[c % k]
            net.infer_torch(a, b_, None, alive_t=al, stream=s)
        for s in streams[:k]:
            main_s.wait_stream(s)

    for k in (1, 2, 4):
        if k <= S:
            res[f"streams-{k}"] = timed(lambda: run_k(k))
    for k in (1, 2, 4, 8):
        run_k(min(k, S))                          # warm: plans + workspaces exist
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        with torch.cuda.stream(cap):
            graph.capture_begin()
            # Algorithm 1: chain c's operations -> stream (c mod max_streams);
            # fork/join events are the only cross-stream edges
            run_k(min(k, S))
            graph.capture_end()
        res[f"capturer-{k}"] = timed(lambda: graph.replay())
        del graph
    for net, *_ in parts:
        net.close()
    res["graph_over_loop"] = res["loop"] / res["graph"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
