"""f1: launch-path study on B200.

The paper's only LSDNN GPU-side claims are that a cudaFlow (one CUDA graph of
the whole GPU task graph) beats stream-based execution, 1.5x at one GPU
(PAPER.md:2862-2866), and that the capturer (Algorithm 1)
with 2-4 streams is about as fast as the cudaFlow.

The task graph is the library's real one (sdnn_flow_infer): the batch split
into P partitions, each on its own handle, per partition densify -> every
kernel of the layer chain -> readout into its slice of the global category
bitmask, joined by the device decode.  Launched as
  graph        explicit DAG (the cudaFlow analogue)
  capturer-k   Algorithm 1 with max_streams = k, captured into one graph
  streams-k    Algorithm 1's stream assignment launched directly (no graph)
plus, for reference, the single-handle inference (one captured graph, and the
same kernels as a plain stream loop, SDNN_F_NO_GRAPH).  Every mode's category
ids are compared with the single-handle result (the GPU tests compare them
with the oracle).

Run on the GPU box:  python tools/f1_launch_study.py [c1|c2|c3] [P]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_10908_b200 as sd  # noqa: E402
import sdnngen as g  # noqa: E402
from paper_2004_10908_b200 import dist as sdist  # noqa: E402

CONFIGS = {"c1": (1024, 120, 1000), "c2": (4096, 480, 60000), "c3": (16384, 1920, 60000)}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    n, L, B = CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    spec = g.rn_spec(n, L)
    rp, idx = g.ms_inputs(n, B)
    rp_t, idx_t = torch.from_numpy(rp).to(dev), torch.from_numpy(idx).to(dev)
    out = {"config": cfg, "partitions": P}
    # single handle: one captured graph vs the same kernels as a stream loop
    ref = None
    for name, flags in (("single-graph", 0), ("single-loop", sd.SDNN_F_NO_GRAPH)):
        with sd.Net.from_spec(spec, fmt="ell", flags=flags | sd.SDNN_F_NO_RESIDENT) as net:
            for _ in range(2):
                a = net.infer_torch(rp_t, idx_t)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                a = net.infer_torch(rp_t, idx_t)
            e1.record()
            torch.cuda.synchronize()
            out[name] = round(e0.elapsed_time(e1) / 5, 3)
            ids = sd.bitmask_to_ids(a.cpu().numpy(), B)
            ref = ids if ref is None else ref
            assert np.array_equal(ids, ref)
            out[name + "_launches"] = net.stats()["launches_per_infer"]
    nets = [sd.Net.from_spec(spec, fmt="ell", flags=sd.SDNN_F_NO_RESIDENT) for _ in range(P)]
    parts = []
    for r in range(P):
        lo, hi = sdist.partition(B, P, r)
        srp, sidx, _ = sdist.slice_csr(rp, idx, None, lo, hi)
        parts.append((torch.from_numpy(srp).to(dev), torch.from_numpy(np.ascontiguousarray(sidx)).to(dev), lo))
    ids, ms, nt = sd.flow_infer(nets, parts, B, sd.SDNN_FLOW_GRAPH, 1, reps=5)
    assert np.array_equal(ids, ref)
    out["tasks"] = nt
    out["graph"] = round(ms, 3)
    for mode, name in ((sd.SDNN_FLOW_CAPTURER, "capturer"), (sd.SDNN_FLOW_STREAMS, "streams")):
        for k in (1, 2, 4, 8):
            ids, ms, _ = sd.flow_infer(nets, parts, B, mode, k, reps=5)
            assert np.array_equal(ids, ref), (name, k)
            out[f"{name}-{k}"] = round(ms, 3)
    for x in nets:
        x.close()
    out["graph_over_best_streams"] = round(min(out[f"streams-{k}"] for k in (1, 2, 4, 8)) / out["graph"], 3)
    out["single_graph_over_loop"] = round(out["single-loop"] / out["single-graph"], 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
