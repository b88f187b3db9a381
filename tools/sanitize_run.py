"""Small inferences through the C ABI for compute-sanitizer (memcheck /
racecheck / synccheck): every kernel path (bulk, register-staged uniform,
general per-slot, K > 32, compaction on/off, graph/stream loop, L = 0)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_10908_b200 as sd  # noqa: E402
import sdnngen as g  # noqa: E402


def run(n, layers, rp, idx, val, flags=0, fmt="csr"):
    with sd.Net.from_layers(n, layers, fmt=fmt, flags=flags) as net:
        cats, Y = net.infer(rp, idx, val, want_y=True)
    return cats, Y


def main():
    out = []
    spec = g.rn_spec(256, 6)
    lays = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(256, 300)
    ref = None
    for flags in (0, sd.SDNN_F_NO_BULK, sd.SDNN_F_NO_GROUPS, sd.SDNN_F_NO_COMPACT, sd.SDNN_F_NO_GRAPH):
        c, Y = run(256, lays, rp, idx, None, flags, fmt="ell")
        if ref is None:
            ref = (c, Y)
        assert np.array_equal(c, ref[0]) and np.array_equal(Y, ref[1])
        out.append(c.size)
    for cap in (64, 128, 256):                       # fused multi-layer passes, T = 128/64/32
        with sd.Net.from_layers(256, lays, fmt="ell", fuse_rows=cap) as net:
            c, Y = net.infer(rp, idx, None, want_y=True)
        assert np.array_equal(c, ref[0]) and np.array_equal(Y, ref[1])
    spec2 = g.rn_spec(1024, 8)                       # 512-row single-CTA and 2-/4-CTA cluster passes
    lays2 = list(g.iter_layers(spec2))
    rp2, idx2 = g.ms_inputs(1024, 200)
    ref2 = None
    for cap in (0, 512, 1024, 2048):
        with sd.Net.from_layers(1024, lays2, fmt="ell", fuse_rows=cap, flags=sd.SDNN_F_NO_RESIDENT) as net:
            c, Y = net.infer(rp2, idx2, None, want_y=True)
        if ref2 is None:
            ref2 = (c, Y)
        assert np.array_equal(c, ref2[0]) and np.array_equal(Y, ref2[1])
    for rf in (0, 3):                                # SMEM-resident tail (P = 32 at N = 256)
        with sd.Net.from_layers(256, lays, fmt="ell", resident_from=rf) as net:
            c, Y = net.infer(rp, idx, None, want_y=True)
        assert np.array_equal(c, ref[0]) and np.array_equal(Y, ref[1])
    spec = g.random_spec(100, 3, seed=5, kmin=0, kmax=40, bias=(-0.3, 0.05))
    lays = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(100, 77, seed=5)
    c, Y = run(100, lays, rp, idx, val)
    out.append(c.size)
    with sd.Net(64, 0) as net:
        c, _ = net.infer(np.array([0, 1, 1], np.int64), np.array([3], np.int32), None)
    out.append(c.size)
    # round 2: per-slot weights on the TMA pipeline (k_layer_bulkw), Y_L row
    # gather, device bitmask decode, the f1 task graph (graph / capturer / streams)
    import torch
    spec = g.rw_spec(1024, 4)
    lays = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(1024, 300, seed=7, density=0.3, lo=0.0, hi=2.0)
    with sd.Net.from_layers(1024, lays, fmt="ell") as net:
        c, Y = net.infer(rp, idx, val, want_y=True)
        rows = np.array([0, 5, 299, 17], np.int32)
        assert np.array_equal(net.gather_rows(rows), Y[rows])
    out.append(c.size)
    w = torch.from_numpy(np.random.default_rng(1).integers(0, 2**31, 40, dtype=np.int64).astype(np.int32)).cuda()
    ids, cnt = sd.bitmask_to_ids_torch(w, 1250)
    torch.cuda.synchronize()
    spec = g.rn_spec(1024, 12)
    lays = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(1024, 400, seed=3)
    nets = [sd.Net.from_layers(1024, lays, fmt="ell") for _ in range(2)]
    parts = []
    for r, (lo, hi) in enumerate([(0, 224), (224, 400)]):
        srp = (rp[lo:hi + 1] - rp[lo]).astype(np.int64)
        sidx = np.ascontiguousarray(idx[rp[lo]:rp[hi]])
        parts.append((torch.from_numpy(srp).cuda(), torch.from_numpy(sidx).cuda(), lo))
    got = [sd.flow_infer(nets, parts, 400, mode, 2, reps=1)[0].tolist()
           for mode in (sd.SDNN_FLOW_GRAPH, sd.SDNN_FLOW_CAPTURER, sd.SDNN_FLOW_STREAMS)]
    assert got[0] == got[1] == got[2]
    for x in nets:
        x.close()
    print("sanitize_run ok", out)


if __name__ == "__main__":
    main()
