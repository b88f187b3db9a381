"""f1: the partitioned inference as ONE GPU task graph
(sdnn_flow_infer) -- explicit graph (cudaFlow), the Algorithm-1 capturer with
1/2/3/4/8 streams, and plain stream launches -- must give exactly the oracle's
categories of the whole batch (PAPER.md:820-900 describes the launch paths; the
arithmetic is unchanged)."""
import numpy as np
import pytest

import oracle
import sdnngen as g
from paper_2004_10908_b200 import dist as sdist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sd():
    from paper_2004_10908_b200 import build
    build.build()
    import paper_2004_10908_b200 as sd
    return sd


def _parts(n, rp, idx, P, dev):
    import torch
    B = rp.size - 1
    out = []
    for r in range(P):
        lo, hi = sdist.partition(B, P, r)
        srp, sidx, _ = sdist.slice_csr(rp, idx, None, lo, hi)
        out.append((torch.from_numpy(srp).to(dev), torch.from_numpy(np.ascontiguousarray(sidx)).to(dev), lo))
    return out


@pytest.mark.parametrize("n,L,B,P", [(1024, 40, 1000, 3), (2048, 24, 777, 4)])
def test_flow_modes_match_oracle(sd, n, L, B, P):
    import torch
    dev = torch.device("cuda", 0)
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(n, B, seed=n + P)
    cats, _, _ = oracle.infer(n, layers, rp, idx, None)
    want = np.flatnonzero(cats)
    assert 0 < want.size < B
    nets = [sd.Net.from_layers(n, layers, fmt="ell") for _ in range(P)]
    try:
        parts = _parts(n, rp, idx, P, dev)
        ntask = None
        for mode, ks in ((sd.SDNN_FLOW_GRAPH, [1]), (sd.SDNN_FLOW_CAPTURER, [1, 2, 3, 4, 8]),
                         (sd.SDNN_FLOW_STREAMS, [1, 3])):
            for k in ks:
                ids, ms, nt = sd.flow_infer(nets, parts, B, mode, max_streams=k, reps=2)
                assert ids.tolist() == want.tolist(), (mode, k)
                assert ms > 0
                ntask = ntask or nt
                assert nt == ntask                          # the same task graph every time
        # P partitions x (densify + chain + readout) + the join
        steps = len(nets[0].step_plan())
        assert ntask > P * (steps + 2)
    finally:
        for x in nets:
            x.close()


def test_flow_rejects_shared_handle(sd):
    import torch
    n, L = 256, 4
    layers = list(g.iter_layers(g.rn_spec(n, L)))
    rp, idx = g.ms_inputs(n, 64, seed=1)
    with sd.Net.from_layers(n, layers) as net:
        parts = _parts(n, rp, idx, 2, torch.device("cuda", 0))
        with pytest.raises(sd.SdnnError):
            sd.flow_infer([net, net], parts, 64, sd.SDNN_FLOW_GRAPH)
