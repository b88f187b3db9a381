"""Helper for test_opt_in_knobs (run in a subprocess so that the library reads
the environment knobs afresh): N = 4096 RN net whose plan has 1024-row passes
with 16-position tiles; prints OK when categories and Y_L match the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2004_10908_b200 as sd  # noqa: E402
import sdnngen as g  # noqa: E402

n, L, B = 4096, 24, 700
# SDNN_KNOB_NET=rw: the per-slot-weight variant of the same structure
spec = g.rw_spec(n, L) if os.environ.get("SDNN_KNOB_NET") == "rw" else g.rn_spec(n, L)
layers = list(g.iter_layers(spec))
rp, idx = g.ms_inputs(n, B, seed=11)
cats, Y, prof = oracle.infer(n, layers, rp, idx, None, profile=True)
with sd.Net.from_layers(n, layers, fmt="ell", flags=int(sys.argv[1]) if len(sys.argv) > 1 else 0) as net:
    cg, Yg = net.infer(rp, idx, None, want_y=True)
    st = net.stats()
if os.environ.get("SDNN_KNOB_NET") != "rw" or os.environ.get("SDNN_PASS_GENERAL") == "1":
    assert st["path"] & 4, "expected the position-blocked plan"
assert np.array_equal(cg, np.flatnonzero(cats))
assert np.array_equal(Yg.view(np.uint32), Y.view(np.uint32))
assert st["live_rows"] == prof
print("OK", cg.size)
