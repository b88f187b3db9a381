"""Repeat the C1 full-batch parity run (flags/fmt from argv) and report every
mismatching (row, neuron) range -- a nondeterminism probe."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import sdnngen as g
import paper_2004_10908_b200 as sd

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
combos = [(int(f), fm) for f in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1"])
          for fm in ("csr", "ell")]
layers = list(g.iter_layers(g.rn_spec(1024, 120)))
rp, idx = g.ms_inputs(1024, 1000)
oc, oY, _ = oracle.infer(1024, layers, rp, idx, None)
bad = 0
for flags, fmt in combos:
    for r in range(reps):
        with sd.Net.from_layers(1024, layers, fmt=fmt, flags=flags) as net:
            cats, Y = net.infer(rp, idx, None, want_y=True)
            plan = net.step_plan()
        d = Y.view(np.uint32) != oY.view(np.uint32)
        ok = np.array_equal(cats, np.flatnonzero(oc)) and not d.any()
        if not ok:
            bad += 1
            rows = np.flatnonzero(d.any(1))
            print(f"flags={flags} fmt={fmt} rep={r}: {d.sum()} bad elements in rows {rows[:20].tolist()}",
                  "cols of first:", np.flatnonzero(d[rows[0]])[:8].tolist(), "..", np.flatnonzero(d[rows[0]])[-4:].tolist())
        else:
            print(f"flags={flags} fmt={fmt} rep={r}: ok")
    print("plan", plan if len(str(plan)) < 400 else str(plan)[:400])
print("BAD", bad)
