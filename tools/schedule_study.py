"""Why the RN generator uses an overlapping field schedule (DESIGN.md R-W2).

Survival of MNIST-shaped inputs (sdnngen.ms_inputs) through un-relabelled
radix-32 butterfly nets under three field schedules, evaluated with the CPU
oracle (test infrastructure; this is a workload study, not part of the product):
  r32     non-overlapping fields 0, 5, 10, ... (full mixing in ceil(log2N/5) layers)
  shift1  p_l = l mod (log2N - 4)
  shift2  p_l = 2l mod (log2N - 4)      (first version: never mixes the top bit)
  rn      sdnngen.rn_field: p_l = (2l + l // ceil(span/2)) mod span   <- used by sdnngen.rn_spec
Run: python tools/schedule_study.py [N] [L] [B]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import sdnngen as g  # noqa: E402


def layer(n, p, bias):
    m = np.arange(n, dtype=np.int64)
    outs = (m & ~np.int64(31 << p))[:, None] | (np.arange(32)[None, :] << p)
    return dict(rowptr=np.arange(0, 32 * (n + 1), 32, dtype=np.int64),
                colidx=outs.reshape(-1).astype(np.int32), val=None,
                uniform=1.0 / 16, bias=np.full(n, bias, np.float32))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 500
    bits = n.bit_length() - 1
    rp, idx = g.ms_inputs(n, B, sentinels=False)
    for name in ["r32", "shift1", "shift2", "rn"]:
        o = oracle.Oracle(n, rp, idx, None)
        prof = []
        for l in range(L):
            if name == "r32":
                offs = list(range(0, bits - 4, 5))
                if offs[-1] != bits - 5:
                    offs.append(bits - 5)
                p = offs[l % len(offs)]
            elif name == "shift1":
                p = l % (bits - 4)
            elif name == "shift2":
                p = (2 * l) % (bits - 4)
            else:
                p = g.rn_field(n, l)
            lay = layer(n, p, g.bias_value(n))
            o.layer(lay["rowptr"], lay["colidx"], None, lay["uniform"], lay["bias"])
            prof.append(o.live_rows())
        pick = [0, 1, 2, 3, 4, 8, 16, L - 1]
        print(f"N={n} {name:7s} live rows after layers {pick}: {[prof[i] for i in pick if i < L]} of {B}")


if __name__ == "__main__":
    main()
