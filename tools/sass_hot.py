"""Top SASS instructions of an ncu report by warp-stall samples (profiling aid).
    ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv
    python tools/sass_hot.py x.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(float(r[iS] or 0) for r in data)
print(f"total samples {tot:.0f}")
agg = {}
for r in data:
    op = r[iSrc].split()[0] if r[iSrc].split() else "?"
    if op.startswith("@"):
        op = r[iSrc].split()[1]
    op = op.split(".")[0]
    agg[op] = agg.get(op, 0) + float(r[iS] or 0)
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]))
top = sorted(data, key=lambda r: -float(r[iS] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    s = float(r[iS] or 0)
    why = sorted(((float(r[h.index(k)] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% {r[0]:>6s} {r[iSrc][:60]:60s} " + " ".join(f"{k}:{v:.0f}" for v, k in why if v))
