"""Binding-level utilisation of one ncu --set full capture (raw CSV page), for
profiles/: HBM (against MEASURED_PEAKS.json), L2, L1/shared, FMA pipe, issue.
    python tools/ncu_levels.py <raw.csv> [label]   -> one JSON line
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def levels(path, label=None):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (num(v[i]), u[i]) for i in range(len(h))}
    get = lambda k: d.get(k, (None, ""))[0]       # noqa: E731
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tunit = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0}
    rd = get("dram__bytes_read.sum") * scale.get(d["dram__bytes_read.sum"][1], 1)
    wr = get("dram__bytes_write.sum") * scale.get(d["dram__bytes_write.sum"][1], 1)
    t = get("gpu__time_duration.sum") * tunit.get(d["gpu__time_duration.sum"][1], 1e-9)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6454.3
    out = {
        "kernel": label or v[h.index("Kernel Name")][:80],
        "duration_ms": t * 1e3,
        "dram_bytes": rd + wr,
        "hbm_gbs": (rd + wr) / t / 1e9,
        "hbm_frac_of_measured": (rd + wr) / t / 1e9 / peak,
        "dram_pct_of_ncu_peak": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_pct": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "l1_pct": get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
        "smem_wavefront_pct": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "smem_bank_conflict_share": (get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") or 0) /
        max(1.0, get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or 1),
        "fma_pipe_pct": get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "lsu_pipe_pct": get("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "issue_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": get("launch__registers_per_thread"),
        "source": os.path.basename(path),
    }
    return out


if __name__ == "__main__":
    print(json.dumps(levels(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)))
