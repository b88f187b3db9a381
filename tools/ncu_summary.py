"""Summarise ncu outputs for profiles/: a launch list CSV (gpu__time_duration)
into per-kernel shares, and a --set full report into the key metrics.
    python tools/ncu_summary.py launches <csv>
    python tools/ncu_summary.py full <ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'avg us':>9s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {c:8d} {t:10.2f} {100 * t / tot:5.1f}% {1e3 * t / c:9.1f}")
    print(f"{'total':44s} {sum(c for c, _ in agg.values()):8d} {tot:10.2f}")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name[:100]}")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:62s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
