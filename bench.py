#!/usr/bin/env python
"""Benchmark of the sparse-DNN inference hot path (BASELINE.json metric:
edges/sec = inputs x sum_l nnz(W_l) / time, 65536-neuron x 1920-layer net).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference          # the CPU oracle, timed on host cores

A step is one whole inference (all hot-path rows a2-a6): densify the input
CSR, run every layer (one captured CUDA Graph), read out the categories and,
for N > 1, all-gather the category bitmasks over NCCL.  Inputs are resident in
HBM when the timed region starts (`value`); `e2e` repeats the measurement
through the host-buffer call sdnn_infer (H2D of Y0 + D2H of the categories
inside the timed region).  Multi-GPU (torchrun, N > 1) is strong scaling by
default, BASELINE configs[3]: the one 60,000-input batch is split into
word-aligned contiguous row slices, every rank infers its slice against its
replica of the weights, the category bitmasks are all-gathered over NCCL and
decoded on the device; --scaling weak gives every rank
its own 60,000-input batch.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (neurons, layers, inputs) -- BASELINE.json "configs"
    "c1": (1024, 120, 1000),
    "c2": (4096, 480, 60000),
    "c3": (16384, 1920, 60000),
    "c4": (65536, 1920, 60000),
}
# configs[4]: the width/depth sweep for roofline and scaling curves (tools/sweep.sh)
for _n in (1024, 4096, 16384, 65536):
    for _l in (120, 480, 1920):
        CONFIGS[f"s{_n}x{_l}"] = (_n, _l, 60000)
METRIC = "edges/sec (inputs×nnz/time) for 65536-neuron×1920-layer net at 1/2/4/8 B200"
UNIT = "edges/s"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def lib_flags(sd, names):
    f = 0
    for nm in filter(None, names.split(",")):
        f |= getattr(sd, "SDNN_F_" + nm.upper())
    return f


NETS = {
    # --net: (spec factory, description)
    "rn": (lambda g, n, L: g.rn_spec(n, L),
           "RadiX-Net-shaped (sdnngen.rn_spec), overlapping field schedule, uniform w=1/16"),
    "rn-plain": (lambda g, n, L: g.rn_plain_spec(n, L),
                 "RadiX-Net-shaped, SURVEY 8.4 non-overlapping field schedule (sdnngen.rn_plain_spec), "
                 "uniform w=1/16"),
    "rw": (lambda g, n, L: g.rw_spec(n, L),
           "RadiX-Net-shaped structure with per-slot weights U(-0.05,0.15) (sdnngen.rw_spec): "
           "the general-weight path"),
    "rr": (lambda g, n, L: g.rr_spec(n, L),
           "random 32-regular, no shared source sets (sdnngen.rr_spec), uniform w=1/16"),
}


def net_spec(g, args, n, L):
    """The network family (NETS): rn is the headline; rn-plain, rw and rr are
    robustness rows reported beside it."""
    return NETS[args.net][0](g, n, L)


def schedule_desc(g, spec):
    """The field schedule of an RN-structured net (disclosed in `config`)."""
    if spec.kind != "rn":
        return None
    sch = spec.extra.get("schedule", "overlap")
    first = [g.rn_field(spec.n, l, sch) for l in range(min(spec.L, 24))]
    formula = ("p_l = (2l + floor(l/c)) mod (log2N-4), c = ceil((log2N-4)/2): consecutive 5-bit fields "
               "overlap in 3 bits (DESIGN.md R-W2)" if sch == "overlap" else
               "non-overlapping 5-bit fields 0, 5, 10, ... (last clamped to log2N-5), SURVEY.md 8.4")
    return {"name": sch, "formula": formula, "first_fields": first}


def kernel_name(net, args=None):
    st = net.stats()
    if st.get("fused_layers", 0) == 0:
        return "k_layer_bulkw" if args is not None and args.net == "rw" else "k_layer_bulk"
    return "fused passes (k_pass_t32 / k_pass_wide / k_pass)"


def make_inputs(n, B, rank):
    import sdnngen as g
    seed = g.input_seed(n) if rank == 0 else g.input_seed(n) ^ (0x9E37 * rank)
    return g.ms_inputs(n, B, seed=seed)


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    """The CPU oracle as it stands, on the GPU arm's workload: each step infers a
    bounded sample of the 60,000 inputs through all layers; edges/s counts
    sample_rows x sum nnz per oracle-second (generation of the layers excluded)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import sdnngen as g
    n, L, B = CONFIGS[args.config]
    spec = net_spec(g, args, n, L)
    rp, idx = make_inputs(n, B, 0)
    cores = oracle.default_threads()
    rows_per_step = args.ref_rows or max(1, cores)
    r = np.random.default_rng(1234)
    nsteps = args.warmup + args.steps
    samples = [np.sort(r.choice(B, rows_per_step, replace=False)) for _ in range(nsteps)]
    objs = []
    for rows in samples:
        srp, sidx, _ = oracle.subset_rows(rp, idx, None, rows)
        objs.append(oracle.Oracle(n, srp, sidx, None))
    total_nnz = 0
    for l in range(L):
        lay = g.gen_layer(spec, l, fmt="csr" if spec.wdist == "uniform" else "both")
        total_nnz += lay.colidx.size
        for o in objs:
            o.apply(lay, nthreads=cores)
    secs = [o.layer_seconds for o in objs[args.warmup:]]
    t = sum(secs) / len(secs)
    value = rows_per_step * total_nnz / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{args.net}{n}x{L}-ms{B}", "neurons": n, "layers": L,
                   "nnz_per_column": 32, "inputs_sampled_per_step": rows_per_step, "inputs_full": B,
                   "global_batch": B},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{rows_per_step} random rows of the {B}-input batch per step, "
                                   f"all {L} layers (oracle/sdnn_oracle.c, {cores} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(n, L, spec, rp, idx, rows):
    """Bounded oracle sample timed on host cores (rank 0, N = 1 only)."""
    import oracle
    cores = oracle.default_threads()
    t0 = time.time()
    _, _, _, secs = oracle.infer_spec_rows(spec, rp, idx, None, rows, nthreads=cores)
    total_nnz = 32 * n * L
    return {"value": rows.size * total_nnz / secs, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{rows.size} random rows of the 60000-input batch, all {L} layers "
                      f"({secs:.1f} s oracle time, {time.time() - t0:.1f} s incl. layer generation)"}


# ---------------------------------------------------------------- GPU arm

def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2004_10908_b200 as sd
    import sdnngen as g

    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())   # >1 rank per GPU only in tests
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        backend = os.environ.get("SDNN_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2004_10908_b200 import dist as sdist
    n, L, B = CONFIGS[args.config]
    spec = net_spec(g, args, n, L)
    t0 = time.time()
    net = sd.Net.from_spec(spec, fmt="ell", threads=args.load_threads, device=local,
                           flags=sd.SDNN_F_PROFILE | lib_flags(sd, args.flags),
                           fuse_rows=args.fuse_rows, fuse_layers=args.fuse_layers,
                           stream_slots=args.stream_slots)
    t_load = time.time() - t0
    strong = args.scaling == "strong"
    if strong:
        # one global batch, contiguous word-aligned slices (dist.partition)
        rp, idx = make_inputs(n, B, 0)
        lo, hi = sdist.partition(B, ws, rank)
        rp, idx, _ = sdist.slice_csr(rp, idx, None, lo, hi)
        words = sdist.words_per_rank(B, ws)
    else:
        # weak scaling: every rank its own B-input batch (seeded by rank)
        rp, idx = make_inputs(n, B, rank)
        words = (B + 31) // 32
    batch = rp.size - 1
    rp_t = torch.from_numpy(rp).to(dev)
    idx_t = torch.from_numpy(np.ascontiguousarray(idx)).to(dev)
    alive = torch.zeros(words, dtype=torch.int32, device=dev)
    alive_view = alive[: (batch + 31) // 32]
    stream = torch.cuda.current_stream(dev)

    gB = B if strong else batch * ws                  # rows of the global bitmask
    gev = []                                          # (before, after) the collective, per timed step
    # f4: the gather fused into the readout over NVLS multicast when the group
    # has one (--gather auto), else / with --gather nccl the NCCL all-gather
    nvg = None
    if ws > 1 and args.gather != "nccl" and dist.get_backend() == "nccl":
        try:
            nvg = sdist.NvlsGather(words * ws, device=dev)
        except Exception as e:                        # no multicast mapping
            if args.gather == "nvls":
                raise
            print(f"NVLS gather unavailable ({e}); NCCL all-gather", file=sys.stderr)
    lo_row = sdist.partition(B, ws, rank)[0] if strong else rank * batch

    def step(timed=False):
        if nvg is not None:
            nv, allw = nvg.params(lo_row // 32)
            net.infer_torch_nvls(rp_t, idx_t, nv, stream=stream)
            sdist.decode_device(allw, gB, stream)
            return
        net.infer_torch(rp_t, idx_t, None, alive_t=alive_view, stream=stream)
        if ws > 1:
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            allw = sdist.gather_bitmask(alive)          # the single collective (NCCL all-gather)
            if timed:
                e1.record(stream)
                gev.append((e0, e1))
            sdist.decode_device(allw, gB, stream)      # global ascending ids, on the device

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step(timed=True)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = net.stats()
    layer_ms = net.layer_times()                     # per-layer kernel durations, last step
    if nvg is not None and nvg.timed_out():
        raise RuntimeError("NVLS gather timed out on this rank: the measurement is invalid")
    multi = None
    if ws > 1:
        gms = sum(a.elapsed_time(b) for a, b in gev) / max(1, len(gev)) if gev else None
        got = [None] * ws
        dist.all_gather_object(got, [ms, gms])
        allt = np.array([[x if x is not None else np.nan for x in r] for r in got], np.float64).reshape(ws, 2)
        per_rank = allt[:, 0].tolist()
        ms = float(allt[:, 0].max())
        multi = {"per_rank_ms": per_rank, "imbalance_max_over_mean": ms / float(np.mean(per_rank)),
                 "allgather_ms_per_step": (float(np.nanmax(allt[:, 1])) if nvg is None else None),
                 "gather": ("nvls: readout kernel stores the category words through the multicast "
                            "mapping (multimem.st) + arrival counter (k_readout_nvls)" if nvg is not None
                            else "nccl all_gather_into_tensor"),
                 "rows_per_rank": [int(min(B, (r + 1) * sdist.chunk_rows(B, ws)) - min(B, r * sdist.chunk_rows(B, ws)))
                                   for r in range(ws)] if strong else [batch] * ws,
                 "collective": "torch.distributed.all_gather_into_tensor (NCCL) of ceil(rows/32) "
                               "uint32 bitmask words per rank, then k_bitmask_ids on every rank"}
    total_nnz = st["total_nnz"]
    edges_rank = batch * total_nnz
    value = edges_rank * ws / (ms * 1e-3) if not strong else B * total_nnz / (ms * 1e-3)

    # ---- roofline of the dominant kernels (the layer steps) ---------------------
    # A step (one kernel) runs m layers: k_layer_bulk (m = 1) or a fused pass
    # k_pass (m > 1).  Its algorithmic HBM traffic: read every neuron row of the
    # rows entering the step (4 B) and write every output row (4 B) once,
    # = 8 * N bytes per live row per STEP (intermediate layers stay in SMEM).
    live = st["live_rows"]
    kept0 = st["kept_rows"]
    live_in = [kept0] + live[:-1]                    # rows entering each layer
    plan = net.step_plan()
    starts = np.cumsum([0] + plan[:-1]).tolist()
    alg_bytes = sum(8.0 * n * live_in[a] for a in starts)
    kern_s = sum(layer_ms) * 1e-3
    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    achieved = alg_bytes / kern_s / 1e9 if kern_s > 0 else None
    traffic, traffic_src, levels = None, None, None
    try:
        # dram__bytes_read.sum + dram__bytes_write.sum of one captured launch of
        # the dominant variant (ncu --set full, profiles/layer_traffic.json),
        # expressed per average launch through its ratio to that launch's
        # algorithmic bytes; plus the binding-level utilisations (HBM, L2,
        # L1/shared, FMA pipe, issue) of the captured kernels of this config
        prof = json.load(open(os.path.join(ROOT, "profiles", "layer_traffic.json")))
        if prof.get("config") == args.config and prof.get("kernel") == kernel_name(net, args) and args.net == "rn":
            traffic = prof["dram_over_alg"] * alg_bytes / len(plan)
            traffic_src = prof["source"]
        key = args.config + ("" if args.net == "rn" else "-" + args.net)
        if key in prof.get("levels", {}):
            levels = {x["kernel"].split("(")[0].replace("void ", ""):
                      {k: (round(x[k], 3) if isinstance(x[k], float) else x[k])
                       for k in ("duration_ms", "hbm_frac_of_measured", "l2_pct", "l1_pct",
                                 "smem_wavefront_pct", "smem_bank_conflict_share", "fma_pipe_pct",
                                 "issue_pct", "warps_active_pct")}
                      for x in prof["levels"][key]}
    except Exception:
        pass
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "traffic_source": traffic_src,
            "kernel": f"{kernel_name(net, args)} ({len(plan)} launches per inference, "
                      f"{sum(1 for m in plan if m > 1)} fused passes covering "
                      f"{sum(m for m in plan if m > 1)} layers; avg over the last timed "
                      "inference, CUDA events on the launching stream)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback 6.65 TB/s",
            "kernel_share_of_step": kern_s / (ms * 1e-3),
            "alg_bytes_per_launch": alg_bytes / len(plan),
            "alg_bytes_per_live_edge": alg_bytes / max(1, st["live_edges"]),
            "levels": levels,
            "note": ("N <= 1024: the shared-memory-resident kernel runs the last layers (HBM only at "
                     "entry and exit), so the HBM fraction is not its bound; at C1 (1000 rows = 63 CTAs "
                     "of 16 positions for 148 SMs) it is latency/occupancy bound, see levels"
                     if st.get("resident_layers", 0) > 0 else None),
            "levels_source": "ncu --set full, one launch per kernel (profiles/layer_traffic.json, raw CSVs "
                             "under profiles/r02/ncu; "
                             "percentages of each unit's peak)" if levels else None}

    # ---- e2e through the public host-buffer call --------------------------------
    e2e = None
    if not args.no_e2e:
        # pinned host copies of this rank's rows; every step copies them in
        rp_h = torch.from_numpy(rp).pin_memory().numpy()
        idx_h = torch.from_numpy(idx).pin_memory().numpy()
        if ws == 1 and not args.e2e_sync:
            call = None                                              # pipelined, below
            what = ("sdnn_infer_submit / sdnn_infer_wait (host CSR in, host categories out; the input "
                    "copy of step k+1 overlaps the layers of step k, every step's copies in the timed region)")
        elif ws == 1:
            call = lambda: net.infer(rp_h, idx_h, None)[0]           # noqa: E731
            what = "sdnn_infer (host CSR in, host categories out)"
        else:
            part = sdist.Partitioned(net, gB, device=dev)            # weak: gB = batch * ws
            call = lambda: part(rp_h, idx_h)                          # noqa: E731
            what = ("paper_2004_10908_b200.dist.Partitioned: pinned host slice -> H2D -> "
                    "sdnn_infer_device -> NCCL all-gather -> k_bitmask_ids -> D2H of the ids")
        if call is None:
            # warm-up through both input slots (their device buffers and pinned
            # result buffers are allocated on first use), then at least ~0.5 s
            # of steps so that short configs are not timed on 3 calls
            w0 = net.infer_submit(rp_h, idx_h)
            w1 = net.infer_submit(rp_h, idx_h)
            net.infer_wait(w0)
            cats = net.infer_wait(w1)
            K = max(2, args.e2e_steps, min(32, int(0.5 / max(ms * 1e-3, 1e-4))))
            t1 = time.perf_counter()
            tickets = [net.infer_submit(rp_h, idx_h)]
            for k in range(K):
                if k + 1 < K:
                    tickets.append(net.infer_submit(rp_h, idx_h))
                cats = net.infer_wait(tickets[k])
            te = (time.perf_counter() - t1) / K
        else:
            cats = call()
            times = []
            for _ in range(args.e2e_steps):
                if ws > 1:
                    dist.barrier()
                t1 = time.perf_counter()
                cats = call()
                times.append(time.perf_counter() - t1)
            te = float(np.mean(times))
        if ws > 1:
            t = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": (edges_rank * ws if not strong else B * total_nnz) / te, "unit": UNIT,
               "h2d_bytes_per_step": int(rp_h.nbytes + idx_h.nbytes) * ws,
               "d2h_bytes_per_step": int(4 + 4 * cats.size) * ws, "ms_per_step": te * 1e3,
               "call": what}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        r = np.random.default_rng(99)
        rows = np.sort(r.choice(batch, args.cpu_rows, replace=False))
        cpu = cpu_baseline(n, L, spec, rp, idx, rows)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.net}{n}x{L}-ms{B}", "neurons": n, "layers": L,
                       "nnz_per_column": 32, "inputs_per_gpu": batch,
                       "global_batch": batch * ws if not strong else B,
                       "network": NETS[args.net][1] + ", b=%g" % spec.bias,
                       "field_schedule": schedule_desc(g, spec),
                       "nominal_edges_per_step": int(gB * total_nnz) if ws > 1 else int(batch * total_nnz),
                       "fma_per_step": int(st["executed_fma"]) * ws,
                       "fma_over_nominal_edges": (st["executed_fma"] / max(1, batch * total_nnz)),
                       "work_note": ("with uniform weights the members of a column group share one "
                                     "canonical chain (same sources, same weight): one FMA per group "
                                     "source per computed row, not per edge; rows that die are "
                                     "dropped at the compactions between steps"),
                       "inputs": "binary MNIST-shaped strokes (sdnngen.ms_inputs)",
                       "parallelism": f"dp{ws}" if ws > 1 else "single",
                       "l2": "inputs larger than L2 (Y = %.1f GB per GPU)" % (4.0 * n * batch / 1e9)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(st["launches_per_infer"] * args.steps),
            "clocks": clk.summary(),
            "live_edges_per_s": st["live_edges"] * ws / (ms * 1e-3),
            "survivors": {"kept_after_densify": kept0, "after_layer": {str(i): live[i] for i in
                          sorted(set([0, 1, 2, 4, 8, 16, 32, 64, L // 2, L - 1])) if i < L},
                          "categories": int(live[-1]) if live else None,
                          "category_fraction": (live[-1] / batch) if live and batch else None},
            "multi_gpu": multi,
            "load_seconds": t_load,
            "flags": args.flags or None,
            "fuse": {"rows": args.fuse_rows, "layers": args.fuse_layers,
                     "steps": len(plan), "fused_layers": st["fused_layers"]},
            "weight_streaming": ({"slots": args.stream_slots, "h2d_bytes_per_step": st["stream_bytes"],
                                  "slot_bytes": st["stream_slot_bytes"]} if args.stream_slots else None),
        }
        print(json.dumps(line), flush=True)
    net.close()
    if ws > 1:
        dist.destroy_process_group()


def run_oneshot(args):
    """Minimal driver for ncu: no e2e, no oracle, no collectives."""
    import torch

    import paper_2004_10908_b200 as sd
    import sdnngen as g
    n, L, B = CONFIGS[args.config]
    net = sd.Net.from_spec(net_spec(g, args, n, L), fmt="ell", threads=args.load_threads, device=0,
                           flags=lib_flags(sd, args.flags), fuse_rows=args.fuse_rows,
                           fuse_layers=args.fuse_layers, stream_slots=args.stream_slots)
    rp, idx = make_inputs(n, B, 0)
    rp_t, idx_t = torch.from_numpy(rp).cuda(), torch.from_numpy(idx).cuda()
    for _ in range(args.warmup + args.steps):
        net.infer_torch(rp_t, idx_t, None)
    torch.cuda.synchronize()
    print(json.dumps({"oneshot": args.config, "stats": {k: v for k, v in net.stats().items()
                                                         if k != "live_rows"}}))
    net.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sdnn", choices=["sdnn", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the one 60,000-input batch split across ranks "
                         "(BASELINE configs[3], default); weak = every rank its own batch")
    ap.add_argument("--gather", default="auto", choices=["auto", "nccl", "nvls"],
                    help="N > 1: category gather fused into the readout over NVLS (auto: when the "
                         "group has a multicast mapping) or the NCCL all-gather")
    ap.add_argument("--net", default="rn", choices=sorted(NETS),
                    help="network family: rn = RadiX-Net-shaped (headline); rn-plain, rw, rr = robustness rows")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-sync", action="store_true",
                    help="e2e through the synchronous sdnn_infer instead of the pipelined submit/wait")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=16)
    ap.add_argument("--ref-rows", type=int, default=0)
    ap.add_argument("--load-threads", type=int, default=8)
    ap.add_argument("--fuse-rows", type=int, default=-1,
                    help="component cap for fused multi-layer passes (0 = off, -1 = library default)")
    ap.add_argument("--fuse-layers", type=int, default=-1)
    ap.add_argument("--stream-slots", type=int, default=0,
                    help="f3 weight streaming: ring of S device slots (0 = weights resident)")
    ap.add_argument("--flags", default="",
                    help="comma list of library flags, e.g. no_graph,no_bulk (f1 studies)")
    ap.add_argument("--oneshot", action="store_true",
                    help="profiling helper: load, run warmup+steps inferences, print timing only")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "sdnn":
        print("warning: the contract asks for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.oneshot:
        run_oneshot(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
