"""Seeded synthetic workload generators for the sparse-DNN inference path.

This module is shared by the oracle side (``oracle/``, ``tests/``) and the
product side (``bench.py``, the binding's callers).  It holds **none of the
method's arithmetic**: it only draws network *structure* (which input neuron k
feeds which output neuron j), the stored weight values, the bias vectors and
the binary input matrices.  No layer is ever evaluated here.

What the paper fixes (``/root/reference/PAPER.md``, §7.4 "Large Sparse Neural
Network Inference", lines 2552-2572): each dataset is "a sparse matrix of the
input data for the network, 1920 layers of neurons stored in sparse matrices,
truth categories, and the bias values" (L2557-2559).  The challenge data itself
is not available, so every input here is synthetic.

Families
--------
``rn``  RadiX-Net-shaped (the headline workload).  Every layer is a radix-32
        butterfly stage on one 5-bit field of the neuron id: output m reads the
        32 ids equal to m except in bits [p_l, p_l+5).  Hence every column has
        exactly 32 distinct sources, every row exactly 32 out-edges, and the
        layer is a (relabelled) set of N/32 dense 32x32 blocks.  The field
        schedule is p_l = (2 l + floor(l / c)) mod (log2 N - 4), c =
        ceil((log2 N - 4) / 2) (overlapping fields that reach every offset; see
        DESIGN.md reading R-W2 for why the non-overlapping radix-32 schedule is
        not used).  Neurons are relabelled at every internal layer boundary by
        a seeded permutation pi_l applied consistently to the outputs of layer
        l-1 and the inputs of layer l, so the dynamics are those of the plain
        butterfly network while device accesses scatter.
``rr``  random 32-regular: column j of layer l reads
        sigma_l((tau_l(j) + o_{l,t}) mod N), t < 32, with 32 distinct offsets.
        No two columns share a source set (general-gather robustness family).
``ka``  known-answer family: block-diagonal up to relabelling.  Layer l maps
        output group g (32 neurons) to input group beta_l(g) with a dense 32x32
        block, so every group evolves independently and its fate is known in
        closed form (tests/test_oracle_pins.py).

Inputs
------
``ms_inputs``  binary "MNIST-shaped" digits: 2-4 quadratic Bezier strokes of
        radius ~1.25 px drawn on a 28x28 canvas inside the central 20x20 box,
        nearest-neighbour upscaled to an h x w canvas (h*w = N), flattened
        row-major.  Sentinel rows: every row i with i % 1000 == 999 is all
        ones, every row with i % 1000 == 998 is empty.
``ka_inputs``  per 32-neuron input group a seeded count of ones.

Seeds: network seed ``0x5D11 ^ (N << 8) ^ L``; input seed ``0x1A9E ^ N``
(SURVEY.md §8.4).  All randomness comes from numpy PCG64 streams keyed by
(seed, purpose, layer), so any layer can be regenerated independently.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass, field
from typing import Iterator, Optional

import numpy as np

__all__ = [
    "K", "W_VALUE", "bias_value", "net_seed", "input_seed", "NetSpec", "Layer",
    "rn_spec", "rr_spec", "rw_spec", "rw_bias", "rn_plain_spec", "plain_bias", "ka_spec", "random_spec", "gen_layer", "iter_layers",
    "ms_inputs", "ka_inputs", "random_inputs", "structure_hash", "csr_from_dense",
    "dense_from_csr", "ka_group_counts",
]

K = 32                      # nonzeros per column (north_star: "fixed nonzeros per column")
W_VALUE = np.float32(1.0 / 16.0)   # challenge-style uniform weight (DESIGN.md R-W1)

_BIAS = {1024: -0.30, 4096: -0.35, 16384: -0.40, 65536: -0.45}


def bias_value(n: int) -> float:
    """Per-width bias constant (recalled challenge values, DESIGN.md R-W1)."""
    if n in _BIAS:
        return _BIAS[n]
    # geometric interpolation between the four challenge widths
    lg = np.log2(n) / 2.0 - 5.0           # 0 at 1024, 1 at 4096, ...
    return float(np.clip(-0.30 - 0.05 * lg, -0.45, -0.30))


def net_seed(n: int, L: int) -> int:
    return 0x5D11 ^ (n << 8) ^ L


def input_seed(n: int) -> int:
    return 0x1A9E ^ n


def _rng(*key: int) -> np.random.Generator:
    return np.random.default_rng([int(k) & 0xFFFFFFFFFFFF for k in key])


@dataclass
class Layer:
    """One layer W_l in both supported host formats plus its bias.

    csr: rowptr int64[N+1], colidx int32[nnz]; row = input neuron k,
         col = output neuron j (W_l[k][j] connects k to j).
    ell: int32[N, k] per OUTPUT j the source list (unsorted), -1 = padding.
    val: None for a uniform layer (every stored value == uniform), else
         float32 aligned with colidx (csr) -- ell_val aligned with ell.
    """
    rowptr: np.ndarray
    colidx: np.ndarray
    val: Optional[np.ndarray]
    ell: np.ndarray
    ell_val: Optional[np.ndarray]
    uniform: float
    bias: np.ndarray


@dataclass
class NetSpec:
    kind: str
    n: int
    L: int
    seed: int
    bias: float = 0.0
    wdist: str = "uniform"            # "uniform" | "random" (per-slot values)
    extra: dict = field(default_factory=dict)


def rn_spec(n: int, L: int, seed: Optional[int] = None, schedule: str = "overlap", **kw) -> NetSpec:
    assert n >= 32 and n & (n - 1) == 0, "RN needs a power-of-two width >= 32"
    assert schedule in ("overlap", "plain")
    extra = dict(kw.pop("extra", {}))
    if schedule != "overlap":                 # the default keeps extra empty (structure hashes)
        extra["schedule"] = schedule
    return NetSpec("rn", n, L, net_seed(n, L) if seed is None else seed,
                   kw.pop("bias", bias_value(n)), extra=extra, **kw)


# RW (general weights): the RN structure with one seeded value per slot drawn
# from U(-0.05, 0.15) (mean 0.05 < 1/16); the per-width biases below keep
# 29-45 % of the MS inputs alive through the whole network (measured with the
# oracle on sampled rows, reading R-W4)
_RW_BIAS = {1024: -0.125, 4096: -0.15, 16384: -0.175, 65536: -0.225}


def rw_bias(n: int) -> float:
    if n in _RW_BIAS:
        return _RW_BIAS[n]
    lg = np.log2(n) / 2.0 - 5.0
    return float(np.clip(-0.125 - 0.025 * lg, -0.225, -0.125))


def rw_spec(n: int, L: int, seed: Optional[int] = None, **kw) -> NetSpec:
    """RN structure with per-slot random weights (the general-weight path)."""
    return rn_spec(n, L, seed=seed, wdist="random", bias=kw.pop("bias", rw_bias(n)), **kw)


# Plain (non-overlapping) field schedule: with the challenge biases it kills all
# but ~0.4 % of the MS rows within 4 layers (DESIGN.md R-W2); these biases keep
# ~44 % alive (oracle, sampled rows; DESIGN.md R-W5)
_PLAIN_BIAS = {1024: -0.2, 4096: -0.225, 16384: -0.25, 65536: -0.275}


def plain_bias(n: int) -> float:
    if n in _PLAIN_BIAS:
        return _PLAIN_BIAS[n]
    lg = np.log2(n) / 2.0 - 5.0
    return float(np.clip(-0.2 - 0.025 * lg, -0.275, -0.2))


def rn_plain_spec(n: int, L: int, seed: Optional[int] = None, **kw) -> NetSpec:
    """RN with SURVEY.md 8.4's non-overlapping field schedule (robustness row)."""
    return rn_spec(n, L, seed=seed, schedule="plain", bias=kw.pop("bias", plain_bias(n)), **kw)


def rr_spec(n: int, L: int, seed: Optional[int] = None, **kw) -> NetSpec:
    assert n >= 32
    return NetSpec("rr", n, L, net_seed(n, L) ^ 0x7777 if seed is None else seed,
                   kw.pop("bias", bias_value(n)), **kw)


def ka_spec(n: int, L: int, seed: Optional[int] = None, **kw) -> NetSpec:
    assert n >= 32 and n % 32 == 0
    return NetSpec("ka", n, L, net_seed(n, L) ^ 0x4B41 if seed is None else seed,
                   kw.pop("bias", bias_value(n)), **kw)


def random_spec(n: int, L: int, seed: int, kmin: int = 0, kmax: int = 32,
                bias=(-0.25, 0.0), wdist: str = "random", **kw) -> NetSpec:
    """Irregular test networks: column j has a seeded number of sources in
    [kmin, kmax] (so padding, empty columns and K < 32 occur), random values."""
    return NetSpec("irr", n, L, seed, 0.0, wdist,
                   extra=dict(kmin=kmin, kmax=kmax, bias_range=bias, **kw))


# --------------------------------------------------------------------------
# permutations shared by the structured families
# --------------------------------------------------------------------------

def _perm(spec: NetSpec, boundary: int) -> np.ndarray:
    """Relabelling pi_b of the neurons at layer boundary b (0 = input, L = output).
    pi_0 is the identity so that input neuron == image pixel."""
    if boundary == 0:
        return np.arange(spec.n, dtype=np.int64)
    return _rng(spec.seed, 1, boundary).permutation(spec.n)


def _inv(p: np.ndarray) -> np.ndarray:
    q = np.empty_like(p)
    q[p] = np.arange(p.size, dtype=p.dtype)
    return q


def rn_field(n: int, l: int, schedule: str = "overlap") -> int:
    """Offset of layer l's 5-bit butterfly field.

    "overlap" (default, DESIGN.md R-W2): steps of 2 (consecutive fields overlap
    in 3 bits, which keeps image locality for a few layers) and every cycle of
    ceil(span/2) layers shifted by one, so odd offsets -- and with them the top
    id bit -- are mixed too.
    "plain" (SURVEY.md 8.4 as written): non-overlapping fields cycling over
    0, 5, 10, ..., the last one clamped to log2 N - 5 (full mixing within
    ceil(log2 N / 5) layers; the robustness row, with its own bias R-W5)."""
    bits = n.bit_length() - 1
    span = bits - 4                      # valid offsets 0 .. bits-5
    if schedule == "plain":
        offs = list(range(0, span, 5))
        if offs[-1] != bits - 5:
            offs.append(bits - 5)
        return offs[l % len(offs)]
    c = (span + 1) // 2
    return (2 * l + l // c) % span


def _rn_sets(n: int, l: int, m: np.ndarray, schedule: str = "overlap") -> np.ndarray:
    """Butterfly set of internal ids m (vector): [len(m), 32] ids equal to m
    except in the 5-bit field at offset p_l."""
    p = rn_field(n, l, schedule)
    base = m & ~np.int64(31 << p)
    return base[:, None] | (np.arange(32, dtype=np.int64)[None, :] << p)


def _csr_from_out_lists(n: int, out_lists: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """out_lists[k] = the output neurons fed by input k (fixed fan-out)."""
    fan = out_lists.shape[1]
    rowptr = np.arange(0, (n + 1) * fan, fan, dtype=np.int64)
    return rowptr, out_lists.reshape(-1).astype(np.int32)


def _csr_from_ell(n: int, ell: np.ndarray, ell_val: Optional[np.ndarray]):
    """Transpose per-output source lists to CSR (row = input).  Pure index
    bookkeeping, stable in j within each row."""
    j = np.repeat(np.arange(n, dtype=np.int64), ell.shape[1])
    k = ell.reshape(-1).astype(np.int64)
    keep = k >= 0
    j, k = j[keep], k[keep]
    order = np.argsort(k, kind="stable")
    counts = np.bincount(k, minlength=n)
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rowptr[1:])
    colidx = j[order].astype(np.int32)
    val = None
    if ell_val is not None:
        val = ell_val.reshape(-1)[keep][order].astype(np.float32)
    return rowptr, colidx, val


def _rn_lists(n: int, l: int, outer: np.ndarray, inner: np.ndarray, schedule: str = "overlap") -> np.ndarray:
    lib = _helper()
    if lib is None:
        return outer[_rn_sets(n, l, inner, schedule)].astype(np.int32)
    out = np.empty((n, 32), np.int32)
    outer = np.ascontiguousarray(outer, np.int64)
    inner = np.ascontiguousarray(inner, np.int64)
    lib.rn_lists(n, rn_field(n, l, schedule), _p(outer), _p(inner), _p(out))
    return out


def gen_layer(spec: NetSpec, l: int, fmt: str = "both") -> Layer:
    """Layer l of the network.  fmt: "both" (CSR + ELL), "csr" or "ell" (the
    other format's fields are left empty where producing them costs time)."""
    n = spec.n
    want_csr, want_ell = fmt in ("both", "csr"), fmt in ("both", "ell")
    empty_i64, empty_i32 = np.zeros(0, np.int64), np.zeros((0, 32), np.int32)
    if spec.kind == "rn":
        pin, pout = _perm(spec, l), _perm(spec, l + 1)
        sch = spec.extra.get("schedule", "overlap")
        ell = _rn_lists(n, l, pin, _inv(pout), sch) if want_ell else empty_i32
        if want_csr:
            rowptr = np.arange(0, (n + 1) * 32, 32, dtype=np.int64)
            colidx = _rn_lists(n, l, pout, _inv(pin), sch).reshape(-1)
        else:
            rowptr, colidx = empty_i64, np.zeros(0, np.int32)
        val = ell_val = None
    elif spec.kind == "ka":
        pin, pout = _perm(spec, l), _perm(spec, l + 1)
        beta = _rng(spec.seed, 2, l).permutation(n // 32)
        inv_out = _inv(pout)
        c = np.arange(n, dtype=np.int64)
        g_out = inv_out[c] // 32                                        # output group of c
        src_int = beta[g_out][:, None] * 32 + np.arange(32)[None, :]
        ell = pin[src_int].astype(np.int32)
        rowptr, colidx, _ = _csr_from_ell(n, ell, None)
        val = ell_val = None
    elif spec.kind == "rr":
        r = _rng(spec.seed, 3, l)
        sigma, tau = r.permutation(n), r.permutation(n)
        offs = r.choice(n, size=K, replace=False)
        ell = sigma[(tau[:, None] + offs[None, :]) % n].astype(np.int32)
        rowptr, colidx, _ = _csr_from_ell(n, ell, None)
        val = ell_val = None
    elif spec.kind == "irr":
        r = _rng(spec.seed, 4, l)
        kmin, kmax = spec.extra["kmin"], spec.extra["kmax"]
        kk = r.integers(kmin, kmax + 1, size=n)
        width = max(int(kk.max()) if n else 0, 1)
        ell = np.full((n, width), -1, np.int32)
        for j in range(n):
            if kk[j]:
                ell[j, :kk[j]] = r.choice(n, size=min(int(kk[j]), n), replace=False)
        ell_val = None
        if spec.wdist == "random":
            vals = r.uniform(-0.25, 0.5, size=ell.shape).astype(np.float32)
            vals[ell < 0] = 0.0
            ell_val = vals
        rowptr, colidx, val = _csr_from_ell(n, ell, ell_val)
        if ell_val is None:
            val = None
    else:
        raise ValueError(spec.kind)
    if spec.kind != "irr" and spec.wdist == "random":
        r = _rng(spec.seed, 5, l)
        if ell.size == 0:
            raise ValueError("random weights need the ELL structure (fmt='both' or 'ell')")
        ell_val = r.uniform(-0.05, 0.15, size=ell.shape).astype(np.float32)
        rowptr, colidx, val = _csr_from_ell(n, ell, ell_val)
    if spec.kind == "irr":
        lo, hi = spec.extra["bias_range"]
        bias = _rng(spec.seed, 6, l).uniform(lo, hi, size=n).astype(np.float32)
    else:
        bias = np.full(n, spec.bias, np.float32)
    return Layer(rowptr, colidx, val, ell, ell_val, float(W_VALUE), bias)


def iter_layers(spec: NetSpec) -> Iterator[Layer]:
    for l in range(spec.L):
        yield gen_layer(spec, l)


# --------------------------------------------------------------------------
# inputs
# --------------------------------------------------------------------------

_HELPER = None


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _helper():
    """Load (building on first use) the C upscale helper; None -> numpy path."""
    global _HELPER
    if _HELPER is not None:
        return _HELPER or None
    here = os.path.dirname(os.path.abspath(__file__))
    src, so = os.path.join(here, "_msupscale.c"), os.path.join(here, "_msupscale.so")
    try:
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            tmp = so + ".%d.tmp" % os.getpid()
            subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", src, "-o", tmp])
            os.replace(tmp, so)
        lib = ctypes.CDLL(so)
        V, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.ms_count.argtypes = [I64, V, I32, I32, V, V, V, V]
        lib.ms_fill.argtypes = [I64, V, I32, I32, V, V, V, V, V]
        lib.rn_lists.argtypes = [I64, I32, V, V, V]
        _HELPER = lib
    except Exception:                       # pragma: no cover - gcc missing
        _HELPER = False
    return _HELPER or None


def _canvas(n: int) -> tuple[int, int]:
    bits = n.bit_length() - 1
    assert 1 << bits == n, "MS inputs need a power-of-two width"
    h = 1 << (bits // 2)
    return h, n // h


def _digits28(B: int, r: np.random.Generator) -> np.ndarray:
    """[B, 28, 28] bool stroke images (2-4 quadratic Bezier strokes)."""
    ns = r.integers(2, 5, size=B)                       # strokes per image
    ctrl = r.uniform(4.0, 24.0, size=(B, 4, 3, 2))      # control points (y, x)
    rad = r.uniform(1.0, 1.5, size=(B, 1, 1))           # pen radius in pixels
    t = np.linspace(0.0, 1.0, 24)
    b0, b1, b2 = (1 - t) ** 2, 2 * (1 - t) * t, t * t   # Bezier basis
    pts = (b0[None, None, :, None] * ctrl[:, :, None, 0, :]
           + b1[None, None, :, None] * ctrl[:, :, None, 1, :]
           + b2[None, None, :, None] * ctrl[:, :, None, 2, :])  # [B,4,24,2]
    alive = (np.arange(4)[None, :] < ns[:, None])               # [B,4]
    alive = np.broadcast_to(alive[:, :, None], (B, 4, 24)).reshape(B, 96)
    pts = pts.reshape(B, 96, 2)
    out = np.zeros((B, 28 * 28), bool)
    cy, cx = np.floor(pts[..., 0]).astype(np.int64), np.floor(pts[..., 1]).astype(np.int64)
    r2 = rad[:, 0] ** 2                                          # [B,1]
    bidx = np.broadcast_to(np.arange(B)[:, None], (B, 96))
    for dy in range(-2, 3):                                      # stamp a disc of pen radius
        for dx in range(-2, 3):
            py, px = cy + dy, cx + dx
            d2 = (py + 0.5 - pts[..., 0]) ** 2 + (px + 0.5 - pts[..., 1]) ** 2
            hit = alive & (d2 <= r2) & (py >= 0) & (py < 28) & (px >= 0) & (px < 28)
            out[bidx[hit], (py * 28 + px)[hit]] = True
    return out.reshape(B, 28, 28)


def csr_from_dense(dense: np.ndarray):
    """Binary/float dense [B, N] -> (rowptr int64, idx int32, val float32)."""
    rows, cols = np.nonzero(dense)
    rowptr = np.zeros(dense.shape[0] + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=dense.shape[0]), out=rowptr[1:])
    return rowptr, cols.astype(np.int32), dense[rows, cols].astype(np.float32)


def dense_from_csr(rowptr, idx, val, n: int) -> np.ndarray:
    B = rowptr.size - 1
    out = np.zeros((B, n), np.float32)
    rows = np.repeat(np.arange(B), np.diff(rowptr))
    out[rows, idx] = 1.0 if val is None else val
    return out


def ms_inputs(n: int, B: int, seed: Optional[int] = None, sentinels: bool = True,
              chunk: int = 2048):
    """Binary MNIST-shaped inputs as CSR (rowptr int64[B+1], idx int32[nnz]);
    values are implicitly 1.0 (pass val=None to the library/oracle)."""
    seed = input_seed(n) if seed is None else seed
    h, w = _canvas(n)
    ys = ((np.arange(h) * 28) // h).astype(np.int32)     # target row -> source row
    xs = ((np.arange(w) * 28) // w).astype(np.int32)     # target col -> source col
    lib = _helper()
    scratch = np.empty(w, np.int32)
    rowptr = np.zeros(B + 1, np.int64)
    imgs, counts = [], []
    for c0 in range(0, B, chunk):
        c1 = min(B, c0 + chunk)
        img = _digits28(c1 - c0, _rng(seed, 7, c0 // chunk))
        if sentinels:
            i = np.arange(c0, c1)
            img[(i % 1000) == 999] = True
            img[(i % 1000) == 998] = False
        img = np.ascontiguousarray(img.reshape(c1 - c0, 784).astype(np.uint8))
        cnt = np.zeros(c1 - c0, np.int64)
        if lib is not None:
            lib.ms_count(c1 - c0, _p(img), h, w, _p(ys), _p(xs), _p(cnt), _p(scratch))
        else:
            cnt[:] = img[:, (ys[:, None] * 28 + xs[None, :]).reshape(-1)].sum(1)
        imgs.append(img)
        counts.append(cnt)
    np.cumsum(np.concatenate(counts) if counts else np.zeros(0, np.int64), out=rowptr[1:])
    idx = np.empty(int(rowptr[-1]), np.int32)
    for ci, c0 in enumerate(range(0, B, chunk)):
        img = imgs[ci]
        sub_rowptr = np.ascontiguousarray(rowptr[c0:c0 + img.shape[0] + 1])
        if lib is not None:
            lib.ms_fill(img.shape[0], _p(img), h, w, _p(ys), _p(xs), _p(sub_rowptr), _p(idx), _p(scratch))
        else:
            dense = img[:, (ys[:, None] * 28 + xs[None, :]).reshape(-1)]
            f = np.flatnonzero(dense)
            idx[sub_rowptr[0]:sub_rowptr[-1]] = (f % n).astype(np.int32)
    return rowptr, idx


def ka_group_counts(n: int, B: int, seed: int, p_hot: float = 0.5) -> np.ndarray:
    """[B, n//32] number of ones placed in each input group (boundary-0 group g =
    neurons 32g..32g+31).  Cold groups get 0..8 ones; with probability p_hot a
    row gets one hot group with a count uniform in 0..32."""
    r = _rng(seed, 8)
    G = n // 32
    cnt = r.integers(0, 9, size=(B, G))
    hot = r.random(B) < p_hot
    g = r.integers(0, G, size=B)
    cnt[np.arange(B)[hot], g[hot]] = r.integers(0, 33, size=int(hot.sum()))
    return cnt


def ka_inputs(n: int, B: int, seed: int, p_hot: float = 0.5):
    """Binary KA inputs: within each group a random subset of the chosen size."""
    cnt = ka_group_counts(n, B, seed, p_hot)
    r = _rng(seed, 9)
    keys = r.random((B, n // 32, 32)).argsort(-1)           # random rank of each slot
    dense = (keys < cnt[:, :, None]).reshape(B, n)
    rows, cols = np.nonzero(dense)
    rowptr = np.zeros(B + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=B), out=rowptr[1:])
    return rowptr, cols.astype(np.int32), cnt


def random_inputs(n: int, B: int, seed: int, density: float = 0.2,
                  lo: float = -1.0, hi: float = 2.0):
    """Real-valued inputs (negative entries included) for general-path tests."""
    r = _rng(seed, 10)
    dense = (r.random((B, n)) < density) * r.uniform(lo, hi, size=(B, n))
    dense = dense.astype(np.float32)
    return csr_from_dense(dense)


def structure_hash(spec: NetSpec, layers: Optional[list] = None) -> str:
    """SHA-256 over every layer's CSR structure/values and bias (generator
    drift detector, SPEC.md:496 style)."""
    h = hashlib.sha256()
    for lay in (layers if layers is not None else iter_layers(spec)):
        h.update(lay.rowptr.tobytes())
        h.update(lay.colidx.tobytes())
        if lay.val is not None:
            h.update(lay.val.tobytes())
        h.update(lay.bias.tobytes())
    return h.hexdigest()
