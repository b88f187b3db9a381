"""B200-native sparse-DNN inference (arXiv 2004.10908, Sec. 7.4 hot path).

Thin Python binding of the C ABI in ``include/sdnn.h`` (argument marshalling
only -- every step of the path runs in the CUDA kernels of ``libsdnn.so``):

    sdnn_create / sdnn_create_empty / sdnn_set_layer   load W_l, b_l (resident in HBM)
    sdnn_infer          host CSR Y0 -> ascending category ids (end-to-end call)
    sdnn_infer_device   device CSR Y0 -> device category bitmask (torch / NCCL path)
    sdnn_stats_get      survivor profile, launch count, packed bytes
    sdnn_destroy

There is no CPU fallback: importing this package without the built
``libsdnn.so`` raises, and every call needs a CUDA device.
"""
from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDNN_LIB") or os.path.join(_HERE, "libsdnn.so")

SDNN_OK, SDNN_E_ARG, SDNN_E_FORMAT, SDNN_E_UNSUPPORTED = 0, -1, -2, -3
SDNN_E_NOMEM, SDNN_E_CUDA, SDNN_E_STATE = -4, -5, -6
SDNN_W_CSR, SDNN_W_ELLCOL = 0, 1
SDNN_F_NO_COMPACT, SDNN_F_NO_GROUPS, SDNN_F_NO_GRAPH = 1, 2, 4
SDNN_F_NO_RESIDENT, SDNN_F_TRUST_INPUT, SDNN_F_PROFILE, SDNN_F_NO_BULK = 8, 16, 32, 64
SDNN_F_SATURATE, SDNN_F_SHARE_VALUES = 256, 512

EXPORTS = ["sdnn_create", "sdnn_create_empty", "sdnn_set_layer", "sdnn_infer",
           "sdnn_infer_device", "sdnn_stats_get", "sdnn_validate_layer", "sdnn_destroy",
           "sdnn_last_error", "sdnn_abi_version", "sdnn_layer_times", "sdnn_plan_steps",
           "sdnn_step_plan", "sdnn_gather_rows", "sdnn_bitmask_to_ids",
           "sdnn_flow_infer", "sdnn_infer_device_nvls", "sdnn_nvls_barrier",
           "sdnn_flow_plan", "sdnn_infer_submit", "sdnn_infer_wait"]


class SdnnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sdnn status {status}: {msg}")
        self.status = status


class sdnn_layer(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("ell_k", ctypes.c_int32),
                ("rowptr", ctypes.c_void_p), ("idx", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("uniform_value", ctypes.c_float)]


class sdnn_opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("ymax", ctypes.c_float), ("stream", ctypes.c_void_p),
                ("fuse_rows", ctypes.c_int32), ("fuse_layers", ctypes.c_int32),
                ("resident_from", ctypes.c_int32), ("stream_slots", ctypes.c_int32)]


class sdnn_layer_info(ctypes.Structure):
    _fields_ = [("ngroups", ctypes.c_int32), ("kmax", ctypes.c_int32), ("gmax", ctypes.c_int32),
                ("uniform", ctypes.c_int32), ("regular", ctypes.c_int32),
                ("bias_nonpositive", ctypes.c_int32), ("nnz", ctypes.c_int64)]


SDNN_FLOW_GRAPH, SDNN_FLOW_CAPTURER, SDNN_FLOW_STREAMS = 0, 1, 2


class sdnn_flow_part(ctypes.Structure):
    _fields_ = [("d_rowptr", ctypes.c_void_p), ("d_idx", ctypes.c_void_p), ("d_val", ctypes.c_void_p),
                ("batch", ctypes.c_int64), ("word_offset", ctypes.c_int64)]


class sdnn_nvls(ctypes.Structure):
    _fields_ = [("local_words", ctypes.c_void_p), ("mc_words", ctypes.c_void_p),
                ("local_flag", ctypes.c_void_p), ("mc_flag", ctypes.c_void_p),
                ("word_offset", ctypes.c_int64), ("target", ctypes.c_uint32)]


class sdnn_stats(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("neurons", ctypes.c_int32),
                ("layers", ctypes.c_int32), ("path", ctypes.c_int32),
                ("grouped_layers", ctypes.c_int32), ("max_group", ctypes.c_int32),
                ("max_k", ctypes.c_int32), ("compaction", ctypes.c_int32),
                ("packed_weight_bytes", ctypes.c_int64), ("total_nnz", ctypes.c_int64),
                ("last_batch", ctypes.c_int64), ("last_n_categories", ctypes.c_int64),
                ("launches_per_infer", ctypes.c_int64), ("live_edges", ctypes.c_int64),
                ("kept_rows", ctypes.c_int64), ("steps", ctypes.c_int32),
                ("fused_layers", ctypes.c_int32), ("resident_layers", ctypes.c_int32),
                ("retired_rows", ctypes.c_int64), ("stream_bytes", ctypes.c_int64),
                ("stream_slot_bytes", ctypes.c_int64), ("executed_fma", ctypes.c_int64),
                ("computed_rows", ctypes.c_int64)]


_LIB = None


def lib() -> ctypes.CDLL:
    """Load libsdnn.so (fails loudly when it has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2004_10908_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        V, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        P = ctypes.POINTER
        L.sdnn_create.argtypes = [I32, I32, P(sdnn_layer), V, P(sdnn_opts), P(V)]
        L.sdnn_create_empty.argtypes = [I32, I32, P(sdnn_opts), P(V)]
        L.sdnn_set_layer.argtypes = [V, I32, P(sdnn_layer), V]
        L.sdnn_infer.argtypes = [V, V, V, V, I64, V, P(I64), V]
        L.sdnn_infer_device.argtypes = [V, V, V, V, I64, V, V, V]
        L.sdnn_stats_get.argtypes = [V, P(sdnn_stats), V]
        L.sdnn_validate_layer.argtypes = [I32, P(sdnn_layer), V, U32, P(sdnn_layer_info)]
        L.sdnn_layer_times.argtypes = [V, V]
        L.sdnn_plan_steps.argtypes = [I32, I32, P(sdnn_layer), V, P(sdnn_opts), V, P(I32)]
        L.sdnn_step_plan.argtypes = [V, V, P(I32)]
        L.sdnn_gather_rows.argtypes = [V, V, I64, V, V]
        L.sdnn_bitmask_to_ids.argtypes = [V, I64, V, V, V]
        L.sdnn_infer_device_nvls.argtypes = [V, V, V, V, I64, P(sdnn_nvls), V]
        L.sdnn_nvls_barrier.argtypes = [V, V, U32, V]
        L.sdnn_flow_plan.argtypes = [I32, I32, V, I32, V, V, V, P(I32), V]
        L.sdnn_infer_submit.argtypes = [V, V, V, V, I64, P(I64)]
        L.sdnn_infer_wait.argtypes = [V, I64, V, P(I64)]
        L.sdnn_flow_infer.argtypes = [V, I32, P(sdnn_flow_part), V, I64, V, V, I32, I32, I32,
                                      P(ctypes.c_float), P(I32)]
        L.sdnn_destroy.argtypes = [V]
        L.sdnn_destroy.restype = None
        L.sdnn_last_error.argtypes = []
        L.sdnn_last_error.restype = ctypes.c_char_p
        L.sdnn_abi_version.restype = I32
        for name in ["sdnn_create", "sdnn_create_empty", "sdnn_set_layer", "sdnn_infer",
                     "sdnn_infer_device", "sdnn_stats_get", "sdnn_validate_layer",
                     "sdnn_layer_times", "sdnn_plan_steps", "sdnn_step_plan", "sdnn_gather_rows",
                     "sdnn_bitmask_to_ids", "sdnn_flow_infer", "sdnn_infer_device_nvls",
                     "sdnn_nvls_barrier", "sdnn_flow_plan", "sdnn_infer_submit",
                     "sdnn_infer_wait"]:
            getattr(L, name).restype = I32
        _LIB = L
    return _LIB


def _check(status: int):
    if status != SDNN_OK:
        raise SdnnError(status, lib().sdnn_last_error().decode(errors="replace"))


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _opts(device=-1, flags=0, ymax=32.0, stream=None, fuse_rows=-1, fuse_layers=-1,
          resident_from=-1, stream_slots=0):
    return sdnn_opts(int(device), int(flags), float(ymax), stream, int(fuse_rows),
                     int(fuse_layers), int(resident_from), int(stream_slots))


def make_layer(layer, fmt: str = "csr"):
    """sdnn_layer (plus the arrays it points to) from an object with rowptr,
    colidx, val, ell, ell_val, uniform (sdnngen.Layer) or a dict."""
    get = (lambda k: layer[k]) if isinstance(layer, dict) else (lambda k: getattr(layer, k))
    if fmt == "csr":
        rowptr = np.ascontiguousarray(get("rowptr"), np.int64)
        idx = np.ascontiguousarray(get("colidx"), np.int32)
        val = get("val")
        val = None if val is None else np.ascontiguousarray(val, np.float32)
        keep = (rowptr, idx, val)
        s = sdnn_layer(SDNN_W_CSR, 0, _p(rowptr), _p(idx), _p(val), float(get("uniform")))
    elif fmt == "ell":
        ell = np.ascontiguousarray(get("ell"), np.int32)
        val = get("ell_val")
        val = None if val is None else np.ascontiguousarray(val, np.float32)
        keep = (ell, val)
        s = sdnn_layer(SDNN_W_ELLCOL, int(ell.shape[1]), None, _p(ell), _p(val),
                       float(get("uniform")))
    else:
        raise ValueError(fmt)
    return s, keep


# ----------------------------------------------------------------- raw calls

def sdnn_create(neurons: int, layers: Sequence, bias: np.ndarray, fmt: str = "csr",
                device: int = -1, flags: int = 0, ymax: float = 32.0, fuse_rows: int = -1,
                fuse_layers: int = -1, resident_from: int = -1, stream_slots: int = 0):
    L = len(layers)
    descs = (sdnn_layer * max(L, 1))()
    keep = []
    for l, lay in enumerate(layers):
        descs[l], k = make_layer(lay, fmt)
        keep.append(k)
    bias = np.ascontiguousarray(bias, np.float32).reshape(-1)
    h = ctypes.c_void_p()
    o = _opts(device, flags, ymax, None, fuse_rows, fuse_layers, resident_from, stream_slots)
    _check(lib().sdnn_create(neurons, L, descs, _p(bias), ctypes.byref(o), ctypes.byref(h)))
    return h


def sdnn_create_empty(neurons: int, layers: int, device: int = -1, flags: int = 0,
                      ymax: float = 32.0, fuse_rows: int = -1, fuse_layers: int = -1,
                      resident_from: int = -1, stream_slots: int = 0):
    h = ctypes.c_void_p()
    o = _opts(device, flags, ymax, None, fuse_rows, fuse_layers, resident_from, stream_slots)
    _check(lib().sdnn_create_empty(neurons, layers, ctypes.byref(o), ctypes.byref(h)))
    return h


def sdnn_set_layer(handle, l: int, layer, bias_l: np.ndarray, fmt: str = "csr"):
    desc, keep = make_layer(layer, fmt)
    bias_l = np.ascontiguousarray(bias_l, np.float32)
    _check(lib().sdnn_set_layer(handle, int(l), ctypes.byref(desc), _p(bias_l)))
    del keep


def sdnn_infer(handle, rowptr: np.ndarray, idx: np.ndarray, val: Optional[np.ndarray],
               neurons: int = 0, want_y: bool = False):
    """Host-buffer inference.  Returns (categories int32[ncat], Y_L or None)."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    idx = np.ascontiguousarray(idx, np.int32)
    val = None if val is None else np.ascontiguousarray(val, np.float32)
    batch = rowptr.size - 1
    cats = np.empty(max(batch, 1), np.int32)
    n = ctypes.c_int64()
    y = np.empty((batch, neurons), np.float32) if want_y else None
    _check(lib().sdnn_infer(handle, _p(rowptr), _p(idx), _p(val), batch, _p(cats),
                            ctypes.byref(n), _p(y)))
    return cats[:n.value].copy(), y


def sdnn_infer_device(handle, d_rowptr: int, d_idx: int, d_val: Optional[int], batch: int,
                      d_alive: Optional[int], d_y_out: Optional[int] = None, stream: int = 0):
    _check(lib().sdnn_infer_device(handle, d_rowptr, d_idx, d_val, int(batch), d_alive,
                                   d_y_out, stream or None))


def sdnn_stats_get(handle, layers: int = 0):
    s = sdnn_stats()
    s.struct_size = ctypes.sizeof(sdnn_stats)
    live = np.zeros(max(layers, 1), np.int64)
    _check(lib().sdnn_stats_get(handle, ctypes.byref(s), _p(live)))
    out = {f: getattr(s, f) for f, _ in sdnn_stats._fields_}
    out["live_rows"] = live[:layers].tolist()
    return out


def sdnn_validate_layer(neurons: int, layer, bias_l, fmt: str = "csr", flags: int = 0):
    """Host-only validation + grouping of one layer (no device needed)."""
    desc, keep = make_layer(layer, fmt)
    bias_l = np.ascontiguousarray(bias_l, np.float32)
    info = sdnn_layer_info()
    _check(lib().sdnn_validate_layer(int(neurons), ctypes.byref(desc), _p(bias_l), int(flags),
                                     ctypes.byref(info)))
    del keep
    return {f: getattr(info, f) for f, _ in sdnn_layer_info._fields_}


def sdnn_plan_steps(neurons: int, layers: Sequence, fmt: str = "csr", flags: int = 0,
                    fuse_rows: int = -1, fuse_layers: int = -1):
    """Host-only execution plan: list of step lengths (layers per kernel step)."""
    L = len(layers)
    descs = (sdnn_layer * max(L, 1))()
    keep = []
    for l, lay in enumerate(layers):
        descs[l], k = make_layer(lay, fmt)
        keep.append(k)
    bias = np.concatenate([np.asarray(l.bias if not isinstance(l, dict) else l["bias"], np.float32)
                           for l in layers]) if L else np.zeros(1, np.float32)
    out = np.zeros(max(L, 1), np.int32)
    ns = ctypes.c_int32()
    o = _opts(-1, flags, 32.0, None, fuse_rows, fuse_layers)
    _check(lib().sdnn_plan_steps(int(neurons), L, descs, _p(bias), ctypes.byref(o), _p(out),
                                 ctypes.byref(ns)))
    return out[:ns.value].tolist()


def sdnn_destroy(handle):
    if handle:
        lib().sdnn_destroy(handle)


# ------------------------------------------------------------- convenience

class Net:
    """Owning wrapper around an sdnn_net handle."""

    def __init__(self, neurons: int, layers: int, flags: int = 0, ymax: float = 32.0,
                 device: int = -1, fuse_rows: int = -1, fuse_layers: int = -1,
                 resident_from: int = -1, stream_slots: int = 0):
        self.n, self.L = int(neurons), int(layers)
        self.h = sdnn_create_empty(self.n, self.L, device=device, flags=flags, ymax=ymax,
                                   fuse_rows=fuse_rows, fuse_layers=fuse_layers,
                                   resident_from=resident_from, stream_slots=stream_slots)

    @classmethod
    def from_layers(cls, neurons: int, layers: Sequence, fmt: str = "csr", **kw):
        net = cls.__new__(cls)
        net.n, net.L = int(neurons), len(layers)
        bias = np.concatenate([np.asarray(l.bias if not isinstance(l, dict) else l["bias"],
                                          np.float32) for l in layers]) if layers else np.zeros(0, np.float32)
        net.h = sdnn_create(neurons, layers, bias, fmt=fmt, **kw)
        return net

    @classmethod
    def from_spec(cls, spec, fmt: str = "ell", threads: int = 8, **kw):
        """Generate (sdnngen) and load every layer, `threads` layers at a time
        (ctypes releases the GIL while a layer is packed and uploaded)."""
        import sdnngen
        net = cls(spec.n, spec.L, **kw)

        def one(l):
            lay = sdnngen.gen_layer(spec, l, fmt=fmt)
            sdnn_set_layer(net.h, l, lay, lay.bias, fmt=fmt)

        if threads <= 1:
            for l in range(spec.L):
                one(l)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(one, range(spec.L)))
        return net

    def set_layer(self, l, layer, bias, fmt="csr"):
        sdnn_set_layer(self.h, l, layer, bias, fmt)

    def infer(self, rowptr, idx, val=None, want_y=False):
        return sdnn_infer(self.h, rowptr, idx, val, self.n, want_y)

    def infer_submit(self, rowptr, idx, val=None):
        """sdnn_infer_submit: enqueue a host-buffer inference, return its ticket.
        The arrays must stay alive and unchanged until infer_wait returns (they
        are kept referenced by the handle until then)."""
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        idx = np.ascontiguousarray(idx, np.int32)
        val = None if val is None else np.ascontiguousarray(val, np.float32)
        t = ctypes.c_int64()
        _check(lib().sdnn_infer_submit(self.h, _p(rowptr), _p(idx), _p(val), rowptr.size - 1, ctypes.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (rowptr, idx, val)
        return t.value

    def infer_wait(self, ticket):
        """sdnn_infer_wait: the ascending category ids of a submitted inference."""
        rowptr = self._inflight[ticket][0]
        cats = np.empty(max(rowptr.size - 1, 1), np.int32)
        n = ctypes.c_int64()
        try:
            _check(lib().sdnn_infer_wait(self.h, int(ticket), _p(cats), ctypes.byref(n)))
        finally:
            del self._inflight[ticket]
        return cats[:n.value].copy()

    def infer_device(self, d_rowptr, d_idx, d_val, batch, d_alive, d_y_out=None, stream=0):
        sdnn_infer_device(self.h, d_rowptr, d_idx, d_val, batch, d_alive, d_y_out, stream)

    def infer_torch(self, rowptr_t, idx_t, val_t=None, alive_t=None, y_t=None, stream=None):
        """Device inference on torch CUDA tensors (plumbing only).  Returns the
        int32 bitmask tensor of ceil(B/32) words (bit i%32 of word i//32 = row i)."""
        import torch
        batch = rowptr_t.numel() - 1
        if alive_t is None:
            alive_t = torch.empty((batch + 31) // 32, dtype=torch.int32, device=rowptr_t.device)
        s = stream if stream is not None else torch.cuda.current_stream(rowptr_t.device)
        sdnn_infer_device(self.h, rowptr_t.data_ptr(), idx_t.data_ptr(),
                          None if val_t is None else val_t.data_ptr(), batch,
                          alive_t.data_ptr() if alive_t.numel() else None,
                          None if y_t is None else y_t.data_ptr(), s.cuda_stream)
        return alive_t

    def gather_rows_torch(self, rows_t, y_t=None, stream=None):
        """Y_L of the given original rows (int32 CUDA tensor) of the last
        inference, via sdnn_gather_rows; returns a [len(rows), n] fp32 tensor."""
        import torch
        if y_t is None:
            y_t = torch.empty((rows_t.numel(), self.n), dtype=torch.float32, device=rows_t.device)
        s = stream if stream is not None else torch.cuda.current_stream(rows_t.device)
        _check(lib().sdnn_gather_rows(self.h, rows_t.data_ptr() if rows_t.numel() else None,
                                      int(rows_t.numel()), y_t.data_ptr() if y_t.numel() else None,
                                      s.cuda_stream))
        return y_t

    def gather_rows(self, rows):
        """Host convenience: Y_L rows (numpy) of the given original row ids."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        rows_t = torch.from_numpy(np.ascontiguousarray(rows, np.int32)).to(dev)
        y = self.gather_rows_torch(rows_t)
        torch.cuda.synchronize(dev)
        return y.cpu().numpy()

    def infer_torch_nvls(self, rowptr_t, idx_t, nv: "sdnn_nvls", stream=None):
        """sdnn_infer_device_nvls: inference + readout fused with the NVLS
        multicast gather into every GPU's copy of the global bitmask."""
        import torch
        batch = rowptr_t.numel() - 1
        s = stream if stream is not None else torch.cuda.current_stream(rowptr_t.device)
        _check(lib().sdnn_infer_device_nvls(self.h, rowptr_t.data_ptr(), idx_t.data_ptr() if idx_t.numel() else None,
                                            None, batch, ctypes.byref(nv), s.cuda_stream))

    def stats(self):
        return sdnn_stats_get(self.h, self.L)

    def step_plan(self):
        """Layers per kernel step of the execution plan (after the first inference)."""
        out = np.zeros(max(self.L, 1), np.int32)
        ns = ctypes.c_int32()
        _check(lib().sdnn_step_plan(self.h, _p(out), ctypes.byref(ns)))
        return out[:ns.value].tolist()

    def layer_times(self):
        """Per-layer kernel durations (ms) of the last inference (SDNN_F_PROFILE)."""
        ms = np.zeros(max(self.L, 1), np.float32)
        _check(lib().sdnn_layer_times(self.h, _p(ms)))
        return ms[:self.L].tolist()

    def close(self):
        if getattr(self, "h", None):
            sdnn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def bitmask_to_ids_torch(words_t, batch: int, stream=None):
    """Device decode of a global category bitmask (sdnn_bitmask_to_ids): returns
    (ids int32 CUDA tensor [batch] capacity, count int32 CUDA tensor [1]); the
    first count entries are the ascending category ids."""
    import torch
    dev = words_t.device
    ids = torch.empty(max(int(batch), 1), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    _check(lib().sdnn_bitmask_to_ids(words_t.data_ptr() if batch > 0 else None, int(batch),
                                     ids.data_ptr(), cnt.data_ptr(), s.cuda_stream))
    return ids, cnt


def flow_plan(ntasks: int, edges, max_streams: int):
    """Algorithm 1's stream assignment (sdnn_flow_plan, host only): returns
    (level, id, stream, cross-stream event edges) for the DAG."""
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    lv, ids, st = (np.zeros(max(ntasks, 1), np.int32) for _ in range(3))
    ev = np.zeros(max(2 * len(e), 2), np.int32)
    ne = ctypes.c_int32()
    _check(lib().sdnn_flow_plan(int(ntasks), len(e), _p(e) if len(e) else None, int(max_streams), _p(lv),
                                _p(ids), _p(st), ctypes.byref(ne), _p(ev)))
    return (lv[:ntasks].tolist(), ids[:ntasks].tolist(), st[:ntasks].tolist(),
            [tuple(x) for x in ev[:2 * ne.value].reshape(-1, 2).tolist()])


def flow_infer(nets, parts, total_batch: int, mode: int, max_streams: int = 4, reps: int = 3):
    """f1 task-graph launch (sdnn_flow_infer).  nets: list of Net (one per
    partition); parts: list of (rowptr_t, idx_t, first_row) torch CUDA tensors
    per partition (word-aligned first rows).  Returns (ids numpy, ms per rep,
    tasks in the graph)."""
    import torch
    dev = parts[0][0].device
    P = len(nets)
    hs = (ctypes.c_void_p * P)(*[n.h.value if hasattr(n.h, "value") else n.h for n in nets])
    arr = (sdnn_flow_part * P)()
    for i, (rp, ix, first) in enumerate(parts):
        assert first % 32 == 0
        arr[i] = sdnn_flow_part(rp.data_ptr(), ix.data_ptr() if ix.numel() else None, None,
                                rp.numel() - 1, first // 32)
    words = torch.zeros((total_batch + 31) // 32, dtype=torch.int32, device=dev)
    ids = torch.empty(max(1, total_batch), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    ms, nt = ctypes.c_float(), ctypes.c_int32()
    _check(lib().sdnn_flow_infer(hs, P, arr, words.data_ptr(), int(total_batch), ids.data_ptr(),
                                 cnt.data_ptr(), int(mode), int(max_streams), int(reps),
                                 ctypes.byref(ms), ctypes.byref(nt)))
    torch.cuda.synchronize(dev)
    return ids[:int(cnt.item())].cpu().numpy(), ms.value, nt.value


def bitmask_to_ids(words: np.ndarray, batch: int) -> np.ndarray:
    """Decode a category bitmask (uint32/int32 words) into ascending row ids."""
    w = np.asarray(words).view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:batch]
    return np.flatnonzero(bits).astype(np.int32)
