"""CPU oracle for the sparse-DNN inference hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2004_10908_b200``) never imports it and shares no code
with it.

The arithmetic lives in ``sdnn_oracle.c`` (plain C, fp32 canonical chain, see
its header for the passages and readings it follows).  This module only
marshals arrays and drives the layer loop in the order the method defines:
Y_0 -> layer 0 -> ... -> layer L-1 -> categories (
BASELINE.json north_star).

Pins: tests/test_oracle_pins.py (hand nets from tests/golden/, dyadic brute
force against float64 dense matmul, closed-form layer 0, the KA known-answer
family, invariants I1-I6).  RN/RR/MS workloads beyond those are "parity
unpinned except through the oracle".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from typing import Iterable, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sdnn_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_LIB = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC", "-pthread"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (called by __graft_entry__.build and tests)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(build())
        V, I32, I64, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        lib.oracle_densify.argtypes = [I32, I64, V, V, V, V]
        lib.oracle_densify.restype = ctypes.c_int
        lib.oracle_layer.argtypes = [I32, I64, V, V, V, V, V, F, V, F, I32, I32]
        lib.oracle_layer.restype = ctypes.c_int
        lib.oracle_categories.argtypes = [I32, I64, V, V]
        lib.oracle_categories.restype = I64
        lib.oracle_live_rows.argtypes = [I32, I64, V]
        lib.oracle_live_rows.restype = I64
        _LIB = lib
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


class Oracle:
    """Layer-by-layer state: dense row-major Y[B][n] in fp32."""

    def __init__(self, n: int, rowptr: np.ndarray, idx: np.ndarray,
                 val: Optional[np.ndarray] = None):
        self.n = int(n)
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        idx = np.ascontiguousarray(idx, np.int32)
        val = None if val is None else np.ascontiguousarray(val, np.float32)
        self.B = rowptr.size - 1
        self.Y = np.empty((self.B, self.n), np.float32)
        self._Z = np.empty_like(self.Y)
        rc = _lib().oracle_densify(self.n, self.B, _p(rowptr), _p(idx), _p(val), _p(self.Y))
        if rc != 0:
            raise ValueError("oracle_densify: invalid Y0 CSR")
        self.layer_seconds = 0.0

    def layer(self, rowptr, colidx, val, uniform: float, bias, ymax: float = 32.0,
              skip_zero: bool = True, nthreads: Optional[int] = None):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        colidx = np.ascontiguousarray(colidx, np.int32)
        val = None if val is None else np.ascontiguousarray(val, np.float32)
        bias = np.ascontiguousarray(bias, np.float32)
        assert rowptr.size == self.n + 1 and bias.size == self.n
        t0 = time.perf_counter()
        rc = _lib().oracle_layer(self.n, self.B, _p(self.Y), _p(self._Z), _p(rowptr),
                                 _p(colidx), _p(val), float(uniform), _p(bias), float(ymax),
                                 int(bool(skip_zero)),
                                 int(nthreads or default_threads()))
        self.layer_seconds += time.perf_counter() - t0
        if rc != 0:
            raise ValueError("oracle_layer: invalid W CSR")
        self.Y, self._Z = self._Z, self.Y

    def apply(self, lay, **kw):
        """Apply an sdnngen.Layer (CSR form)."""
        self.layer(lay.rowptr, lay.colidx, lay.val, lay.uniform, lay.bias, **kw)

    def categories(self) -> np.ndarray:
        cat = np.empty(self.B, np.uint8)
        _lib().oracle_categories(self.n, self.B, _p(self.Y), _p(cat))
        return cat.astype(bool)

    def live_rows(self) -> int:
        return int(_lib().oracle_live_rows(self.n, self.B, _p(self.Y)))


def infer(n: int, layers: Iterable, rowptr, idx, val=None, ymax: float = 32.0,
          skip_zero: bool = True, nthreads: Optional[int] = None, profile: bool = False):
    """Full inference.  Returns (categories bool[B], Y_L float32[B, n], live
    profile list or None).  ``layers`` yields objects with rowptr, colidx, val,
    uniform, bias (sdnngen.Layer)."""
    o = Oracle(n, rowptr, idx, val)
    prof = [] if profile else None
    for lay in layers:
        o.apply(lay, ymax=ymax, skip_zero=skip_zero, nthreads=nthreads)
        if profile:
            prof.append(o.live_rows())
    return o.categories(), o.Y, prof


def subset_rows(rowptr, idx, val, rows):
    """CSR restricted to the given rows (row independence, invariant I4)."""
    rows = np.asarray(rows, np.int64)
    starts, ends = rowptr[rows], rowptr[rows + 1]
    lens = ends - starts
    sub_ptr = np.zeros(rows.size + 1, np.int64)
    np.cumsum(lens, out=sub_ptr[1:])
    take = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if rows.size else np.zeros(0, np.int64)
    take = take.astype(np.int64)
    return sub_ptr, idx[take], (None if val is None else val[take])


def infer_spec_rows(spec, rowptr, idx, val=None, rows=None, ymax: float = 32.0,
                    nthreads: Optional[int] = None, profile: bool = False):
    """Oracle on a subset of rows of a generated network (sdnngen spec),
    generating one CSR layer at a time (bounded host memory at 65536 x 1920).
    Row independence (invariant I4) makes the subset exact.  Returns
    (categories, Y_L, live profile, oracle seconds excluding generation)."""
    import sdnngen
    if rows is not None:
        rowptr, idx, val = subset_rows(rowptr, idx, val, rows)
    o = Oracle(spec.n, rowptr, idx, val)
    prof = [] if profile else None
    for l in range(spec.L):
        lay = sdnngen.gen_layer(spec, l, fmt="csr" if spec.wdist == "uniform" else "both")
        o.apply(lay, ymax=ymax, nthreads=nthreads)
        if profile:
            prof.append(o.live_rows())
    return o.categories(), o.Y, prof, o.layer_seconds
