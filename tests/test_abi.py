"""CPU-side checks of the C-ABI boundary: the library builds, loads and exports
every symbol include/sdnn.h declares; host validation and grouping (no device
needed); the product path never imports the oracle and fails loudly without a
device."""
import ast
import os
import re

import numpy as np
import pytest

import sdnngen as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sd():
    from paper_2004_10908_b200 import build
    build.build()
    import paper_2004_10908_b200 as sd
    sd.lib()
    return sd


def header_functions():
    src = open(os.path.join(ROOT, "include", "sdnn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdnn_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(sd):
    declared = header_functions()
    assert len(declared) >= 9
    L = sd.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(sd.EXPORTS) == declared
    assert L.sdnn_abi_version() == 3


def test_struct_layouts_match_header(sd, tmp_path):
    """The ctypes mirrors of sdnn_layer / sdnn_opts / sdnn_stats /
    sdnn_layer_info have the C header's size and field offsets (compiled with
    gcc against include/sdnn.h)."""
    import ctypes
    import subprocess
    structs = {"sdnn_layer": sd.sdnn_layer, "sdnn_opts": sd.sdnn_opts, "sdnn_stats": sd.sdnn_stats,
               "sdnn_layer_info": sd.sdnn_layer_info}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sdnn.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, f"{name}.{f}"


def test_destroy_null_is_safe(sd):
    sd.lib().sdnn_destroy(None)


def _csr(n, edges, vals=None):
    rowptr = np.zeros(n + 1, np.int64)
    edges = sorted(edges)
    for k, j in edges:
        rowptr[k + 1] += 1
    rowptr = np.cumsum(rowptr).astype(np.int64)
    colidx = np.array([j for k, j in edges], np.int32)
    return dict(rowptr=rowptr, colidx=colidx, val=vals, uniform=0.0625)


def test_validate_errors(sd):
    n = 4
    b = np.zeros(n, np.float32)
    ok = _csr(n, [(0, 1), (1, 1), (3, 2)])
    info = sd.sdnn_validate_layer(n, ok, b)
    assert info["nnz"] == 3 and info["uniform"] == 1 and info["kmax"] == 2
    bad_range = dict(ok, colidx=np.array([1, 1, 7], np.int32))
    with pytest.raises(sd.SdnnError) as e:
        sd.sdnn_validate_layer(n, bad_range, b)
    assert e.value.status == sd.SDNN_E_FORMAT
    dup = _csr(n, [(0, 1), (0, 2)])
    dup["colidx"] = np.array([1, 1], np.int32)
    with pytest.raises(sd.SdnnError) as e:
        sd.sdnn_validate_layer(n, dup, b)
    assert e.value.status == sd.SDNN_E_FORMAT and "duplicate" in str(e.value)
    nonmono = dict(ok, rowptr=np.array([0, 2, 1, 3, 3], np.int64))
    with pytest.raises(sd.SdnnError):
        sd.sdnn_validate_layer(n, nonmono, b)
    nan_w = dict(ok, val=np.array([1, np.nan, 1], np.float32))
    with pytest.raises(sd.SdnnError):
        sd.sdnn_validate_layer(n, nan_w, b)
    with pytest.raises(sd.SdnnError):
        sd.sdnn_validate_layer(n, ok, np.array([0, np.inf, 0, 0], np.float32))
    with pytest.raises(sd.SdnnError) as e:
        sd.sdnn_validate_layer(70000, ok, np.zeros(70000, np.float32))
    assert e.value.status == sd.SDNN_E_UNSUPPORTED
    info = sd.sdnn_validate_layer(n, ok, np.array([0, 0.5, 0, 0], np.float32))
    assert info["bias_nonpositive"] == 0


def test_validate_ellcol(sd):
    n = 4
    ell = np.array([[1, -1], [-1, -1], [3, 0], [2, 1]], np.int32)
    info = sd.sdnn_validate_layer(n, dict(ell=ell, ell_val=None, uniform=0.5), np.zeros(n, np.float32),
                                  fmt="ell")
    assert info["nnz"] == 5 and info["kmax"] == 2
    bad = np.array([[1, 1], [-1, -1], [3, 0], [2, 1]], np.int32)
    with pytest.raises(sd.SdnnError):
        sd.sdnn_validate_layer(n, dict(ell=bad, ell_val=None, uniform=0.5),
                               np.zeros(n, np.float32), fmt="ell")
    oob = np.array([[9, -1], [-1, -1], [3, 0], [2, 1]], np.int32)
    with pytest.raises(sd.SdnnError):
        sd.sdnn_validate_layer(n, dict(ell=oob, ell_val=None, uniform=0.5),
                               np.zeros(n, np.float32), fmt="ell")


@pytest.mark.parametrize("fmt", ["csr", "ell"])
def test_grouping_rn_rr(sd, fmt):
    n = 1024
    lay = g.gen_layer(g.rn_spec(n, 3), 1)
    info = sd.sdnn_validate_layer(n, lay, lay.bias, fmt=fmt)
    assert (info["ngroups"], info["gmax"], info["kmax"], info["regular"], info["uniform"]) == \
        (n // 32, 32, 32, 1, 1)
    info = sd.sdnn_validate_layer(n, lay, lay.bias, fmt=fmt, flags=sd.SDNN_F_NO_GROUPS)
    assert (info["ngroups"], info["gmax"]) == (n, 1)
    lay = g.gen_layer(g.rr_spec(n, 3), 1)
    info = sd.sdnn_validate_layer(n, lay, lay.bias, fmt=fmt)
    assert (info["ngroups"], info["gmax"], info["kmax"]) == (n, 1, 32)


def test_irregular_layer_info(sd):
    spec = g.random_spec(200, 1, seed=3, kmin=0, kmax=40)
    lay = g.gen_layer(spec, 0)
    info = sd.sdnn_validate_layer(200, lay, lay.bias)
    assert info["uniform"] == 0 and info["regular"] == 0 and info["kmax"] == 40
    assert info["nnz"] == lay.colidx.size


def test_no_device_fails_loudly(sd):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(sd.SdnnError) as e:
        sd.Net(64, 1)
    assert e.value.status == sd.SDNN_E_CUDA


def test_product_path_never_touches_oracle():
    """The product package must not import, link or execute anything under
    oracle/ (only tests, smoke and bench's cpu_baseline may)."""
    pkg = os.path.join(ROOT, "paper_2004_10908_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if f.endswith((".cu", ".cpp", ".h", ".py")):
                txt = open(p).read()
                assert "sdnn_oracle" not in txt and "liboracle" not in txt, p


def test_plan_steps_rn_and_rr(sd, monkeypatch):
    """Fused multi-layer passes: in a RadiX-Net layer every group is a dense
    32x32 block varying one 5-bit field of the neuron id, so the connected
    components over layers a..b span 2^|union of their fields' bits| neurons.
    A pass keeps all layers but the last in one CTA (sub-components of <= 512
    slots) and lets the last layer read across a cluster of cap/512 CTAs; the
    planner extends every pass while that holds (greedy, maximal).
    Random-regular layers have one giant component and are never fused.
    (Row-major activations: 512 slots per CTA; see the blocked variant below.)"""
    monkeypatch.setenv("SDNN_YBLOCK", "0")
    monkeypatch.setenv("SDNN_PLAN", "greedy")        # maximality is the greedy cover's property
    rn = list(g.iter_layers(g.rn_spec(1024, 24)))
    fields = [g.rn_field(1024, l) for l in range(24)]

    def comp(a, m):
        bits = set()
        for p in fields[a:a + m]:
            bits |= set(range(p, p + 5))
        return 2 ** len(bits)

    def feasible(a, m, cap):
        sub, full = comp(a, m - 1), comp(a, m)
        cta = min(cap, 512)
        return sub <= cta and -(-full // (cta // sub * sub)) <= max(1, cap // 512)

    default = sd.sdnn_plan_steps(1024, rn)                         # fusion on by default
    assert default == sd.sdnn_plan_steps(1024, rn, fuse_rows=1024)
    assert sd.sdnn_plan_steps(1024, rn, fuse_rows=4096) == sd.sdnn_plan_steps(1024, rn, fuse_rows=2048)
    for cap in (128, 256, 512, 1024, 2048):
        plan = sd.sdnn_plan_steps(1024, rn, fuse_rows=cap)
        assert sum(plan) == 24 and max(plan) > 1
        a = 0
        for m in plan:                      # every pass fits, and is maximal (greedy)
            assert m == 1 or feasible(a, m, cap)
            if a + m < 24 and m < 8 and cap <= 512:   # larger caps: the 8 KB record may end a pass first
                assert not feasible(a, m + 1, cap)
            a += m
    assert max(sd.sdnn_plan_steps(1024, rn, fuse_rows=512)) == 5   # 512-row components: 9 of 10 id bits
    assert max(sd.sdnn_plan_steps(1024, rn, fuse_rows=128)) == 2
    assert sd.sdnn_plan_steps(1024, rn, fuse_rows=0) == [1] * 24
    assert sd.sdnn_plan_steps(1024, rn, fuse_rows=64) == [1] * 24    # 2 layers need 128 rows
    assert sd.sdnn_plan_steps(1024, rn, flags=sd.SDNN_F_SATURATE) == [1] * 24
    rr = list(g.iter_layers(g.rr_spec(1024, 5)))
    assert sd.sdnn_plan_steps(1024, rr) == [1] * 5
    ka = list(g.iter_layers(g.ka_spec(1024, 20)))
    assert sd.sdnn_plan_steps(1024, ka, fuse_layers=16) == [16, 4]
    assert max(sd.sdnn_plan_steps(1024, ka, fuse_layers=2)) == 2
    big = [g.gen_layer(g.rn_spec(65536, 12), l, fmt="ell") for l in range(12)]
    assert sd.sdnn_plan_steps(65536, big, fmt="ell", fuse_rows=512) == [3, 3, 3, 3]
    assert sd.sdnn_plan_steps(65536, big, fmt="ell", fuse_rows=128) == [2] * 6
    assert sd.sdnn_plan_steps(65536, big, fmt="ell", fuse_rows=2048) == [4, 2, 4, 2]   # 4-CTA clusters; field wrap after 6


@pytest.mark.parametrize("plan", ["cost", "greedy"])
def test_plan_steps_cost_cover(sd, monkeypatch, plan):
    """The default cost-weighted cover and the greedy one both tile the layers
    with feasible passes (component cap 1024, one CTA with blocked activations);
    the cost cover never pays more than the greedy one under its own model
    (1 per pass, +0.3 for components above 512 rows)."""
    monkeypatch.setenv("SDNN_YBLOCK", "1")
    L = 72
    fields = [g.rn_field(65536, l) for l in range(L)]
    big = [g.gen_layer(g.rn_spec(65536, L), l, fmt="ell") for l in range(L)]

    def comp(a, m):
        bits = set()
        for p in fields[a:a + m]:
            bits |= set(range(p, p + 5))
        return 2 ** len(bits)

    def cost(plan_):
        a, c = 0, 0.0
        for m in plan_:
            assert comp(a, m) <= 1024 or m == 1
            c += 1.0 + (0.3 if m > 1 and comp(a, m) > 512 else 0.0)
            a += m
        assert a == L
        return c

    monkeypatch.setenv("SDNN_PLAN", plan)
    mine = cost(sd.sdnn_plan_steps(65536, big, fmt="ell"))
    monkeypatch.setenv("SDNN_PLAN", "greedy")
    assert mine <= cost(sd.sdnn_plan_steps(65536, big, fmt="ell")) + 1e-9


def test_plan_steps_blocked_layout(sd, monkeypatch):
    """With position-blocked activations (the default) a CTA holds up to 1024
    slots (16-position tiles), so the default cap 1024 needs no cluster: every
    pass is feasible for one CTA and maximal, except where its metadata
    record (<= 10224 B) ends it first."""
    monkeypatch.setenv("SDNN_YBLOCK", "1")
    fields = [g.rn_field(65536, l) for l in range(24)]
    big = [g.gen_layer(g.rn_spec(65536, 24), l, fmt="ell") for l in range(24)]

    def comp(a, m):
        bits = set()
        for p in fields[a:a + m]:
            bits |= set(range(p, p + 5))
        return 2 ** len(bits)

    plan = sd.sdnn_plan_steps(65536, big, fmt="ell")
    assert sum(plan) == 24 and max(plan) == 3   # (a lone layer runs as a one-layer pass)
    a = 0
    for m in plan:
        assert comp(a, m) <= 1024
        a += m
    monkeypatch.setenv("SDNN_YBLOCK", "0")
    assert sum(sd.sdnn_plan_steps(65536, big, fmt="ell")) == 24


def identity_layer(n):
    """W = I, uniform 1, bias 0: Y -> min(max(Y, 0), 32) (the identity on Y in [0, 32])."""
    from types import SimpleNamespace
    return SimpleNamespace(rowptr=np.arange(n + 1, dtype=np.int64), colidx=np.arange(n, dtype=np.int32),
                           val=None, uniform=1.0, bias=np.zeros(n, np.float32),
                           ell=np.arange(n, dtype=np.int32).reshape(n, 1), ell_val=None)


def test_plan_splits_oversized_records(sd, monkeypatch):
    """A pass's per-component metadata record must fit kPassRecMax (10224 B):
    [identity, identity, rn0, rn1] forms 128-row components (plan [4] by the
    component cap alone) but each identity layer has 128 singleton groups per
    component (~8.4 KB of record each), so the pass drops its last layer (32-row
    components, ~4.4 KB) and the rest is planned again -> [3, 1];
    [identity, rn0, rn1] (~9.2 KB) still fits."""
    n = 1024
    rn = [g.gen_layer(g.rn_spec(n, 2), l) for l in range(2)]
    ident = identity_layer(n)
    assert sd.sdnn_plan_steps(n, rn) == [2]
    assert sd.sdnn_plan_steps(n, [ident] + rn) == [3]
    assert sd.sdnn_plan_steps(n, [ident, ident] + rn) == [3, 1]
    assert sd.sdnn_plan_steps(n, [ident] + rn, fuse_layers=2) == [2, 1]


def test_plan_steps_not_in_place_not_fused(sd):
    """A layer whose source rows feed several groups cannot be the non-last
    layer of a pass (its groups could not overwrite their source slots)."""
    n = 256
    lays = list(g.iter_layers(g.random_spec(n, 3, seed=4, kmin=2, kmax=4, wdist="uniform")))
    assert sd.sdnn_plan_steps(n, lays, fuse_rows=128) == [1, 1, 1]


def test_plan_steps_nonuniform_not_fused(sd):
    lays = list(g.iter_layers(g.rn_spec(1024, 4, wdist="random")))
    assert sd.sdnn_plan_steps(1024, lays) == [1, 1, 1, 1]


def test_binding_constants_match_header(sd):
    """Every SDNN_F_* / SDNN_E_* / SDNN_W_* value in include/sdnn.h is mirrored
    exactly by the Python binding."""
    src = open(os.path.join(ROOT, "include", "sdnn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    vals = {}
    for name, expr in re.findall(r"\b(SDNN_[FEW]_[A-Z_]+|SDNN_OK)\s*=\s*([^,}\n]+)", src):
        expr = expr.strip().replace("u <<", " <<")
        vals[name] = eval(expr)
    assert len(vals) >= 15
    for name, v in vals.items():
        assert getattr(sd, name) == v, name
