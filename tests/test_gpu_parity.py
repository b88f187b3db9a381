"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.  The bar (BASELINE.json north_star):
categories bit-exact; activations within 1e-5 rel / 1e-6 abs -- this build is
held to the stricter bit-exact standard for activations too, because both
sides evaluate the same canonical fp32 chain (A5)."""
import numpy as np
import pytest

import oracle
import sdnngen as g

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6            # north_star tolerance (asserted in addition to bit-exactness)


@pytest.fixture(scope="module")
def sd():
    from paper_2004_10908_b200 import build
    build.build()
    import paper_2004_10908_b200 as sd
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return sd


def assert_parity(cats_gpu, Y_gpu, cats_or, Y_or):
    assert np.array_equal(cats_gpu, np.flatnonzero(cats_or).astype(np.int32))
    if Y_gpu is not None:
        np.testing.assert_allclose(Y_gpu, Y_or, rtol=RTOL, atol=ATOL)
        assert np.array_equal(Y_gpu.view(np.uint32), Y_or.view(np.uint32))


def run_gpu(sd, n, layers, rp, idx, val, fmt="csr", flags=0, ymax=32.0, want_y=True,
            fuse_rows=-1, fuse_layers=-1, resident_from=-1, stream_slots=0):
    with sd.Net.from_layers(n, layers, fmt=fmt, flags=flags, ymax=ymax, fuse_rows=fuse_rows,
                            fuse_layers=fuse_layers, resident_from=resident_from,
                            stream_slots=stream_slots) as net:
        cats, Y = net.infer(rp, idx, val, want_y=want_y)
        st = net.stats()
    return cats, Y, st


FLAGS = [0, 1, 2, 4]   # default, NO_COMPACT, NO_GROUPS, NO_GRAPH


@pytest.mark.parametrize("name", ["H1", "H2", "H3", "H3_ymax2", "H4", "H5"])
@pytest.mark.parametrize("flags", FLAGS)
def test_hand_nets(sd, hand_nets, name, flags):
    net = hand_nets[name]
    layers = [dict(l, uniform=0.0) for l in net.layers]
    cats, Y, _ = run_gpu(sd, net.n, layers, net.y0_rowptr, net.y0_idx, net.y0_val,
                         flags=flags, ymax=net.ymax)
    assert cats.tolist() == net.expected_categories
    assert np.array_equal(Y.view(np.uint32), net.expected_Y.view(np.uint32))


@pytest.fixture(scope="module")
def c1():
    """configs[0]: 1024 neurons x 120 layers, 32 nnz/column, 1000 binary inputs."""
    spec = g.rn_spec(1024, 120)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(1024, 1000)
    cats, Y, prof = oracle.infer(1024, layers, rp, idx, None, profile=True)
    return spec, layers, rp, idx, cats, Y, prof


@pytest.mark.parametrize("fmt", ["csr", "ell"])
@pytest.mark.parametrize("flags", FLAGS)
def test_c1_full(sd, c1, fmt, flags):
    spec, layers, rp, idx, cats, Y, prof = c1
    cg, Yg, st = run_gpu(sd, 1024, layers, rp, idx, None, fmt=fmt, flags=flags)
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof
    assert 0 < cats.sum() < cats.size


@pytest.mark.parametrize("resident_from", [0, 1, 7, 24, 119])
def test_c1_smem_resident(sd, c1, resident_from):
    """SMEM-resident tail (P = 16 positions per CTA at N = 1024): layers before
    resident_from stream with compaction, the rest stay in shared memory."""
    spec, layers, rp, idx, cats, Y, prof = c1
    for flags in (0, 1):                                  # with / without compaction
        cg, Yg, st = run_gpu(sd, 1024, layers, rp, idx, None, fmt="ell", flags=flags,
                             resident_from=resident_from)
        assert st["resident_layers"] == 120 - resident_from and st["path"] & 2
        assert_parity(cg, Yg, cats, Y)
        assert st["live_rows"] == prof


@pytest.mark.parametrize("n,L,B", [(4096, 12, 301), (2048, 9, 77), (512, 10, 500), (256, 6, 65)])
def test_smem_resident_widths(sd, n, L, B):
    """P = 4 / 8 / 32 / 32 positions per CTA; ragged last CTA."""
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(n, B, seed=n)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, None, profile=True)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, None, fmt="ell", resident_from=2)
    assert st["resident_layers"] == L - 2
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof


def test_smem_resident_irregular_and_positive_bias(sd):
    """Uniform-valued irregular layers (1..32 sources per column, singleton
    groups, per-neuron bias including positive values -> no compaction, no
    early stop)."""
    n, L = 384, 6
    spec = g.random_spec(n, L, seed=77, kmin=1, kmax=32, wdist="uniform", bias=(-0.4, 0.1))
    layers = list(g.iter_layers(spec))
    for lay in layers:
        lay.uniform = 0.1875
    rp, idx, val = g.random_inputs(n, 200, seed=78, density=0.3, lo=0.0, hi=2.0)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val, resident_from=0)
    assert st["resident_layers"] == L and st["compaction"] == 0
    assert_parity(cg, Yg, cats, Y)


def test_smem_resident_ka(sd):
    from test_oracle_pins import ka_expected
    spec = g.ka_spec(1024, 40)
    layers = list(g.iter_layers(spec))
    rp, idx, cnt = g.ka_inputs(1024, 1500, seed=9)
    cg, Yg, st = run_gpu(sd, 1024, layers, rp, idx, None, fmt="ell", resident_from=3)
    assert st["resident_layers"] == 37
    Yx = ka_expected(spec, cnt)
    assert np.array_equal(Yg.view(np.uint32), Yx.view(np.uint32))
    assert np.array_equal(cg, np.flatnonzero((Yx > 0).any(1)))


@pytest.mark.parametrize("fuse_rows,fuse_layers", [(0, -1), (128, -1), (256, -1),
                                                   (256, 2), (256, 16), (512, -1), (512, 3),
                                                   (512, 16), (1024, -1), (1024, 16),
                                                   (2048, -1), (2048, 4)])
def test_fused_passes_rn(sd, fuse_rows, fuse_layers):
    """Multi-layer passes (model decomposition): single-CTA passes (cap <= 512:
    tiles of 128 / 64 / 32 positions for 128- / 256- / 512-row components) and
    2- / 4-CTA cluster passes whose last layer reads through distributed shared
    memory (cap 1024 / 2048), pass lengths 2..16, compaction between passes,
    ragged batch."""
    n, L, B = 1024, 40, 700
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(n, B, seed=31)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, None, profile=True)
    for flags in (0, 4, 512):                 # default, stream loop, SDNN_F_SHARE_VALUES
        cg, Yg, st = run_gpu(sd, n, layers, rp, idx, None, fmt="ell", flags=flags,
                             fuse_rows=fuse_rows, fuse_layers=fuse_layers)
        assert (st["fused_layers"] > 0) == (fuse_rows > 0)
        assert_parity(cg, Yg, cats, Y)
        assert st["live_rows"] == prof


@pytest.mark.parametrize("spec_fn,n,fuse_rows", [("rn", 8192, 4096), ("rn", 8192, 2048), ("rn", 8192, -1),
                                                  ("plain", 4096, -1), ("plain", 8192, -1)])
def test_large_caps_and_schedules(sd, spec_fn, n, fuse_rows):
    """Component caps above one CTA at N = 8192 (the planner must fall back from
    shapes without a kernel instance), and the plain field schedule
    whose 1024-row passes have two layers (k_pass_wide) -- full Y_L parity."""
    L, B = 24, 300
    spec = g.rn_spec(n, L) if spec_fn == "rn" else g.rn_plain_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(n, B, seed=41)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, None, profile=True)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, None, fmt="ell", fuse_rows=fuse_rows)
    assert st["fused_layers"] > 0
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof


def test_fused_t64_and_irregular_components(sd):
    """N = 512: component sizes 128 / 256 -> tiles of T = 64 / 32 positions."""
    n, L = 512, 30
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, 333, seed=12, density=0.4, lo=0.0, hi=1.5)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    for cap in (128, 256):
        cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val, fuse_rows=cap)
        assert st["fused_layers"] > 0
        assert_parity(cg, Yg, cats, Y)


@pytest.mark.parametrize("cap", [128, 512, 2048])
def test_fused_nonuniform_bias(sd, cap):
    """Per-neuron biases (record carries a bias per member) next to uniform
    ones (stored once): RN structure with seeded biases in [-0.6, -0.2] on
    every other layer, binary and real-valued inputs."""
    import dataclasses
    n, L = 1024, 20
    layers = list(g.iter_layers(g.rn_spec(n, L)))
    rng = np.random.default_rng(77)
    layers = [dataclasses.replace(la, bias=rng.uniform(-0.6, -0.2, n).astype(np.float32)) if l % 2 else la
              for l, la in enumerate(layers)]
    rp, idx = g.ms_inputs(n, 517, seed=8)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, None, profile=True)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, None, fuse_rows=cap, flags=sd.SDNN_F_NO_RESIDENT)
    assert st["fused_layers"] > 0
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof


@pytest.mark.parametrize("share", [0, 512])
def test_fused_ka_long_passes(sd, share):
    """16-layer passes over KA blocks; with SDNN_F_SHARE_VALUES every layer but
    the last stores one value per group (free-slot allocation after the first)."""
    from test_oracle_pins import ka_expected
    spec = g.ka_spec(2048, 40)
    layers = list(g.iter_layers(spec))
    rp, idx, cnt = g.ka_inputs(2048, 999, seed=5)
    cg, Yg, st = run_gpu(sd, 2048, layers, rp, idx, None, fmt="ell", fuse_rows=256,
                         fuse_layers=16, flags=sd.SDNN_F_NO_RESIDENT | share)
    assert st["steps"] == 3 and st["fused_layers"] == 40
    Yx = ka_expected(spec, cnt)
    assert np.array_equal(Yg.view(np.uint32), Yx.view(np.uint32))
    assert np.array_equal(cg, np.flatnonzero((Yx > 0).any(1)))


def test_fused_record_split_and_singletons(sd):
    """Identity layers (singleton groups, K = G = 1) inside fused passes: a pass
    whose metadata record would exceed 8 KB is split; [identity, rn0] fuses
    with 32 singleton groups per component."""
    from test_abi import identity_layer
    n, B = 1024, 613
    rn = [g.gen_layer(g.rn_spec(n, 6), l) for l in range(6)]
    layers = [identity_layer(n)] + rn[:3] + [identity_layer(n)] + rn[3:]
    rp, idx = g.ms_inputs(n, B, seed=41)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, None, profile=True)
    for fl in (2, -1):
        cg, Yg, st = run_gpu(sd, n, layers, rp, idx, None, fuse_layers=fl, flags=sd.SDNN_F_NO_RESIDENT)
        assert st["fused_layers"] > 0
        assert_parity(cg, Yg, cats, Y)
        assert st["live_rows"] == prof


# ---------------------------------------------------------------------------
# f3: weight streaming through a ring of device slots (stream_slots > 0)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("slots", [1, 2, 3])
@pytest.mark.parametrize("flags", [0, 4])
def test_weight_streaming_c1(sd, c1, slots, flags):
    """Fused passes and single layers with their weight blocks copied into S
    slots during the chain (graph and stream loop): bit-exact, and every step's
    block crosses the host link once per inference."""
    spec, layers, rp, idx, cats, Y, prof = c1
    cg, Yg, st = run_gpu(sd, 1024, layers, rp, idx, None, fmt="ell", flags=flags, stream_slots=slots)
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof
    assert st["resident_layers"] == 0 and st["fused_layers"] > 0
    assert st["stream_bytes"] > 0 and st["packed_weight_bytes"] == 0
    assert 0 < st["stream_slot_bytes"] < st["stream_bytes"]


def test_weight_streaming_general_and_saturate(sd):
    """Per-slot weights (general kernel) and f2 saturation tracking read their
    arrays from the slot ring; repeated inferences reuse the captured graph."""
    n, L = 300, 7
    spec = g.random_spec(n, L, seed=91, kmin=0, kmax=40, bias=(-0.3, 0.0))
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, 257, seed=92)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    with sd.Net.from_layers(n, layers, stream_slots=2) as net:
        for _ in range(3):
            cg, Yg = net.infer(rp, idx, val, want_y=True)
            assert_parity(cg, Yg, cats, Y)
    spec = g.rn_spec(1024, 40)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(1024, 640, seed=93)
    cats, Y, _ = oracle.infer(1024, layers, rp, idx, None)
    cg, Yg, st = run_gpu(sd, 1024, layers, rp, idx, None, fmt="ell", flags=sd.SDNN_F_SATURATE,
                         stream_slots=2)
    assert_parity(cg, Yg, cats, Y)
    assert st["retired_rows"] > 0


# ---------------------------------------------------------------------------
# f2: exact saturated-row retirement (SDNN_F_SATURATE)
# ---------------------------------------------------------------------------
def test_saturate_c1(sd, c1):
    spec, layers, rp, idx, cats, Y, prof = c1
    cg, Yg, st = run_gpu(sd, 1024, layers, rp, idx, None, fmt="ell", flags=sd.SDNN_F_SATURATE)
    assert_parity(cg, Yg, cats, Y)
    # RN survivors saturate to all-32 rows and are retired; the survivor profile
    # still counts them
    assert 0 < st["retired_rows"] <= cats.sum() and st["live_rows"] == prof


def test_saturate_ka_and_device_bitmask(sd):
    import torch
    from test_oracle_pins import ka_expected
    spec = g.ka_spec(1024, 30)
    layers = list(g.iter_layers(spec))
    rp, idx, cnt = g.ka_inputs(1024, 1200, seed=13)
    Yx = ka_expected(spec, cnt)
    with sd.Net.from_layers(1024, layers, fmt="ell", flags=sd.SDNN_F_SATURATE) as net:
        cg, Yg = net.infer(rp, idx, None, want_y=True)
        # KA rows keep one saturated group and zeros elsewhere: never all-YMAX
        assert net.stats()["retired_rows"] == 0
        dev = torch.device("cuda", 0)
        alive = net.infer_torch(torch.from_numpy(rp).to(dev), torch.from_numpy(idx).to(dev))
        torch.cuda.synchronize()
        assert np.array_equal(sd.bitmask_to_ids(alive.cpu().numpy(), 1200), cg)
    assert np.array_equal(Yg.view(np.uint32), Yx.view(np.uint32))
    assert np.array_equal(cg, np.flatnonzero((Yx > 0).any(1)))


def test_saturate_respects_non_preserving_suffix(sd):
    """A late layer with some bias < -32 maps all-32 rows to non-saturated rows,
    so nothing may be retired before it."""
    n, L = 1024, 30
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    layers[25].bias = layers[25].bias.copy()
    layers[25].bias[::7] = -40.0                         # 64 - 40 = 24 < 32 = YMAX
    rp, idx = g.ms_inputs(n, 600, seed=3)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, None)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, None, fmt="ell", flags=sd.SDNN_F_SATURATE)
    assert_parity(cg, Yg, cats, Y)


def test_ka_known_answer(sd):
    from test_oracle_pins import ka_expected
    spec = g.ka_spec(1024, 24)
    layers = list(g.iter_layers(spec))
    rp, idx, cnt = g.ka_inputs(1024, 2000, seed=21)
    cg, Yg, _ = run_gpu(sd, 1024, layers, rp, idx, None, fmt="ell")
    Yx = ka_expected(spec, cnt)
    assert np.array_equal(Yg.view(np.uint32), Yx.view(np.uint32))
    assert np.array_equal(cg, np.flatnonzero((Yx > 0).any(1)))


def test_rr_general_gather(sd):
    n, L = 2048, 20
    spec = g.rr_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, 700, seed=4, density=0.3, lo=0.0, hi=3.0)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val)
    assert st["max_group"] == 1
    assert_parity(cg, Yg, cats, Y)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_irregular_random_weights(sd, seed):
    """Per-slot weights (general kernel), K up to 40 (>32 path), empty columns,
    width not a multiple of 32, negative inputs, some positive biases (so
    compaction must switch itself off)."""
    n, L = 300, 5
    spec = g.random_spec(n, L, seed=40 + seed, kmin=0, kmax=40, bias=(-0.3, 0.05))
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, 333, seed=50 + seed)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    for flags in (0, 2):
        cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val, flags=flags)
        assert st["compaction"] == 0
        assert_parity(cg, Yg, cats, Y)


def test_rn_random_weights_grouped(sd):
    """Groups of 32 with per-slot weights: one source load, 32 chains."""
    n, L = 1024, 12
    spec = g.rn_spec(n, L, wdist="random", bias=-0.2)
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, 500, seed=8, density=0.3, lo=0.0, hi=2.0)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    for fmt in ("csr", "ell"):
        cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val, fmt=fmt)
        assert st["max_group"] == 32
        assert_parity(cg, Yg, cats, Y)


def _pair_layer(n, w, bias):
    """Column j has sources j and j^1 (a group of 2 per pair) with weights
    (+w, -w) when w is a pair of values, or uniform w; bias per column."""
    from types import SimpleNamespace
    ell = np.stack([np.arange(n) & ~1, np.arange(n) | 1], 1).astype(np.int32)
    rows = np.repeat(np.arange(n), 2)                       # CSR row k feeds columns k&~1, k|1
    cols = np.stack([np.arange(n) & ~1, np.arange(n) | 1], 1).reshape(-1).astype(np.int32)
    rowptr = np.arange(0, 2 * n + 1, 2, dtype=np.int64)
    if np.ndim(w) == 0:
        val = ell_val = None
        uni = float(w)
    else:
        # W[k][j]: +w0 if k is even, -w0 if k is odd (for both columns of the pair)
        val = np.where(rows % 2 == 0, w[0], w[1]).astype(np.float32)
        ell_val = np.tile(np.array([w[0], w[1]], np.float32), (n, 1))
        uni = 0.0
    return SimpleNamespace(rowptr=rowptr, colidx=cols, val=val, uniform=uni,
                           bias=np.asarray(bias, np.float32), ell=ell, ell_val=ell_val)


def test_signed_zero_and_exact_cancellation(sd):
    """The 2-FMNMX clamp and the max-bias liveness test rely on z never being
    -0 (A6 note): exact cancellations (+w, -w on equal inputs),
    -0.0 biases, -0.0 and negative inputs, through the general (per-slot) and
    uniform kernels, fused and unfused.  Outputs and categories bit-exact."""
    n, B = 256, 97
    r = np.random.default_rng(2026)
    dense = np.zeros((B, n), np.float32)
    for i in range(B):
        for k in range(0, n, 2):
            u = r.random()
            if u < 0.3:
                dense[i, k] = dense[i, k + 1] = np.float32(r.choice([0.5, 1.25, 3.0]))   # cancels
            elif u < 0.4:
                dense[i, k] = -0.0
                dense[i, k + 1] = np.float32(r.uniform(0, 2))
            elif u < 0.5:
                dense[i, k] = np.float32(r.uniform(-1, 2))
    rp, idx, val = g.csr_from_dense(dense)
    val[r.random(val.size) < 0.05] = -0.0
    bias_negzero = np.full(n, -0.0, np.float32)
    bias_mixed = np.where(np.arange(n) % 3 == 0, -0.0, -0.125).astype(np.float32)
    layers = [_pair_layer(n, (0.75, -0.75), bias_negzero), _pair_layer(n, 0.5, bias_mixed),
              _pair_layer(n, 2.0, bias_mixed), _pair_layer(n, (1.0, -1.0), bias_negzero),
              _pair_layer(n, 0.25, bias_mixed), _pair_layer(n, 1.5, bias_negzero)]
    assert sd.sdnn_plan_steps(n, layers) == [1, 2, 1, 2]            # fused uniform pairs
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val)
    assert 0 < cats.sum() < B
    for flags, fr in ((0, -1), (0, 0), (2, -1), (4, -1)):
        cg, Yg, _ = run_gpu(sd, n, layers, rp, idx, val, flags=flags | sd.SDNN_F_NO_RESIDENT, fuse_rows=fr)
        assert_parity(cg, Yg, cats, Y)
    cg, Yg, _ = run_gpu(sd, n, layers, rp, idx, val, resident_from=0)
    assert_parity(cg, Yg, cats, Y)


@pytest.mark.parametrize("B", [1, 31, 33, 127, 129, 1000, 4097])
def test_ragged_batches(sd, B):
    n, L = 1024, 16
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(n, B, seed=77)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, None)
    cg, Yg, _ = run_gpu(sd, n, layers, rp, idx, None, fmt="ell")
    assert_parity(cg, Yg, cats, Y)


def test_edge_cases(sd):
    n = 64
    spec = g.rn_spec(n, 3)
    layers = list(g.iter_layers(spec))
    # empty batch
    cg, Yg, _ = run_gpu(sd, n, layers, np.zeros(1, np.int64), np.zeros(0, np.int32), None)
    assert cg.size == 0 and Yg.shape == (0, n)
    # all rows empty -> nothing survives, everything compacted away after densify
    rp = np.zeros(40, np.int64)
    cg, Yg, st = run_gpu(sd, n, layers, rp, np.zeros(0, np.int32), None)
    assert cg.size == 0 and not Yg.any()
    # zero layers: categories = rows with a positive entry
    rp = np.array([0, 2, 2, 3, 4], np.int64)
    idx = np.array([1, 3, 0, 5], np.int32)
    val = np.array([0.5, -1.0, -2.0, 3.0], np.float32)
    with sd.Net(n, 0) as net:
        cg, Yg = net.infer(rp, idx, val, want_y=True)
    assert cg.tolist() == [0, 3]
    assert np.array_equal(Yg, g.dense_from_csr(rp, idx, val, n))
    # invalid Y0 is rejected by the host call
    with sd.Net.from_layers(n, layers) as net:
        with pytest.raises(sd.SdnnError):
            net.infer(np.array([0, 2], np.int64), np.array([3, 3], np.int32), None)
        with pytest.raises(sd.SdnnError):
            net.infer(np.array([0, 1], np.int64), np.array([n], np.int32), None)
    # inference before all layers are set
    net = sd.Net(n, 2)
    with pytest.raises(sd.SdnnError) as e:
        net.infer(np.array([0, 1], np.int64), np.array([3], np.int32), None)
    assert e.value.status == sd.SDNN_E_STATE
    net.close()


def test_device_api_torch(sd, c1):
    import torch
    spec, layers, rp, idx, cats, Y, prof = c1
    with sd.Net.from_layers(1024, layers, fmt="ell") as net:
        dev = torch.device("cuda:0")
        rp_t = torch.from_numpy(rp).to(dev)
        idx_t = torch.from_numpy(idx).to(dev)
        y_t = torch.empty((rp.size - 1, 1024), dtype=torch.float32, device=dev)
        alive = net.infer_torch(rp_t, idx_t, None, y_t=y_t)
        torch.cuda.synchronize()
        ids = sd.bitmask_to_ids(alive.cpu().numpy(), rp.size - 1)
        assert np.array_equal(ids, np.flatnonzero(cats))
        assert np.array_equal(y_t.cpu().numpy().view(np.uint32), Y.view(np.uint32))
        # on a side stream, twice (determinism, reuse of the captured graph)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            a2 = net.infer_torch(rp_t, idx_t, None)
            a3 = net.infer_torch(rp_t, idx_t, None, alive_t=torch.empty_like(a2))
        s.synchronize()
        assert torch.equal(a2, alive) and torch.equal(a3, alive)


def test_row_independence_on_gpu(sd, c1):
    spec, layers, rp, idx, cats, Y, prof = c1
    rows = np.random.default_rng(5).choice(rp.size - 1, 123, replace=False)
    srp, sidx, _ = oracle.subset_rows(rp, idx, None, rows)
    cg, Yg, _ = run_gpu(sd, 1024, layers, srp, sidx, None)
    assert np.array_equal(cg, np.flatnonzero(cats[rows]))
    assert np.array_equal(Yg.view(np.uint32), Y[rows].view(np.uint32))


# ---------------------------------------------------------------------------
# BASELINE.json's full sizes, in the launch configuration bench.py times: the
# full 60000-input batch on the GPU, checked on sampled rows the oracle
# computes one by one (row independence, I4), sentinel rows included.
# ---------------------------------------------------------------------------
def _full_size(sd, spec, nsample, batch=60000, flags=0):
    """The full batch on the GPU (default options = the benchmarked launch
    configuration), then on `nsample` random rows plus the sentinel rows:
    categories bit-exact AND final activations Y_L bit-exact and within the
    north_star tolerance, the rows gathered on the device (sdnn_gather_rows)
    so no [batch x N] host copy is needed."""
    n, L = spec.n, spec.L
    rp, idx = g.ms_inputs(n, batch)
    with sd.Net.from_spec(spec, fmt="ell", threads=8, flags=flags) as net:
        cats, _ = net.infer(rp, idx, None)
        st = net.stats()
        r = np.random.default_rng(n ^ L)
        sent = [i for i in (998, 999, 1998, 1999, batch - 2, batch - 1) if i < batch]
        rows = np.unique(np.concatenate([r.choice(batch, nsample, replace=False), sent])).astype(np.int32)
        Yg = net.gather_rows(rows)
        Yg2 = net.gather_rows(rows[::-1].copy())[::-1]                # any order
    oc, oY, _, _ = oracle.infer_spec_rows(spec, rp, idx, None, rows)
    got = np.isin(rows, cats)
    assert np.array_equal(got, oc), rows[got != oc]
    np.testing.assert_allclose(Yg, oY, rtol=RTOL, atol=ATOL)
    assert np.array_equal(Yg.view(np.uint32), oY.view(np.uint32))
    assert np.array_equal(Yg2, Yg)
    assert np.array_equal((Yg > 0).any(1), got)
    if spec.wdist == "uniform":
        assert got[np.isin(rows, [999, 1999, batch - 1])].all()   # all-ones sentinels
    assert not got[np.isin(rows, [998, 1998, batch - 2])].any()   # empty sentinels
    # survivor profile sanity: non-increasing, final == number of categories
    live = st["live_rows"]
    assert all(a >= b for a, b in zip(live, live[1:])) and live[-1] == cats.size
    return cats, st, oY


def test_full_size_c2(sd):
    _full_size(sd, g.rn_spec(4096, 480), 200)


@pytest.mark.slow
def test_full_size_c3(sd):
    _full_size(sd, g.rn_spec(16384, 1920), 96)


@pytest.mark.slow
def test_full_size_c4(sd):
    cats, st, oY = _full_size(sd, g.rn_spec(65536, 1920), 64)
    assert st["path"] & 4                      # the benchmarked (position-blocked) layout
    assert st["steps"] < 1920                  # fused passes (the cost-cover plan)


@pytest.mark.slow
def test_full_size_plain_schedule_c3(sd):
    """SURVEY 8.4's non-overlapping field schedule (R-W5) at C3 size: a
    different pass structure (2-layer passes of 1024-row components)."""
    cats, st, oY = _full_size(sd, g.rn_plain_spec(16384, 1920), 64)
    assert st["fused_layers"] == 1920 and 0.2 * 60000 < cats.size < 0.7 * 60000


@pytest.mark.slow
def test_full_size_per_slot_weights_c3_width(sd):
    """General weights (one fp32 value per slot, RN structure, bias chosen so
    ~45 % of the rows survive) at C3 width on the full 60,000-input batch."""
    cats, st, oY = _full_size(sd, g.rw_spec(16384, 480), 64)
    assert st["fused_layers"] == 0 or st["max_group"] == 32
    assert 0.2 * 60000 < cats.size < 0.7 * 60000
    assert (oY > 0).any() and ((oY > 0) & (oY < 32)).any()      # unsaturated values are compared too


def test_gather_rows_edge_cases(sd, c1):
    """Rows out of range and dead rows gather as zeros; repeated rows; before
    any inference the call is refused."""
    spec, layers, rp, idx, cats, Y, prof = c1
    with sd.Net.from_layers(1024, layers, fmt="ell") as net:
        with pytest.raises(sd.SdnnError) as e:
            net.gather_rows(np.array([0], np.int32))
        assert e.value.status == sd.SDNN_E_STATE
        net.infer(rp, idx, None)
        rows = np.array([0, 5, 5, -1, 1000, 999, 998, 3], np.int32)
        Yg = net.gather_rows(rows)
    for q, r in enumerate(rows):
        want = Y[r] if 0 <= r < 1000 else np.zeros(1024, np.float32)
        assert np.array_equal(Yg[q].view(np.uint32), want.view(np.uint32))


def ragged_block_layers(n, L, w, seed, sb=64, shift=0.0, bmin=1):
    """Block-diagonal layers inside super-blocks of `sb` neurons: every layer
    splits each super-block into dense blocks of 1..32 neurons (K = G = block
    size, sources a seeded permutation of the block's input neurons), so fused
    passes see groups of different K and G side by side in one warp; odd
    layers carry per-neuron biases, even ones a uniform bias."""
    rng = np.random.default_rng(seed)
    layers = []
    for l in range(L):
        ks, js = [], []
        for s0 in range(0, n, sb):
            outs = s0 + rng.permutation(sb)
            ins = s0 + rng.permutation(sb)
            p = 0
            while p < sb:
                sz = int(min(sb - p, rng.integers(bmin, 33)))
                for j in outs[p:p + sz]:
                    for k in ins[p:p + sz]:
                        ks.append(k)
                        js.append(j)
                p += sz
        ks, js = np.array(ks, np.int64), np.array(js, np.int64)
        o = np.lexsort((js, ks))
        ks, js = ks[o], js[o]
        rowptr = np.zeros(n + 1, np.int64)
        np.add.at(rowptr, ks + 1, 1)
        rowptr = np.cumsum(rowptr)
        kmax = int(np.bincount(js, minlength=n).max())
        ell = np.full((n, kmax), -1, np.int32)
        fill = np.zeros(n, np.int64)
        for k, j in zip(ks, js):
            ell[j, fill[j]] = k
            fill[j] += 1
        bias = (rng.uniform(-0.3 + shift, shift, n) if l % 2 else np.full(n, -0.1 + shift)).astype(np.float32)
        layers.append(g.Layer(rowptr, js.astype(np.int32), None, ell, None, float(w), bias))
    return layers


@pytest.mark.parametrize("sb,bmin,shift", [(64, 1, -0.8), (128, 1, -0.5), (512, 24, -0.7)])
def test_fused_ragged_groups(sd, sb, bmin, shift):
    """Fused passes whose groups differ in K and G inside one warp (the padded
    zero-weight chain path, partial member loops, several unit rounds per
    layer, late tile release), per-neuron and uniform biases, real-valued
    inputs; components of sb rows -> tiles of 256 / 128 / 32 positions.
    Bit-exact against the oracle."""
    n, L = 1024, 12
    layers = ragged_block_layers(n, L, 0.125, seed=3, sb=sb, shift=shift, bmin=bmin)
    rp, idx, val = g.random_inputs(n, 389, seed=21, density=0.3, lo=0.0, hi=2.0)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, val, profile=True)
    assert 0 < len(np.flatnonzero(cats)) < 389
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val, flags=sd.SDNN_F_NO_RESIDENT)
    assert st["fused_layers"] >= L // 2
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof


@pytest.mark.parametrize("yblk", ["1", "0"])
@pytest.mark.parametrize("n,L,B", [(1024, 40, 700), (512, 30, 333), (2048, 24, 1100)])
def test_blocked_layout_on_off(sd, monkeypatch, yblk, n, L, B):
    """Position-blocked activations (every step a fused pass, lone layers as
    one-layer passes: Y is [B/32][N][32] with per-boundary storage orders)
    against the neuron-major layout: both bit-exact against the oracle, path
    bit 2 reports the layout."""
    monkeypatch.setenv("SDNN_YBLOCK", yblk)
    layers = list(g.iter_layers(g.rn_spec(n, L)))
    rp, idx, val = g.random_inputs(n, B, seed=n + L, density=0.3, lo=0.0, hi=1.5)
    cats, Y, prof = oracle.infer(n, layers, rp, idx, val, profile=True)
    cg, Yg, st = run_gpu(sd, n, layers, rp, idx, val, flags=sd.SDNN_F_NO_RESIDENT, fuse_rows=512)
    assert bool(st["path"] & 4) == (yblk == "1")     # lone layers run as one-layer passes
    assert_parity(cg, Yg, cats, Y)
    assert st["live_rows"] == prof


def test_pipelined_submit_wait(sd, c1):
    """sdnn_infer_submit / sdnn_infer_wait: two submissions in flight (the
    second's input copy overlaps the first's layers), each bit-exact against
    the oracle; a third submission, or sdnn_infer, while two are outstanding is
    refused; invalid input is reported by the wait."""
    spec, layers, rp, idx, cats, Y, prof = c1
    rows = np.arange(0, 1000, 3)
    srp, sidx, _ = oracle.subset_rows(rp, idx, None, rows)
    with sd.Net.from_layers(1024, layers, fmt="ell") as net:
        t0 = net.infer_submit(rp, idx)
        t1 = net.infer_submit(srp, sidx)
        with pytest.raises(sd.SdnnError) as e:
            net.infer_submit(rp, idx)
        assert e.value.status == sd.SDNN_E_STATE
        with pytest.raises(sd.SdnnError):
            net.infer(rp, idx, None)
        assert np.array_equal(net.infer_wait(t0), np.flatnonzero(cats))
        t2 = net.infer_submit(rp, idx)                      # slot of t0 again, t1 still in flight
        assert np.array_equal(net.infer_wait(t1), np.flatnonzero(cats[rows]))
        assert np.array_equal(net.infer_wait(t2), np.flatnonzero(cats))
        bad = idx.copy()
        bad[5] = 5000                                       # out of range: reported, device memory-safe
        t3 = net.infer_submit(rp, bad)
        with pytest.raises(sd.SdnnError) as e:
            net.infer_wait(t3)
        assert e.value.status == sd.SDNN_E_FORMAT
        cg, _ = net.infer(rp, idx, None)                    # the handle is still usable
        assert np.array_equal(cg, np.flatnonzero(cats))


_T16 = {"SDNN_PASS_WIDE": "0"}     # 16-position k_pass tiles for 1024-row components


@pytest.mark.parametrize("env,flags", [({**_T16, "SDNN_PASS_VT": "1"}, 0), ({**_T16, "SDNN_PASS_TMA16": "1"}, 0),
                                       ({**_T16, "SDNN_BLK16": "1"}, 0), (_T16, 0), (_T16, 512),
                                       ({**_T16, "SDNN_PASS_PARITY": "1"}, 0), ({"SDNN_PASS_T32": "0"}, 0),
                                       ({"SDNN_PASS_T32": "2", "SDNN_PASS_T32_S": "2"}, 0), ({"SDNN_PASS_X2": "1"}, 0), ({"SDNN_PASS_X2": "0"}, 0), ({"SDNN_PASS_WIDE": "1"}, 0), ({"SDNN_PASS_GENERAL": "1", "SDNN_KNOB_NET": "rw"}, 0),
                                       ({"SDNN_KNOB_NET": "rw"}, 0),
                                       ({"SDNN_PASS_ORDER": "tile"}, 0), ({"SDNN_PASS_ORDER": "comp"}, 0),
                                       ({"SDNN_PASS_NB": "1", "SDNN_PASS_X2": "1"}, 0), ({}, 512)])
def test_opt_in_knobs(sd, env, flags):
    """The measured-off alternatives stay exact (each in a fresh process, since
    the library reads its knobs once): value tables, TMA tensor-map loads and
    16-position blocks for the 1024-row passes, tile-major order everywhere,
    single tile buffers with packed FFMA2, shared-value stores."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, os.path.join(here, "_knob_check.py"), str(flags)],
                         env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stderr[-2000:]
