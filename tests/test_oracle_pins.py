"""Pins for the CPU oracle (oracle/) against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle -- a dropped term,
a wrong sign or index, a transposed W, a non-canonical summation order, an
unfused multiply-add, a wrong clamp, a missing bias -- fails at least one test:

* hand nets (tests/golden/hand_nets.{md,json}): literal matrices derived by
  hand from the north_star formula; H4 pins the ascending-k order, H5 the fused
  multiply-add, H1/H3 clip, death, negative weights, explicit zeros, padding,
  H2 positive-bias revival;
* dyadic brute force: float64 dense ``Y @ W`` on nets whose every partial sum is
  exactly representable in fp32, so the fp32 chain must equal it bit for bit;
* random fp32 nets: per-layer float64 evaluation within the fp32 chain's
  rounding-error bound (a transposed W or a dropped term is far outside it);
* layer 0 closed form: binary inputs and w = 1/16 give Z = count/16 exactly;
* KA known-answer family: block-diagonal nets whose groups evolve by a scalar
  recurrence evaluated here in numpy float32 (a different formulation);
* invariants I1-I6 of SURVEY.md 8.3 and sentinel rows on the RN/MS workload.
"""
import numpy as np
import pytest

import oracle
import sdnngen as g


def _run(net, skip_zero=True, nthreads=2):
    o = oracle.Oracle(net.n, net.y0_rowptr, net.y0_idx, net.y0_val)
    for lay in net.layers:
        o.layer(lay["rowptr"], lay["colidx"], lay["val"], 0.0, lay["bias"], ymax=net.ymax,
                skip_zero=skip_zero, nthreads=nthreads)
    return o


@pytest.mark.parametrize("name", ["H1", "H2", "H3", "H3_ymax2", "H4", "H5"])
@pytest.mark.parametrize("skip_zero", [True, False])
def test_hand_nets(hand_nets, name, skip_zero):
    net = hand_nets[name]
    o = _run(net, skip_zero)
    # bit-exact, including the sign of zero (canonical +0)
    assert o.Y.view(np.uint32).tolist() == net.expected_Y.view(np.uint32).tolist()
    assert np.flatnonzero(o.categories()).tolist() == net.expected_categories


def _dense_w(lay, n):
    W = np.zeros((n, n), np.float64)
    k = np.repeat(np.arange(n), np.diff(lay.rowptr))
    W[k, lay.colidx] = lay.uniform if lay.val is None else lay.val.astype(np.float64)
    return W


@pytest.mark.parametrize("seed", range(6))
def test_dyadic_bruteforce_exact(seed):
    """All intermediates dyadic with < 24 significant bits => fp32 chain == exact."""
    r = np.random.default_rng(seed)
    n = int(r.choice([8, 33, 96, 256]))
    L = int(r.integers(1, 4))
    spec = g.random_spec(n, L, seed=100 + seed, kmin=0, kmax=min(32, n), wdist="uniform")
    layers = list(g.iter_layers(spec))
    dyadic = r.random() < 0.5
    for l, lay in enumerate(layers):
        lay.bias = r.choice(np.float32([-0.25, -0.125, 0.0]), size=n).astype(np.float32)
        if dyadic:       # per-slot dyadic weights (both signs)
            lay.val = r.choice(np.float32([0.5, -0.5, 0.25, -0.25, 0.125, 0.0625]),
                               size=lay.colidx.size).astype(np.float32)
        else:            # uniform layer (val=None) with a per-layer dyadic value
            lay.uniform = float(r.choice([0.0625, 0.125, 0.1875, -0.0625]))
    B = 64
    Y0 = (r.random((B, n)) < 0.3).astype(np.float32)
    Y0[r.random((B, n)) < 0.1] = 2.0
    rp, idx, val = g.csr_from_dense(Y0)
    cats, Y, _ = oracle.infer(n, layers, rp, idx, val, nthreads=2)
    Y64 = Y0.astype(np.float64)
    for lay in layers:
        Y64 = np.clip(Y64 @ _dense_w(lay, n) + lay.bias.astype(np.float64), 0.0, 32.0)
    assert np.array_equal(Y.astype(np.float64), Y64)
    assert np.array_equal(cats, (Y64 > 0).any(1))


@pytest.mark.parametrize("seed", range(4))
def test_random_fp32_within_rounding_bound(seed):
    """Random fp32 values: each oracle layer equals the exact (float64) layer of
    its own fp32 input within the fp32 chain's error bound gamma_{K+1}*sum|terms|."""
    n, L, B = 128, 6, 48
    spec = g.random_spec(n, L, seed=200 + seed, kmin=8, kmax=32)
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, B, seed=300 + seed)
    o = oracle.Oracle(n, rp, idx, val)
    for lay in layers:
        Yin = o.Y.astype(np.float64)
        o.apply(lay, nthreads=2)
        W = _dense_w(lay, n)
        exact = np.clip(Yin @ W + lay.bias, 0.0, 32.0)
        mag = np.abs(Yin) @ np.abs(W) + np.abs(lay.bias)
        K = int(np.diff(lay.rowptr).max(initial=0)) + 2
        bound = 1.01 * K * 2.0 ** -24 * mag / (1 - K * 2.0 ** -24) + 1e-30
        err = np.abs(o.Y.astype(np.float64) - exact)
        assert (err <= bound).all(), (err - bound).max()
        # a transposed W would be far outside the bound
        if n > 1 and np.abs(Yin @ W.T - Yin @ W).max() > 1e-3:
            assert np.abs(np.clip(Yin @ W.T + lay.bias, 0, 32) - o.Y).max() > bound.max()


def test_layer0_closed_form_binary_uniform():
    """Binary Y0, w = 1/16: partial sums t/16 are exact, so Y1 = clamp(count/16 + b)."""
    n, B = 1024, 300
    spec = g.rn_spec(n, 1)
    lay = g.gen_layer(spec, 0)
    rp, idx = g.ms_inputs(n, B, seed=5)
    Y0 = g.dense_from_csr(rp, idx, None, n).astype(np.int64)
    A = np.zeros((n, n), np.int64)
    A[np.repeat(np.arange(n), 32), lay.colidx] = 1
    count = Y0 @ A                                             # integer counts
    z = (count.astype(np.float32) / np.float32(16)) + lay.bias   # one fp32 add
    expected = np.where(z > 0, np.minimum(z, np.float32(32)), np.float32(0)).astype(np.float32)
    o = oracle.Oracle(n, rp, idx, None)
    o.apply(lay, nthreads=2)
    assert np.array_equal(o.Y.view(np.uint32), expected.view(np.uint32))


# ----------------------------------------------------------------- KA family

def ka_scalar_trajectory(count: int, b: float, L: int) -> np.ndarray:
    """Value of a 32-neuron KA group after each layer, from the group's input
    count, by the scalar recurrence (numpy float32 arithmetic):
    layer 0: acc = count * (1/16) (exact), y = clamp(acc + b);
    layer l>0: acc = 32 sequential float32 adds of y/16, y = clamp(acc + b)."""
    f = np.float32
    b = f(b)
    out = np.zeros(L, np.float32)
    y = f(0)
    for l in range(L):
        if l == 0:
            acc = f(count) / f(16)
        else:
            acc = f(0)
            t = y / f(16)
            for _ in range(32):
                acc = f(acc + t)
        z = f(acc + b)
        y = f(min(z, f(32))) if z > 0 else f(0)
        out[l] = y
    return out


@pytest.mark.parametrize("n,bias,thr", [(1024, -0.30, 10), (4096, -0.35, 12),
                                        (16384, -0.40, 13), (65536, -0.45, 15)])
def test_ka_thresholds(n, bias, thr):
    """a KA group survives iff its input count >= 10/12/13/15."""
    fates = [ka_scalar_trajectory(c, bias, 40)[-1] > 0 for c in range(33)]
    assert fates == [c >= thr for c in range(33)]
    # survivors saturate at exactly 32 within 13 layers; the dead reach 0
    for c in range(33):
        tr = ka_scalar_trajectory(c, bias, 40)
        assert tr[13] in (0.0, 32.0)


def ka_expected(spec, cnt):
    """Exact Y_L for KA inputs with per-group counts cnt[B, G]."""
    n, L = spec.n, spec.L
    G = n // 32
    # lineage: input group (boundary 0) -> output group at boundary L (internal ids)
    grp = np.arange(G)
    for l in range(L):
        beta = g._rng(spec.seed, 2, l).permutation(G)   # output group h reads input group beta[h]
        inv = np.empty(G, np.int64)
        inv[beta] = np.arange(G)
        grp = inv[grp]
    piL = g._perm(spec, L)
    traj = {c: ka_scalar_trajectory(c, spec.bias, L)[-1] for c in range(33)}
    Y = np.zeros((cnt.shape[0], n), np.float32)
    for g0 in range(G):
        cols = piL[grp[g0] * 32 + np.arange(32)]
        vals = np.array([traj[int(c)] for c in cnt[:, g0]], np.float32)
        Y[:, cols] = vals[:, None]
    return Y


@pytest.mark.parametrize("n,L", [(1024, 24), (2048, 17)])
def test_ka_known_answer(n, L):
    spec = g.ka_spec(n, L)
    rp, idx, cnt = g.ka_inputs(n, 256, seed=11)
    cats, Y, _ = oracle.infer(n, g.iter_layers(spec), rp, idx, None, nthreads=2)
    Yx = ka_expected(spec, cnt)
    assert np.array_equal(Y.view(np.uint32), Yx.view(np.uint32))
    assert np.array_equal(cats, (Yx > 0).any(1))
    assert 0 < cats.sum() < cats.size


# ----------------------------------------------------- invariants on RN / MS

@pytest.fixture(scope="module")
def rn_run():
    n, L, B = 1024, 40, 1000
    spec = g.rn_spec(n, L)
    layers = list(g.iter_layers(spec))
    rp, idx = g.ms_inputs(n, B)
    o = oracle.Oracle(n, rp, idx, None)
    hist = [o.Y.copy()]
    for lay in layers:
        o.apply(lay, nthreads=4)
        hist.append(o.Y.copy())
    return spec, layers, rp, idx, hist, o.categories()


def test_invariants_bounds_and_monotone_death(rn_run):
    spec, layers, rp, idx, hist, cats = rn_run
    live_prev = None
    for l, Y in enumerate(hist[1:]):
        assert Y.min() >= 0.0 and Y.max() <= 32.0                      # I1
        assert not np.signbit(Y).any()                                  # canonical +0
        live = (Y != 0).any(1)
        if live_prev is not None:
            assert not (live & ~live_prev).any()                        # I2 monotone death
            assert live.sum() <= live_prev.sum()                        # I6
        live_prev = live
    assert np.array_equal(cats, (hist[-1] > 0).any(1))


def test_invariants_sentinels_and_empty_rows(rn_run):
    spec, layers, rp, idx, hist, cats = rn_run
    i = np.arange(cats.size)
    assert cats[i % 1000 == 999].all()                                 # all-ones row survives
    empty = np.diff(rp) == 0
    assert empty[i % 1000 == 998].all()
    assert not cats[empty].any()                                        # I3
    assert 0 < cats.sum() < cats.size


def test_invariant_row_independence_and_permutation(rn_run):
    spec, layers, rp, idx, hist, cats = rn_run
    rows = np.random.default_rng(3).choice(cats.size, 97, replace=False)
    srp, sidx, _ = oracle.subset_rows(rp, idx, None, rows)
    c2, Y2, _ = oracle.infer(spec.n, layers, srp, sidx, None, nthreads=3)
    assert np.array_equal(Y2.view(np.uint32), hist[-1][rows].view(np.uint32))   # I4
    assert np.array_equal(c2, cats[rows])                                          # I5


def test_skip_zero_is_exact(rn_run):
    spec, layers, rp, idx, hist, cats = rn_run
    rows = np.arange(0, 1000, 37)
    srp, sidx, _ = oracle.subset_rows(rp, idx, None, rows)
    _, Ya, _ = oracle.infer(spec.n, layers[:12], srp, sidx, None, skip_zero=False)
    _, Yb, _ = oracle.infer(spec.n, layers[:12], srp, sidx, None, skip_zero=True)
    assert np.array_equal(Ya.view(np.uint32), Yb.view(np.uint32))
    assert np.array_equal(Ya.view(np.uint32), hist[12][rows].view(np.uint32))


def test_thread_count_does_not_change_results():
    n = 256
    spec = g.random_spec(n, 3, seed=9, kmin=4, kmax=32)
    layers = list(g.iter_layers(spec))
    rp, idx, val = g.random_inputs(n, 33, seed=9)
    _, Y1, _ = oracle.infer(n, layers, rp, idx, val, nthreads=1)
    _, Y7, _ = oracle.infer(n, layers, rp, idx, val, nthreads=7)
    assert np.array_equal(Y1.view(np.uint32), Y7.view(np.uint32))


def test_zero_layers_and_empty_batch():
    n = 8
    rp = np.array([0, 2, 2, 3], np.int64)
    idx = np.array([1, 3, 0], np.int32)
    val = np.array([0.5, -1.0, -2.0], np.float32)
    cats, Y, _ = oracle.infer(n, [], rp, idx, val)
    assert cats.tolist() == [True, False, False]           # only positive entries count
    cats, Y, _ = oracle.infer(n, [], np.zeros(1, np.int64), np.zeros(0, np.int32), None)
    assert cats.size == 0 and Y.shape == (0, n)


# ------------------------------------------------ survivor profile (live rows)
# oracle_live_rows counts rows with at least one nonzero entry; the GPU tests
# compare the library's per-layer survivor profile against it, so it is pinned
# here on its own: a hand-counted matrix and the KA closed form per layer.

def test_live_rows_hand_count():
    """Rows (n = 4): empty | explicit +0.0 | -0.0 | denormal 2^-149 | -3 |
    all 32 | +0.5 in the last column | +0.0 and -0.0 together.  By hand: rows
    3, 4, 5, 6 are nonzero (a -0.0 entry is zero), so the count is 4."""
    tiny = float.fromhex("0x1p-149")
    rows = [[], [(1, 0.0)], [(2, -0.0)], [(0, tiny)], [(3, -3.0)],
            [(0, 32.0), (1, 32.0), (2, 32.0), (3, 32.0)], [(3, 0.5)], [(0, 0.0), (3, -0.0)]]
    rp = np.zeros(len(rows) + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    idx = np.array([k for r in rows for k, _ in r], np.int32)
    val = np.array([v for r in rows for _, v in r], np.float32)
    o = oracle.Oracle(4, rp, idx, val)
    assert o.live_rows() == 4
    cats = o.categories()                     # categories need a POSITIVE entry (reading A7)
    assert cats.tolist() == [False, False, False, True, False, True, True, False]


@pytest.mark.parametrize("n,L,seed", [(1024, 20, 11), (2048, 17, 5)])
def test_live_rows_ka_profile(n, L, seed):
    """KA closed form per layer: after layer l a row is live iff one of its
    groups has a nonzero scalar trajectory value at l (groups are independent
    and uniform after layer 0)."""
    spec = g.ka_spec(n, L)
    rp, idx, cnt = g.ka_inputs(n, 300, seed=seed)
    _, _, prof = oracle.infer(n, g.iter_layers(spec), rp, idx, None, nthreads=2, profile=True)
    traj = np.stack([ka_scalar_trajectory(c, spec.bias, L) for c in range(33)])   # [count, layer]
    want = [int((traj[cnt, l] > 0).any(1).sum()) for l in range(L)]
    assert prof == want
    assert want[0] > want[-1] > 0


def test_live_rows_hand_nets(hand_nets):
    """The last entry of the profile of every golden hand net equals the number
    of nonzero rows of its hand-derived Y_L."""
    for net in hand_nets.values():
        o = oracle.Oracle(net.n, net.y0_rowptr, net.y0_idx, net.y0_val)
        for lay in net.layers:
            o.layer(lay["rowptr"], lay["colidx"], lay["val"], 0.0, lay["bias"], ymax=net.ymax)
        assert o.live_rows() == int((net.expected_Y != 0).any(1).sum()), net.name
