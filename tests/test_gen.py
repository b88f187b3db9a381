"""Generator (sdnngen) structure tests: regularity, group structure, sentinels,
determinism, and golden structure hashes (drift detector)."""
import json
import os

import numpy as np
import pytest

import sdnngen as g

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "gen_hashes.json")


@pytest.mark.parametrize("kind,n", [("rn", 1024), ("rn", 4096), ("rr", 1024), ("ka", 2048)])
def test_regular_32_in_32_out(kind, n):
    spec = {"rn": g.rn_spec, "rr": g.rr_spec, "ka": g.ka_spec}[kind](n, 6)
    for lay in g.iter_layers(spec):
        src = np.sort(lay.ell, 1)
        assert src.shape == (n, 32) and (src >= 0).all() and (src < n).all()
        assert (np.diff(src, axis=1) > 0).all()                    # 32 distinct sources
        assert (np.diff(lay.rowptr) == 32).all()                    # 32 out-edges per input
        # CSR and ELL describe the same edge set
        e_csr = np.repeat(np.arange(n), 32) * n + lay.colidx
        e_ell = lay.ell.reshape(-1).astype(np.int64) * n + np.repeat(np.arange(n), 32)
        assert np.array_equal(np.sort(e_csr), np.sort(e_ell))


def _groups(lay):
    keys = {}
    for j, s in enumerate(np.sort(lay.ell, 1)):
        keys.setdefault(s.tobytes(), []).append(j)
    return keys


def test_rn_is_dense_32x32_blocks():
    n = 1024
    for lay in g.iter_layers(g.rn_spec(n, 4)):
        grp = _groups(lay)
        assert len(grp) == n // 32 and all(len(v) == 32 for v in grp.values())
        # the 32 source sets partition the inputs
        allsrc = np.concatenate([np.frombuffer(k, np.int32) for k in grp])
        assert np.array_equal(np.sort(allsrc), np.arange(n))


def test_rr_has_no_shared_source_sets():
    lay = g.gen_layer(g.rr_spec(1024, 3), 1)
    assert len(_groups(lay)) == 1024


def test_rn_relabelling_is_consistent():
    """Layer l's outputs and layer l+1's inputs use the same labels: composing
    two layers equals composing the unrelabelled butterflies (pi cancels)."""
    n, spec = 256, g.rn_spec(256, 3)
    l0, l1 = g.gen_layer(spec, 0), g.gen_layer(spec, 1)
    A0 = np.zeros((n, n), int); A0[np.repeat(np.arange(n), 32), l0.colidx] = 1
    A1 = np.zeros((n, n), int); A1[np.repeat(np.arange(n), 32), l1.colidx] = 1
    # plain butterflies on internal ids
    def bfly(l):
        B = np.zeros((n, n), int)
        m = np.arange(n)
        B[np.repeat(m, 32), g._rn_sets(n, l, m).reshape(-1)] = 1
        return B
    P = lambda p: np.eye(n, dtype=int)[p]         # P[i, p[i]] = 1
    pi1, pi2 = g._perm(spec, 1), g._perm(spec, 2)
    # A0 = B0 relabelled on outputs by pi1; A1 = pi1 on inputs, pi2 on outputs
    assert np.array_equal(A0, bfly(0) @ P(pi1))
    assert np.array_equal(A1, P(pi1).T @ bfly(1) @ P(pi2))
    assert np.array_equal(A0 @ A1, bfly(0) @ bfly(1) @ P(pi2))       # pi1 cancels


def test_ms_inputs_shape_density_sentinels():
    for n in (1024, 4096):
        rp, idx = g.ms_inputs(n, 2000)
        dens = idx.size / (2000 * n)
        assert 0.08 < dens < 0.2, dens
        i = np.arange(2000)
        assert (np.diff(rp)[i % 1000 == 999] == n).all()
        assert (np.diff(rp)[i % 1000 == 998] == 0).all()
        for r in range(0, 2000, 97):                               # sorted, in range
            row = idx[rp[r]:rp[r + 1]]
            assert (np.diff(row) > 0).all() and (row < n).all()


def test_ms_chunking_is_deterministic():
    a = g.ms_inputs(1024, 700, chunk=2048)
    b = g.ms_inputs(1024, 700, chunk=2048)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_ka_inputs_counts():
    rp, idx, cnt = g.ka_inputs(1024, 50, seed=1)
    dense = g.dense_from_csr(rp, idx, None, 1024).reshape(50, 32, 32)
    assert np.array_equal(dense.sum(-1).astype(int), cnt)


SPECS = {
    "rn_1024_120": lambda: g.rn_spec(1024, 120),
    "rr_1024_8": lambda: g.rr_spec(1024, 8),
    "ka_2048_8": lambda: g.ka_spec(2048, 8),
    "irr_300_3_s7": lambda: g.random_spec(300, 3, seed=7),
}


def test_structure_hashes_golden():
    """Hashes written once by tests/golden/make_gen_hashes.py; a change means the
    workload changed and every recorded number must be re-derived."""
    want = json.load(open(GOLDEN))
    for name, mk in SPECS.items():
        assert g.structure_hash(mk()) == want[name], name
    rp, idx = g.ms_inputs(1024, 1000)
    import hashlib
    h = hashlib.sha256(rp.tobytes() + idx.tobytes()).hexdigest()
    assert h == want["ms_1024_1000"]
