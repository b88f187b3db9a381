"""Algorithm 1 (Sec. 4.6.2 "Scheduling GPU Tasks", make_graph)
as the library runs it for the f1 task graphs (sdnn_flow_plan, host only):
levelize, id = index in the level, stream = id mod max_streams, events only on
cross-stream edges."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def sd():
    from paper_2004_10908_b200 import build
    build.build()
    import paper_2004_10908_b200 as sd
    return sd


def test_paper_example_two_streams(sd):
    """The worked example of Fig. fig::capturer: A and B get
    ids 0 and 1, C, D and E get 0, 1 and 2; with max_streams = 2 the only
    cross-stream dependencies are A->D and B->E, which need events."""
    A, B, C, D, E = range(5)
    edges = [(A, C), (A, D), (B, D), (B, E)]
    level, ids, stream, events = sd.flow_plan(5, edges, 2)
    assert level == [0, 0, 1, 1, 1]
    assert ids == [0, 1, 0, 1, 2]
    assert stream == [0, 1, 0, 1, 0]
    assert events == [(A, D), (B, E)]
    # one stream: no events at all; three streams (E moves to stream 2): still
    # exactly A->D and B->E
    assert sd.flow_plan(5, edges, 1)[3] == []
    assert sd.flow_plan(5, edges, 3)[2] == [0, 1, 0, 1, 2]
    assert sd.flow_plan(5, edges, 3)[3] == [(A, D), (B, E)]


@pytest.mark.parametrize("seed", range(6))
def test_random_dags_against_longest_path(sd, seed):
    r = np.random.default_rng(seed)
    n = int(r.integers(1, 60))
    edges = sorted({(int(u), int(v)) for u, v in r.integers(0, n, size=(3 * n, 2)) if u < v})
    k = int(r.integers(1, 6))
    level, ids, stream, events = sd.flow_plan(n, edges, k)
    # levels = longest path from a source (Kahn rounds), computed independently
    ref = [0] * n
    for v in range(n):                                   # edges go from lower to higher index
        ref[v] = max([ref[u] + 1 for u, w in edges if w == v], default=0)
    assert level == ref
    for lv in set(level):
        assert sorted(i for i, l in zip(ids, level) if l == lv) == list(range(level.count(lv)))
    assert stream == [i % k for i in ids]
    assert sorted(events) == sorted((u, v) for u, v in edges if stream[u] != stream[v])


def test_cycle_rejected(sd):
    with pytest.raises(sd.SdnnError) as e:
        sd.flow_plan(3, [(0, 1), (1, 2), (2, 0)], 2)
    assert e.value.status == sd.SDNN_E_FORMAT
