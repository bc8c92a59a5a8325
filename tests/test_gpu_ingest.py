"""GPU graph construction and LCC extraction (
graph.py:114-232) against the host restatement (itself CPU-tested in
test_host.py): identical arrays, labels and drop counts."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_19703_b200 as gu
    return gu


def _same(a, b):
    assert a.n == b.n and a.m == b.m
    assert np.array_equal(a.adj_indptr, b.adj_indptr)
    assert np.array_equal(a.adj_indices, b.adj_indices)
    assert np.array_equal(a.edges, b.edges)
    assert tuple(a.labels) == tuple(b.labels)
    assert a.dropped_self_loops == b.dropped_self_loops
    assert a.dropped_duplicates == b.dropped_duplicates


def test_build_graph_gpu_vs_host(gu, monkeypatch):
    from paper_2509_19703_b200 import graph as G

    rng = np.random.default_rng(7)
    for npairs, idmax in ((100, 50), (70000, 30000), (300000, 5_000_000_000)):
        ids = rng.integers(0, idmax, size=npairs * 2)
        pairs = ids.reshape(-1, 2)
        pairs[: npairs // 50, 1] = pairs[: npairs // 50, 0]        # self loops
        pairs[npairs // 2: npairs // 2 + npairs // 20] = pairs[: npairs // 20][:, ::-1]  # dups
        monkeypatch.setattr(G, "GPU_BUILD_MIN_PAIRS", 1 << 60)
        host = G.build_graph(pairs)
        monkeypatch.setattr(G, "GPU_BUILD_MIN_PAIRS", 1)
        dev = G.build_graph(pairs)
        _same(dev, host)
        # the resident CSR the GPU build registered feeds the BFS directly
        _, k1 = gu.partial_bfs(dev, 5, seed=1)
        _, k2 = gu.partial_bfs(host, 5, seed=1)
        assert np.array_equal(k1.dst, k2.dst) and np.array_equal(k1.dist, k2.dist)
    with pytest.raises(G.GraphError):
        G.build_graph(np.array([[3, 3], [4, 4]]))


def test_build_graph_string_labels(gu):
    g = gu.build_graph([("b", "a"), ("a", "c"), ("c", "c"), ("a", "b")])
    assert g.labels == ("a", "b", "c") and g.m == 2
    assert g.dropped_self_loops == 1 and g.dropped_duplicates == 1


def test_lcc_gpu_vs_host(gu, monkeypatch):
    from paper_2509_19703_b200 import graph as G

    rng = np.random.default_rng(11)
    cases = []
    # several components, the two largest tied in size
    e = [(i, i + 1) for i in range(0, 9)] + [(i, i + 1) for i in range(20, 29)] + [(40, 41)]
    cases.append(G.build_graph(np.array(e)))
    n = 50000
    pairs = rng.integers(0, n, size=(30000, 2))
    cases.append(G.build_graph(pairs))
    cases.append(gu.synth_graph("grid", 400))  # connected: identity
    for g in cases:
        monkeypatch.setattr(G, "_gpu_available", lambda: False)
        host = G.largest_connected_component(g)
        monkeypatch.setattr(G, "_gpu_available", lambda: True)
        dev = G.largest_connected_component(g)
        if host is g:
            assert dev is g
        else:
            _same(dev, host)
