"""build_graph / largest_connected_component against the live reference's
outputs (tests/golden/ingest.json, frozen by make_golden.py gen_ingest from
graph.py:132-232): label types (ints, strings, numeric strings, floats),
dropped self-loop / duplicate counts, components and the label tie rule of
graph.py:211-214.  The small cases run the host path here; the GPU module
runs the same cases plus a 200k-pair input through csrc/ingest.cu."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, sha

with open(os.path.join(GOLDEN, "ingest.json")) as f:
    GOLD = json.load(f)


def _same(g, exp):
    assert g.n == exp["n"] and g.m == exp["m"]
    assert np.array_equal(np.asarray(g.edges), np.asarray(exp["edges"], np.int64).reshape(-1, 2))
    assert list(g.labels) == exp["labels"]
    assert [type(x) for x in g.labels] == [type(x) for x in exp["labels"]]
    assert np.array_equal(np.asarray(g.adj_indptr), exp["indptr"])
    assert np.array_equal(np.asarray(g.adj_indices), exp["indices"])
    assert g.dropped_self_loops == exp["dropped_self_loops"]
    assert g.dropped_duplicates == exp["dropped_duplicates"]


def _tuples(pairs):
    return [tuple(p) for p in pairs]


def check_all(gu):
    for case in GOLD["cases"]:
        g = gu.build_graph(_tuples(case["pairs"]))
        _same(g, case["graph"])
        _same(gu.largest_connected_component(g), case["lcc"])
    t = GOLD["tie"]["graph"]
    from paper_2509_19703_b200.graph import graph_from_edges
    g = graph_from_edges(t["n"], np.asarray(t["edges"], np.int64), labels=tuple(t["labels"]))
    _same(gu.largest_connected_component(g), GOLD["tie"]["lcc"])


def test_ingest_host_vs_reference():
    import paper_2509_19703_b200 as gu
    from paper_2509_19703_b200 import graph as G
    orig = G._gpu_available
    G._gpu_available = lambda: False
    try:
        check_all(gu)
    finally:
        G._gpu_available = orig


@pytest.mark.gpu
def test_ingest_gpu_vs_reference():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_19703_b200 as gu
    check_all(gu)  # small builds stay on the host; every LCC runs on the GPU
    L = GOLD["large"]
    rng = np.random.default_rng(L["seed"])
    idv = rng.choice(2**40, size=L["nids"], replace=False)
    pairs = idv[rng.integers(0, L["nids"], size=(L["npairs"], 2))]
    g = gu.build_graph(pairs)  # >= 64k integer pairs: csrc/ingest.cu
    assert (g.n, g.m) == (L["n"], L["m"])
    assert g.dropped_self_loops == L["dropped_self_loops"]
    assert g.dropped_duplicates == L["dropped_duplicates"]
    assert sha(np.asarray(g.edges, np.int64)) == L["edges_sha"]
    assert sha(np.asarray(g.labels, np.int64)) == L["labels_sha"]
    h = gu.largest_connected_component(g)
    assert (h.n, h.m) == (L["lcc_n"], L["lcc_m"])
    assert sha(np.asarray(h.edges, np.int64)) == L["lcc_edges_sha"]
    assert sha(np.asarray(h.labels, np.int64)) == L["lcc_labels_sha"]
