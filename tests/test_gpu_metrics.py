"""GPU layout-quality metrics (csrc/metrics.cu) vs the
reference's own values on its own c1 layouts (tests/golden/quality_c1.npz)
and vs the oracle restatements (oracle/metrics.py, pinned to the reference)
on random graphs and layouts, degenerate ones included.

Tolerances: crossings exact; neighborhood preservation 1e-12 absolute (a
single differing rank moves it by >= 1/(n q), far above); stress 1e-12
relative (summation order only)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

NP_ABS_TOL = 1e-12
STRESS_REL_TOL = 1e-12


@pytest.fixture(scope="module")
def gu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_19703_b200 as gu
    return gu


def _layout(gu, coords):
    return gu.Layout(coords=np.asarray(coords, np.float64))


def test_metrics_on_reference_c1_layouts(gu):
    from paper_2509_19703_b200 import metrics as M

    z = load_golden("quality_c1.npz")
    g = gu.synth_graph("grid", 2500)
    for i, lay in enumerate((z["layout0"], z["layout1"])):
        L = _layout(gu, lay)
        assert abs(M.neighborhood_preservation(g, L) - z["np_"][i]) < NP_ABS_TOL
        s = M.stress(g, L)
        assert abs(s - z["stress"][i]) <= STRESS_REL_TOL * abs(z["stress"][i])
        assert M.count_crossings(g, L) == int(z["crossings"][i])


def _cases(gu):
    from paper_2509_19703_b200.fixtures import random_connected_graph
    from paper_2509_19703_b200.graph import graph_from_edges

    rng = np.random.default_rng(20261019)
    graphs = [gu.synth_graph("grid", 400), gu.synth_graph("scale_free", 600, seed=9, m0=2)]
    for _ in range(3):
        n, edges = random_connected_graph(rng, n_max=300)
        graphs.append(graph_from_edges(n, edges))
    for g in graphs:
        yield g, rng.uniform(-10, 10, size=(g.n, 2))
        # integer lattice: duplicate points, collinear and touching segments
        yield g, rng.integers(0, 6, size=(g.n, 2)).astype(np.float64)


def test_metrics_vs_oracle_random(gu, oracle):
    from oracle import metrics as OM
    from paper_2509_19703_b200 import metrics as M

    for g, coords in _cases(gu):
        L = _layout(gu, coords)
        hop = oracle.all_pairs_bfs(g, nthreads=4)
        for r in (1, 2, 3):
            a = M.neighborhood_preservation(g, L, r=r)
            b = OM.neighborhood_preservation(g, coords, hop.astype(np.float64), r=r)
            assert abs(a - b) < NP_ABS_TOL, (g.n, r, a, b)
        for rescale in (True, False):
            a = M.stress(g, L, rescale=rescale)
            b = OM.stress(g, coords, hop, rescale=rescale)
            assert abs(a - b) <= STRESS_REL_TOL * abs(b), (g.n, rescale, a, b)
        assert M.count_crossings(g, L) == OM.count_crossings(g, coords), g.n


def test_metrics_errors_and_small(gu):
    from paper_2509_19703_b200 import metrics as M
    from paper_2509_19703_b200.graph import graph_from_edges

    g = graph_from_edges(4, [(0, 1), (2, 3)])
    L = _layout(gu, np.arange(8, dtype=np.float64).reshape(4, 2))
    with pytest.raises(M.MetricError):
        M.stress(g, L)
    with pytest.raises(M.MetricError):
        M.neighborhood_preservation(g, _layout(gu, np.zeros((3, 2))))
    one = graph_from_edges(1, [])
    assert M.neighborhood_preservation(one, _layout(gu, np.zeros((1, 2)))) == 1.0
    assert M.stress(one, _layout(gu, np.zeros((1, 2)))) == 0.0
    assert M.count_crossings(g, L) == 0  # two disjoint parallel segments
    x = graph_from_edges(4, [(0, 1), (2, 3)])
    cross = _layout(gu, np.array([[0, 0], [2, 2], [0, 2], [2, 0]], np.float64))
    assert M.count_crossings(x, cross) == 1


def test_quality_c3_exact_vs_reference(gu):
    """Check (c) at SL scale with EXACT metrics on both sides: NP, stress and
    crossings of the GPU c3 SL layouts (GPU metrics) vs those of the
    reference's own c3 SL layouts (oracle metrics, tests/golden/
    quality_c3_full.npz); no worse than 4 standard errors."""
    import math

    from paper_2509_19703_b200 import metrics as M

    z = load_golden("quality_c3_full.npz")
    ref = np.stack([z["np_"], z["stress"], z["crossings"].astype(np.float64)], axis=1)
    if ref.shape[0] < 2:
        pytest.skip("reference fixture holds fewer than 2 seeds")
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    vals = []
    for seed in range(3):
        _, knn = gu.partial_bfs(g, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        E = gk.edge_count
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed,
                                 samp=math.log(0.1 * E) / math.log(E))
        lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0), cfg)
        vals.append((M.neighborhood_preservation(g, lay), M.stress(g, lay), M.count_crossings(g, lay)))
    v = np.array(vals, dtype=np.float64)
    print("check (c) c3 exact mean ratios gpu/ref [np, stress, crossings]:",
          v.mean(axis=0) / ref.mean(axis=0))
    se = ref.std(axis=0, ddof=1) / math.sqrt(ref.shape[0]) + v.std(axis=0, ddof=1) / math.sqrt(v.shape[0])
    assert v.mean(axis=0)[0] >= ref.mean(axis=0)[0] - 4 * se[0]
    assert v.mean(axis=0)[1] <= ref.mean(axis=0)[1] + 4 * se[1]
    assert v.mean(axis=0)[2] <= ref.mean(axis=0)[2] + 4 * se[2]


def test_np_sources_matches_sampled_estimator(gu, oracle):
    """neighborhood_preservation / stress (..., sources=S) are the oracle's
    sampled estimators (oracle/metrics.py): the reference's terms over the
    rows of S (stress: scale fitted on the same pairs)."""
    from oracle.metrics import sample_sources, sampled_neighborhood_preservation
    from paper_2509_19703_b200 import metrics as M

    z = load_golden("quality_c1.npz")
    g = gu.synth_graph("grid", 2500)
    src = sample_sources(g.n, size=400, seed=5)
    rows = oracle.all_pairs_bfs_rows(g, src)
    from oracle.metrics import sampled_stress

    for lay in (z["layout0"], np.random.default_rng(1).integers(0, 7, size=(g.n, 2)).astype(float)):
        a = M.neighborhood_preservation(g, _layout(gu, lay), sources=src)
        b = sampled_neighborhood_preservation(lay, rows, src)
        assert abs(a - b) < NP_ABS_TOL
        a = M.stress(g, _layout(gu, lay), sources=src)
        b = sampled_stress(lay, rows, src)
        assert abs(a - b) <= STRESS_REL_TOL * abs(b)


def test_quality_c4_sampled_vs_reference(gu):
    """Check (c) at 1M scale (c4 SBM): sampled NP / stress over the 2000
    fixed sources of the GPU layouts vs the reference's own c4 layouts
    (tests/golden/quality_c4.npz, same estimators); 4 standard errors."""
    import math
    import os

    from conftest import GOLDEN
    from paper_2509_19703_b200 import metrics as M

    if not os.path.exists(os.path.join(GOLDEN, "quality_c4.npz")):
        pytest.skip("c4 reference fixture not generated")
    z = load_golden("quality_c4.npz")
    ref = np.stack([z["np_"], z["stress"]], axis=1)
    src = z["sources"]
    g = gu.config_graph("c4")
    vals = []
    for seed in range(2):
        _, knn = gu.partial_bfs(g, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0),
                                  gu.OptimizerConfig(iterations=200, k=15, seed=seed))
        vals.append((M.neighborhood_preservation(g, lay, sources=src), M.stress(g, lay, sources=src)))
    v = np.array(vals)
    print("check (c) c4 sampled mean ratios gpu/ref [np, stress]:", v.mean(axis=0) / ref.mean(axis=0))
    se = ref.std(axis=0, ddof=1) / math.sqrt(ref.shape[0]) + v.std(axis=0, ddof=1) / math.sqrt(v.shape[0])
    assert v.mean(axis=0)[0] >= ref.mean(axis=0)[0] - 4 * se[0]
    assert v.mean(axis=0)[1] <= ref.mean(axis=0)[1] + 4 * se[1]


def test_quality_c2_exact_vs_reference(gu):
    """Check (c) at SS scale (c2: SS-GUMAP on the G' fixture, m = 1.09M) with
    exact metrics on both sides.  tests/golden/quality_c2.npz freezes the
    reference's own five final c2 layouts plus the oracle's NP / stress of
    them; the GPU metrics reproduce those values (the metric pin at n = 20k)
    and evaluate the crossings (~1.2e11 per layout, beyond a CPU pass).  The
    GPU c2 layouts must be no worse than 4 standard errors on each metric."""
    import math

    from paper_2509_19703_b200 import metrics as M

    z = load_golden("quality_c2.npz")
    g = gu.config_graph("c2")
    assert g.n == int(z["n"]) and g.m == int(z["m"])
    ref = []
    for i, coords in enumerate(z["layouts"][:3]):
        lay = _layout(gu, coords)
        a, b = M.neighborhood_preservation(g, lay), M.stress(g, lay)
        assert abs(a - z["np_"][i]) < NP_ABS_TOL
        assert abs(b - z["stress"][i]) <= STRESS_REL_TOL * abs(z["stress"][i])
        ref.append((a, b, M.count_crossings(g, lay)))
    dset = gu.all_pairs_bfs(g)
    vals = []
    for seed in range(3):
        knn = gu.knn_from_full_distances(dset, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0),
                               gu.OptimizerConfig(iterations=200, k=15, seed=seed), tag="SS")
        vals.append((M.neighborhood_preservation(g, lay), M.stress(g, lay), M.count_crossings(g, lay)))
    del dset
    v = np.array(vals, dtype=np.float64)
    ref = np.array(ref, dtype=np.float64)
    print("check (c) c2 exact mean ratios gpu/ref [np, stress, crossings]:",
          v.mean(axis=0) / ref.mean(axis=0))
    se = ref.std(axis=0, ddof=1) / math.sqrt(ref.shape[0]) + v.std(axis=0, ddof=1) / math.sqrt(v.shape[0])
    assert v.mean(axis=0)[0] >= ref.mean(axis=0)[0] - 4 * se[0]
    assert v.mean(axis=0)[1] <= ref.mean(axis=0)[1] + 4 * se[1]
    assert v.mean(axis=0)[2] <= ref.mean(axis=0)[2] + 4 * se[2]
