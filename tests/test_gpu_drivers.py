"""The four drivers (reference layout.py:409-485) on BASELINE configs: the
kNN graph each driver feeds C1 is pinned to the reference's goldens, every
RunReport field is checked, and the opt-in deterministic SGD mode gives
bitwise-repeatable layouts (acceptance criterion 9, test_acceptance.py:276-300)."""

import numpy as np
import pytest

from conftest import load_golden, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_19703_b200 as gu
    return gu


@pytest.fixture
def captured(monkeypatch):
    """The DirectedKnn each driver hands to smooth_knn_weights."""
    from paper_2509_19703_b200 import layout as L
    seen = []
    real = L.smooth_knn_weights

    def spy(knn, k=None):
        seen.append(knn)
        return real(knn, k)

    monkeypatch.setattr(L, "smooth_knn_weights", spy)
    return seen


def _check_report(rep, tag, g, seed):
    assert rep.algorithm_tag == tag
    assert rep.n == g.n and rep.m == g.m and rep.seed == seed
    assert rep.c0_ms > 0 and rep.c1_ms > 0 and rep.c2_ms > 0
    assert rep.prep_ms == 0.0
    assert rep.total_ms == rep.c0_ms + rep.c1_ms + rep.c2_ms


def test_gumap_driver_c1(gu, captured):
    z = load_golden("c1.npz")
    g = gu.synth_graph("grid", 2500)
    cfg = gu.OptimizerConfig(iterations=20, k=15, seed=0)
    lay, rep = gu.run_gumap(g, cfg)
    (knn,) = captured
    assert np.array_equal(knn.indptr, z["knn_indptr"])
    assert np.array_equal(knn.dst, z["knn_dst"]) and np.array_equal(knn.dist, z["knn_dist"])
    _check_report(rep, "GUMAP", g, 0)
    assert lay.algorithm_tag == "GUMAP" and lay.coords.shape == (2500, 2)
    assert np.all(np.isfinite(lay.coords))


def test_ss_gumap_driver_c1_identity_sparsifier(gu, captured):
    """c1 is already sparser than n log2 n: G' = G, same kNN graph as GUMAP."""
    z = load_golden("c1.npz")
    g = gu.synth_graph("grid", 2500)
    lay, rep = gu.run_ss_gumap(g, gu.OptimizerConfig(iterations=10, k=15, seed=0))
    (knn,) = captured
    assert np.array_equal(knn.dst, z["knn_dst"]) and np.array_equal(knn.dist, z["knn_dist"])
    assert rep.algorithm_tag == "SS" and lay.algorithm_tag == "SS"
    assert rep.n == g.n and rep.m == g.m and rep.prep_ms >= 0.0


def test_sl_driver_c3(gu, captured):
    z = load_golden("c3.npz")
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    cfg = gu.OptimizerConfig(iterations=20, k=15, seed=2)
    lay, rep = gu.run_sl_gumap(g, cfg)
    (knn,) = captured
    assert sha(knn.indptr) == str(z["knn_indptr_sha"])
    assert sha(knn.dst) == str(z["knn_dst_sha"])
    assert sha(knn.dist) == str(z["knn_dist_sha"])
    _check_report(rep, "SL", g, 2)
    assert lay.algorithm_tag == "SL" and np.all(np.isfinite(lay.coords))


def test_gumap_c0_is_the_bfs(gu, monkeypatch):
    """C0 brackets the BFS (reference layout.py:418-420): the one fused
    BFS-kNN launch of run_gumap happens inside SparseDistanceSet.run_bfs,
    which the driver calls before it closes the C0 bracket."""
    import inspect

    from paper_2509_19703_b200 import neighbors as N
    callers = []
    real = N.full_knn_records

    def spy(*a, **kw):
        callers.append(inspect.stack()[1].function)
        return real(*a, **kw)

    monkeypatch.setattr(N, "full_knn_records", spy)
    g = gu.synth_graph("grid", 400)
    gu.run_gumap(g, gu.OptimizerConfig(iterations=1, k=15, seed=1))
    assert callers == ["run_bfs"]


@pytest.mark.parametrize("env", [False, True])
def test_deterministic_sgd_repeatable(gu, monkeypatch, env):
    """Criterion 9: repeat runs of every driver give bit-identical layouts
    when deterministic SGD is asked for (config field or environment)."""
    graphs = [gu.synth_graph("grid", 100, seed=4), gu.synth_graph("scale_free", 120, seed=4, m0=3)]
    if env:
        monkeypatch.setenv("GU_SGD_DETERMINISTIC", "1")
    for g in graphs:
        for fn in (gu.run_gumap, gu.run_ss_gumap, gu.run_sl_gumap, gu.run_sssl_gumap):
            cfg = gu.OptimizerConfig(iterations=50, k=6, seed=99, deterministic=not env)
            a, _ = fn(g, cfg)
            b, _ = fn(g, cfg)
            assert a.coords.tobytes() == b.coords.tobytes(), fn.__name__
            assert np.all(np.isfinite(a.coords))


def test_deterministic_sgd_quality_c1(gu):
    """The deterministic batches keep the layout quality of the default mode
    (NP of the c1 GUMAP layout within the reference's seed spread)."""
    from oracle.metrics import neighborhood_preservation

    z = load_golden("quality_c1.npz")
    g = gu.synth_graph("grid", 2500)
    dset = gu.all_pairs_bfs(g)
    vals = []
    for seed in range(4):
        gk = gu.smooth_knn_weights(gu.knn_from_full_distances(dset, 15, seed=seed))
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed, deterministic=True)
        lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0), cfg).coords
        vals.append(neighborhood_preservation(g, lay))
    ref = np.asarray(z["np_"])
    print("deterministic NP", np.mean(vals), "reference", ref.mean(), "+-", ref.std())
    assert np.mean(vals) >= ref.mean() - 3 * ref.std()
