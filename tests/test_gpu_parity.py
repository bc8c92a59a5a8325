"""GPU parity: libgumap (through the C ABI / drop-in API) vs golden vectors and
the oracle.  Bit-exact for all integer / index work and for rho / sigma; the
fuzzy weights within 4 ulp (device exp vs numpy's SIMD exp); the float64
replay within 1e-5 relative (north-star check (b), max(|x|, 1) denominator).
"""

import math
import warnings

import numpy as np
import pytest

from conftest import golden_graphs, load_golden, sha, split

pytestmark = pytest.mark.gpu

# tolerances written down where they are used
WEIGHT_ULPS = 4          # device exp vs numpy exp, per weight
REPLAY_REL_TOL = 1e-5    # north star check (b)


@pytest.fixture(scope="module")
def gu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_19703_b200 as gu
    return gu


def _ulps(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a.view(np.int64) - b.view(np.int64))


# ------------------------------------------------------------- C0 partial
def test_partial_bfs_golden_small(gu):
    for g, k, seed, exp in golden_graphs("partial_small.npz"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            dset, knn = gu.partial_bfs(g, k, seed=seed)
        assert np.array_equal(knn.indptr, exp["indptr"])
        assert np.array_equal(knn.dst, exp["dst"])
        assert np.array_equal(knn.dist, exp["dist"])
        assert np.array_equal(dset.nbr, exp["dst"])


def test_partial_bfs_warns_small_component(gu):
    g = gu.build_graph([(0, 1), (1, 2), (3, 4)])
    with pytest.warns(UserWarning, match="smaller than k"):
        dset, _ = gu.partial_bfs(g, k=3, seed=0)
    ids, _ = dset.row(3)
    assert list(ids) == [4]


def test_partial_bfs_rejects_bad_k(gu):
    g = gu.build_graph([(0, 1)])
    with pytest.raises(ValueError):
        gu.partial_bfs(g, 0)


def test_partial_bfs_c3_bitexact(gu):
    z = load_golden("c3.npz")
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    _, knn = gu.partial_bfs(g, 15, seed=2)
    assert sha(knn.indptr) == str(z["knn_indptr_sha"])
    assert sha(knn.dst) == str(z["knn_dst_sha"])
    assert sha(knn.dist) == str(z["knn_dist_sha"])


def test_partial_bfs_all_tiers_and_large_k(gu, oracle):
    """k > 32 (tier 2 only) and hub-heavy balls (tier 1b / 2) vs the oracle."""
    g = gu.synth_graph("scale_free", 3000, seed=5, m0=2)
    for k in (1, 3, 15, 32, 40, 100):
        _, knn = gu.partial_bfs(g, k, seed=11)
        ip, dst, dist = oracle.partial_bfs(g, k, seed=11, nthreads=4)
        assert np.array_equal(knn.indptr, ip) and np.array_equal(knn.dst, dst)
        assert np.array_equal(knn.dist, dist)


# c3 / c4 / c5 every row: tests/test_gpu_fullsize.py


# --------------------------------------------------------------- C0 full
def test_full_knn_golden_small(gu):
    for g, k, seed, exp in golden_graphs("full_small.npz"):
        dset = gu.all_pairs_bfs(g)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            knn = gu.knn_from_full_distances(dset, k, seed=seed)
        assert np.array_equal(knn.indptr, exp["indptr"])
        assert np.array_equal(knn.dst, exp["dst"])
        assert np.array_equal(knn.dist, exp["dist"])
        assert sha(dset.matrix) == exp["apsp_sha"]
        # explicit-matrix path (a set that carries its matrix)
        explicit = gu.SparseDistanceSet(n=g.n, full=True, matrix=np.array(dset.matrix))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            knn2 = gu.knn_from_full_distances(explicit, k, seed=seed)
        assert np.array_equal(knn2.dst, exp["dst"]) and np.array_equal(knn2.dist, exp["dist"])


def test_c1_full_path_bitexact(gu):
    z = load_golden("c1.npz")
    g = gu.synth_graph("grid", 2500)
    dset = gu.all_pairs_bfs(g)
    knn = gu.knn_from_full_distances(dset, 15, seed=0)
    assert np.array_equal(knn.indptr, z["knn_indptr"])
    assert np.array_equal(knn.dst, z["knn_dst"])
    assert np.array_equal(knn.dist, z["knn_dist"])
    knn7 = gu.knn_from_full_distances(dset, 5, seed=7)
    assert np.array_equal(knn7.dst, z["knn7_dst"]) and np.array_equal(knn7.dist, z["knn7_dist"])
    assert sha(dset.matrix) == str(z["apsp_sha"])


# c2 every row: tests/test_gpu_fullsize.py


# --------------------------------------------------------------------- C1
def test_smooth_cases_golden(gu):
    z = load_golden("smooth_cases.npz")
    for i in range(z["n"].shape[0]):
        n, k = int(z["n"][i]), int(z["k"][i])
        knn = gu.DirectedKnn(n=n, k=k, indptr=split(z["indptr"], z["indptr_off"], i),
                             dst=split(z["dst"], z["dst_off"], i),
                             dist=split(z["dist"], z["dist_off"], i))
        gk = gu.smooth_knn_weights(knn)
        assert np.array_equal(gk.rho, split(z["rho"], z["rho_off"], i))
        assert np.array_equal(gk.sigma, split(z["sigma"], z["sigma_off"], i))
        assert np.array_equal(gk.sym_src, split(z["sym_src"], z["sym_src_off"], i))
        assert np.array_equal(gk.sym_dst, split(z["sym_dst"], z["sym_dst_off"], i))
        assert _ulps(gk.sym_w, split(z["sym_w"], z["sym_w_off"], i)).max(initial=0) <= WEIGHT_ULPS
        assert np.array_equal(gk.nbr_indptr, split(z["nbr_indptr"], z["nbr_indptr_off"], i))


def test_smooth_memo_profiles_vs_oracle(gu, oracle):
    """The memoised-sigma path (n >= 4096): rows keyed by run-length profile,
    rows that do not fit a key (> 4 runs, distance > 255, run > 63 long) and
    short rows, mixed in one call -- rho / sigma bit-exact, weights and the
    union as in the oracle."""
    rng = np.random.default_rng(11)
    n, k = 6000, 15
    rows_d, rows_j = [], []
    for v in range(n):
        kind = v % 5
        if kind == 0:    # the common kNN shape: two hop levels, full row
            t0 = int(rng.integers(1, k))
            d = [1] * t0 + [2] * (k - t0)
        elif kind == 1:  # short row, three levels
            c = int(rng.integers(1, k))
            d = sorted(int(x) for x in rng.integers(1, 4, size=c))
        elif kind == 2:  # > 4 runs: solved directly
            d = sorted(int(x) for x in rng.integers(1, 9, size=k))
        elif kind == 3:  # large distances (> 255): solved directly
            d = sorted(int(x) for x in rng.integers(200, 400, size=k))
        else:            # all equal (sigma clamps to 1e3)
            d = [3] * k
        ids = rng.choice(np.setdiff1d(np.arange(n), [v]), size=len(d), replace=False)
        # rows sorted by (distance, id), as the kNN producers emit them
        order = np.lexsort((ids, np.array(d)))
        rows_d.append(np.array(d, dtype=np.int32)[order])
        rows_j.append(ids[order].astype(np.int32))
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows_d])
    dist = np.concatenate(rows_d)
    dst = np.concatenate(rows_j)
    knn = gu.DirectedKnn(n=n, k=k, indptr=indptr, dst=dst, dist=dist)
    gk = gu.smooth_knn_weights(knn)
    o = oracle.smooth_knn_weights(n, indptr, dst, dist, k)
    assert np.array_equal(gk.rho, o["rho"]) and np.array_equal(gk.sigma, o["sigma"])
    assert np.array_equal(gk.sym_src, o["sym_src"]) and np.array_equal(gk.sym_dst, o["sym_dst"])
    assert _ulps(gk.sym_w, o["sym_w"]).max(initial=0) <= WEIGHT_ULPS


def test_smooth_memo_table_overflow_vs_oracle(gu, oracle):
    """More distinct distance profiles than the 8192-entry table: rows that
    find it full are solved directly -- still bit-exact."""
    rng = np.random.default_rng(12)
    n, k = 20000, 15
    rows_d = []
    for v in range(n):
        cuts = np.sort(rng.choice(np.arange(1, k), size=3, replace=False))
        levels = np.sort(rng.choice(np.arange(1, 250), size=4, replace=False))
        d = np.repeat(levels, np.diff(np.concatenate([[0], cuts, [k]])))
        rows_d.append(d.astype(np.int32))
    dist = np.concatenate(rows_d)
    dst = np.concatenate([rng.choice(np.setdiff1d(np.arange(n), [v]), size=k, replace=False)
                          for v in range(n)]).astype(np.int32)
    # rows sorted by (distance, id)
    for v in range(n):
        sl = slice(v * k, (v + 1) * k)
        o = np.lexsort((dst[sl], dist[sl]))
        dst[sl], dist[sl] = dst[sl][o], dist[sl][o]
    indptr = (k * np.arange(n + 1)).astype(np.int64)
    gk = gu.smooth_knn_weights(gu.DirectedKnn(n=n, k=k, indptr=indptr, dst=dst, dist=dist))
    rho, sigma = oracle.smooth_rho_sigma(indptr, dist, k)
    assert np.array_equal(gk.rho, rho) and np.array_equal(gk.sigma, sigma)


def test_smooth_rejects_empty_row(gu):
    knn = gu.DirectedKnn(n=2, k=1, indptr=np.array([0, 1, 1]), dst=np.array([1], np.int32),
                         dist=np.array([1], np.int32))
    with pytest.raises(ValueError):
        gu.smooth_knn_weights(knn)


def test_c1_smooth_golden(gu):
    z = load_golden("c1.npz")
    knn = gu.DirectedKnn(n=2500, k=15, indptr=z["knn_indptr"], dst=z["knn_dst"],
                         dist=z["knn_dist"])
    gk = gu.smooth_knn_weights(knn)
    for key in ("rho", "sigma", "sym_src", "sym_dst", "nbr_indptr", "nbr_indices"):
        assert np.array_equal(getattr(gk, key), z[key]), key
    assert _ulps(gk.sym_w, z["sym_w"]).max() <= WEIGHT_ULPS


def test_c3_smooth_golden(gu):
    z = load_golden("c3.npz")
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    _, knn = gu.partial_bfs(g, 15, seed=2)
    gk = gu.smooth_knn_weights(knn)
    assert sha(gk.rho) == str(z["rho_sha"])
    assert sha(gk.sigma) == str(z["sigma_sha"])
    assert sha(gk.sym_src) == str(z["sym_src_sha"])
    assert sha(gk.sym_dst) == str(z["sym_dst_sha"])
    assert gk.edge_count == int(z["E"])
    assert _ulps(gk.sym_w[:20000], z["sym_w_head"]).max() <= WEIGHT_ULPS


# -------------------------------------------------------- C2 check (b)
def _rel_err(x, ref):
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1.0)))


def test_replay_c1_full_epochs(gu, oracle):
    z = load_golden("c1.npz")
    a, b = float(z["a"]), float(z["b"])
    gk = gu.KnnGraph(n=2500, k=15, directed=None, rho=z["rho"], sigma=z["sigma"],
                     sym_src=z["sym_src"], sym_dst=z["sym_dst"], sym_w=z["sym_w"],
                     nbr_indptr=z["nbr_indptr"], nbr_indices=z["nbr_indices"])
    c = np.array(z["init"], copy=True)
    state = 0 ^ oracle.SPLIT_GAMMA
    for it, key in ((0, "after1"), (1, "after2")):
        order = z["order%d" % it]
        before = c.copy()
        lr = 1.0 - it / 200
        state, negs, th = oracle.sgd_sweep(c, z["sym_src"], z["sym_dst"], z["sym_w"], order,
                                           z["nbr_indptr"], z["nbr_indices"], a, b, lr, 5, state)
        out, nwaves = gu.sgd_replay(gk, before, order, negs, th, a, b, lr, 5)
        assert nwaves > 1
        assert _rel_err(out, z[key]) <= REPLAY_REL_TOL
        c = np.array(z[key], copy=True)


def test_replay_c3_window_epoch(gu, oracle):
    z = load_golden("c3.npz")
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    ip, dst, dist = oracle.partial_bfs(g, 15, seed=2, nthreads=8)
    o = oracle.smooth_knn_weights(g.n, ip, dst, dist, 15, nthreads=8)
    E = o["sym_src"].shape[0]
    samp = math.log(0.1 * E) / math.log(E)
    init = np.random.default_rng(2).uniform(-10.0, 10.0, size=(g.n, 2))
    a, b = float(z["a"]), float(z["b"])
    _, logs = oracle.run_sgd(o, init, 1, a, b, 1.0, 5, 2, samp=samp, windowed=True,
                             epochs_to_log=(0,))
    before, order, negs, th, lr = logs[0]
    c = before.copy()
    oracle.sgd_sweep(c, o["sym_src"], o["sym_dst"], o["sym_w"], order, o["nbr_indptr"],
                     o["nbr_indices"], a, b, lr, 5, 2 ^ oracle.SPLIT_GAMMA)
    gk = gu.KnnGraph(n=g.n, k=15, directed=None, **{k_: o[k_] for k_ in (
        "rho", "sigma", "sym_src", "sym_dst", "sym_w", "nbr_indptr", "nbr_indices")})
    out, _ = gu.sgd_replay(gk, before, order, negs, th, a, b, lr, 5)
    assert _rel_err(out, c) <= REPLAY_REL_TOL


# ---------------------------------------------------- C2 Hogwild epochs
def test_sgd_zero_iterations_identity(gu):
    g = gu.build_graph([(0, 1), (1, 2), (2, 3), (3, 0)])
    _, knn = gu.partial_bfs(g, 2, seed=0)
    gk = gu.smooth_knn_weights(knn)
    init = gu.random_init(g, 0)
    cfg = gu.OptimizerConfig(iterations=0, k=2, seed=0)
    assert np.array_equal(gu.optimize_full(gk, init, cfg).coords, init.coords)
    assert np.array_equal(gu.optimize_sampled(gk, init, cfg).coords, init.coords)


def test_sgd_visit_log_coverage(gu):
    g = gu.synth_graph("scale_free", 300, seed=3, m0=3)
    _, knn = gu.partial_bfs(g, 6, seed=0)
    gk = gu.smooth_knn_weights(knn)
    init = gu.random_init(g, 1)
    E = gk.edge_count
    cfg = gu.OptimizerConfig(iterations=4, k=6, samp=1.0, seed=9)
    lf, ls = [], []
    gu.optimize_full(gk, init, cfg, visit_log=lf)
    gu.optimize_sampled(gk, init, cfg, visit_log=ls)
    for a_, b_ in zip(lf, ls):
        assert sorted(a_.tolist()) == list(range(E)) == sorted(b_.tolist())
    # pigeonhole: ceil(E / window) windows touch every edge
    s = int(math.floor(E ** 0.9))
    cfg2 = gu.OptimizerConfig(iterations=math.ceil(E / s), k=6, samp=0.9, seed=4)
    log = []
    gu.optimize_sampled(gk, init, cfg2, visit_log=log)
    assert set(np.concatenate(log).tolist()) == set(range(E))


def test_sgd_pure_attraction_shrinks_edge(gu):
    g = gu.build_graph([(0, 1)])
    _, knn = gu.partial_bfs(g, 1, seed=0)
    gk = gu.smooth_knn_weights(knn)
    init = gu.Layout(coords=np.array([[-4.0, 0.0], [4.0, 0.0]]))
    cfg = gu.OptimizerConfig(iterations=200, k=1, negative_sample_count=0,
                             learning_rate=0.05, seed=1)
    dists = []
    gu.optimize_full(gk, init, cfg, callback=lambda it, c: dists.append(
        np.linalg.norm(c[0] - c[1])), callback_every=10)
    assert all(b_ <= a_ + 1e-5 for a_, b_ in zip(dists, dists[1:]))
    assert dists[-1] < 1.0


def test_sgd_divergence_detected(gu):
    g = gu.build_graph([(0, 1)])
    _, knn = gu.partial_bfs(g, 1, seed=0)
    gk = gu.smooth_knn_weights(knn)
    init = gu.Layout(coords=np.array([[0.0, 0.0], [1.0, 0.0]]))
    cfg = gu.OptimizerConfig(iterations=5, k=1, learning_rate=1e308, seed=0)
    with pytest.raises(gu.OptimizationDiverged):
        gu.optimize_full(gk, init, cfg)


def test_drivers_run(gu):
    g = gu.build_graph([(i, (i + 1) % 6) for i in range(6)])
    cfg = gu.OptimizerConfig(iterations=30, k=2, seed=0)
    for fn in (gu.run_gumap, gu.run_ss_gumap, gu.run_sl_gumap, gu.run_sssl_gumap):
        lay, rep = fn(g, cfg)
        assert lay.n == 6 and np.all(np.isfinite(lay.coords))
        assert rep.total_ms >= max(rep.c0_ms, rep.c1_ms, rep.c2_ms)


def test_quality_c1_vs_reference(gu):
    """Check (c): NP / stress / crossings of the c1 layout over seeds vs the
    reference's own seed distribution (tests/golden/quality_c1.npz)."""
    from oracle.metrics import count_crossings, neighborhood_preservation, stress

    z = load_golden("quality_c1.npz")
    g = gu.synth_graph("grid", 2500)
    dset = gu.all_pairs_bfs(g)
    hop = np.array(dset.matrix, dtype=np.float64)
    # metric restatement pinned on the reference's own layouts
    for i, lay in enumerate((z["layout0"], z["layout1"])):
        assert abs(neighborhood_preservation(g, lay) - z["np_"][i]) < 1e-12
        assert abs(stress(g, lay, hop) - z["stress"][i]) < 1e-9
        assert count_crossings(g, lay) == int(z["crossings"][i])
    vals = []
    for seed in range(10):
        knn = gu.knn_from_full_distances(dset, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        init = gu.random_init(g, seed, 10.0)
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed)
        lay = gu.optimize_full(gk, init, cfg, tag="GUMAP").coords
        vals.append((neighborhood_preservation(g, lay), stress(g, lay, hop),
                     count_crossings(g, lay)))
    v = np.array(vals)
    ref = np.stack([z["np_"], z["stress"], z["crossings"]], axis=1)
    ratio = v.mean(axis=0) / ref.mean(axis=0)
    print("check (c) mean ratios gpu/ref [np, stress, crossings]:", ratio)
    # NP must not be worse than the reference's own spread allows
    se = ref.std(axis=0, ddof=1) / math.sqrt(ref.shape[0]) + v.std(axis=0, ddof=1) / math.sqrt(v.shape[0])
    assert v.mean(axis=0)[0] >= ref.mean(axis=0)[0] - 4 * se[0]
    assert v.mean(axis=0)[1] <= ref.mean(axis=0)[1] + 4 * se[1]
    assert v.mean(axis=0)[2] <= ref.mean(axis=0)[2] + 4 * se[2]


def test_quality_c3_sampled_vs_reference(gu, oracle):
    """Check (c) at SL scale: sampled NP / stress (2000 fixed sources) of the
    c3 SL-GUMAP layout vs the reference's 5 seeds (tests/golden/quality_c3.npz,
    scripts/quality_c3.py for the full sweep)."""
    from oracle.metrics import sampled_neighborhood_preservation, sampled_stress

    z = load_golden("quality_c3.npz")
    src = z["sources"]
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    rows = oracle.all_pairs_bfs_rows(g, src)
    vals = []
    for seed in range(3):
        _, knn = gu.partial_bfs(g, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        E = gk.edge_count
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed,
                                 samp=math.log(0.1 * E) / math.log(E))
        lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0), cfg).coords
        vals.append((sampled_neighborhood_preservation(lay, rows, src), sampled_stress(lay, rows, src)))
    v = np.array(vals)
    ref = np.stack([z["np_"], z["stress"]], axis=1)
    print("check (c) c3 mean ratios gpu/ref [np, stress]:", v.mean(axis=0) / ref.mean(axis=0))
    se = ref.std(axis=0, ddof=1) / math.sqrt(ref.shape[0]) + v.std(axis=0, ddof=1) / math.sqrt(v.shape[0])
    assert v.mean(axis=0)[0] >= ref.mean(axis=0)[0] - 4 * se[0]
    assert v.mean(axis=0)[1] <= ref.mean(axis=0)[1] + 4 * se[1]


def test_sharded_knn_nccl_single_rank(gu):
    """The NCCL path of distributed.sharded_knn (all_gather of records) on a
    one-rank group: identical to the single-GPU kNN (partial and full)."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2509_19703_b200.distributed import sharded_knn

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        g = gu.synth_graph("scale_free", 5000, seed=3, m0=3)
        knn = sharded_knn(g, 15, seed=7, mode="partial")
        _, ref = gu.partial_bfs(g, 15, seed=7)
        assert np.array_equal(knn.dst, ref.dst) and np.array_equal(knn.dist, ref.dist)
        assert np.array_equal(knn.indptr, ref.indptr)
        g2 = gu.synth_graph("grid", 900)
        knn2 = sharded_knn(g2, 15, seed=1, mode="full")
        ref2 = gu.knn_from_full_distances(gu.all_pairs_bfs(g2), 15, seed=1)
        assert np.array_equal(knn2.dst, ref2.dst) and np.array_equal(knn2.dist, ref2.dist)
    finally:
        dist.destroy_process_group()


def test_pinned_host_inputs(gu):
    """Graph arrays in page-locked host memory take the single-DMA upload
    path (device._is_pinned) and give the same records."""
    import torch

    from paper_2509_19703_b200.device import _is_pinned
    from paper_2509_19703_b200.graph import Graph

    g = gu.synth_graph("scale_free", 20000, seed=3, m0=3)

    def pinned(a):
        out = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True).numpy()
        out[...] = a
        return out

    gp = Graph(n=g.n, m=g.m, adj_indptr=pinned(np.asarray(g.adj_indptr)),
               adj_indices=pinned(np.asarray(g.adj_indices)), edges=g.edges)
    assert _is_pinned(gp.adj_indices) and not _is_pinned(np.asarray(g.adj_indices))
    _, a = gu.partial_bfs(g, 15, seed=7)
    _, b = gu.partial_bfs(gp, 15, seed=7)
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.dst, b.dst)
    assert np.array_equal(a.dist, b.dist)


def test_partial_bfs_host_path_matches_records(gu):
    """The public partial_bfs at a size where its host path engages (chunked
    row copies on a side stream, distances sent as uint8 and widened by host
    threads, all-rows-full indptr copied during the first kernel) returns
    exactly the device records, and the distance set shares them."""
    from paper_2509_19703_b200.device import device_csr
    from paper_2509_19703_b200.neighbors import partial_bfs_records

    g = gu.synth_graph("scale_free", 700_000, seed=5, m0=3)  # n * k * 8 B >= 64 MB
    dset, knn = gu.partial_bfs(g, 15, seed=9)
    assert knn._pending_bytes is not None  # the narrowed copy path ran
    assert knn._pending_bytes == (g.n + 1) * 8 + g.n * 15 * (4 + 1)
    nbr, dist, cnt = partial_bfs_records(device_csr(g), 15, 9, 0, g.n)
    assert np.all(cnt.cpu().numpy() == 15)
    assert knn.indptr.dtype == np.int64 and knn.dst.dtype == np.int32 and knn.dist.dtype == np.int32
    assert np.array_equal(knn.indptr, 15 * np.arange(g.n + 1))
    assert np.array_equal(knn.dst, nbr.cpu().numpy().reshape(-1))
    assert np.array_equal(knn.dist, dist.cpu().numpy().reshape(-1))
    assert np.array_equal(dset.nbr, knn.dst) and np.array_equal(dset.dist, knn.dist)
    assert np.array_equal(dset.indptr, knn.indptr)


def test_sgd_neighbor_filter_covers_neighbors(gu, monkeypatch):
    """The SGD negative-sampling Bloom words (csrc/sgd.cu, REC_TABLE: small
    caps when the exact sets are off) have the bit of every neighbour set, so
    skipping the row search on a clear bit never accepts a neighbour."""
    from paper_2509_19703_b200.layout import REC_TABLE, SgdPlan
    import torch

    monkeypatch.setenv("GU_SGD_HASH", "0")
    g = gu.synth_graph("scale_free", 5000, seed=4, m0=3)
    _, knn = gu.partial_bfs(g, 15, seed=1)
    gk = gu.smooth_knn_weights(knn)
    plan = SgdPlan(gk, 0, torch.device("cuda"))
    assert plan.record_mode == REC_TABLE
    filt = plan.filter.cpu().numpy().view(np.uint32)
    ip, ix = gk.nbr_indptr, gk.nbr_indices
    src = np.repeat(np.arange(gk.n), np.diff(ip))
    assert filt.shape == (gk.n, 2)
    _bloom_covers(filt[src], ix, (0x9E3779B1, 0x85EBCA77), 26)


def test_sgd_neighbor_hash_exact(gu):
    """Small caps use exact open-addressing sets of each head's neighbour ids
    (REC_HASH): every record points at its head's table, the table holds
    exactly the head's row, and the kernel's probe sequence (buckets of 4
    slots, home bucket = top log2(S / 4) bits of the Fibonacci product, linear
    probing over buckets until one holds the id or an empty slot) finds every
    neighbour and rejects every other id tried."""
    from paper_2509_19703_b200.layout import REC_HASH, _plan_for
    import torch

    g = gu.synth_graph("scale_free", 5000, seed=4, m0=3)  # hubs: long rows
    _, knn = gu.partial_bfs(g, 15, seed=1)
    gk = gu.smooth_knn_weights(knn)
    plan = _plan_for(gk, 0, torch.device("cuda"))
    assert plan.record_mode == REC_HASH
    tab = plan.filter.cpu().numpy()
    rec = plan.edges.cpu().numpy()
    perm = plan.perm.cpu().numpy()
    assert np.array_equal(rec[:, 0], gk.sym_src[perm]) and np.array_equal(rec[:, 1], gk.sym_dst[perm])
    ip, ix = gk.nbr_indptr, gk.nbr_indices
    off = np.zeros(gk.n, np.int64)
    lg = np.zeros(gk.n, np.int64)
    off[rec[:, 0]] = rec[:, 3].astype(np.uint32) >> 4
    lg[rec[:, 0]] = rec[:, 3] & 15
    rng = np.random.default_rng(3)

    def member(u, c):
        nb = (1 << int(lg[u])) // 4
        h = ((int(c) * 0x9E3779B1) & 0xFFFFFFFF) >> (34 - int(lg[u])) if lg[u] > 2 else 0
        while True:
            x = tab[off[u] + 4 * h: off[u] + 4 * h + 4]
            if (x == c).any():
                return True
            if (x < 0).any():
                return False
            h = (h + 1) % nb

    for u in np.unique(rec[:, 0]):
        row = ix[ip[u]:ip[u + 1]]
        S = 1 << int(lg[u])
        assert S >= 4 * row.shape[0]
        slots = tab[off[u]:off[u] + S]
        assert np.array_equal(np.sort(slots[slots >= 0]), np.sort(row))
        if u % 7 == 0:
            assert all(member(u, c) for c in row)
            others = np.setdiff1d(rng.integers(0, gk.n, 40), row)
            assert not any(member(u, c) for c in others)


def _bloom_covers(words, ids, mults, shift):
    """Every id has all of its hash bits set in the row's word."""
    for mult in mults:
        h = ((ids.astype(np.uint64) * np.uint64(mult)) & np.uint64(0xFFFFFFFF)) >> np.uint64(shift)
        w = words[np.arange(ids.shape[0]), (h >> np.uint64(5)).astype(np.int64)]
        assert np.all((w >> (h & np.uint64(31)).astype(np.uint32)) & 1)


def test_sgd_record_filter_covers_neighbors(gu):
    """32-byte edge records (GPU-filling epochs) carry their head's 128-bit
    Bloom word (3 hash bits per id): every neighbour of the head is covered,
    and the records hold the sym edges in the plan's order."""
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.layout import SgdPlan
    import torch

    g = gu.synth_graph("scale_free", 700_000, seed=4, m0=3)  # cap n/4 fills the GPU
    _, knn = gu.partial_bfs(g, 15, seed=1)
    gk = gu.smooth_knn_weights(knn)
    assert _lib.load().gu_sgd_record_bytes_for(0) == 32
    plan = SgdPlan(gk, 0, torch.device("cuda"))
    if plan.record_bytes != 32:
        pytest.skip("this graph's concurrency cap keeps 16-byte records")
    rec = plan.edges.cpu().numpy()
    perm = plan.perm.cpu().numpy()
    assert np.array_equal(rec[:, 0], gk.sym_src[perm]) and np.array_equal(rec[:, 1], gk.sym_dst[perm])
    words = rec[:, 4:8].view(np.uint32)
    ip, ix = gk.nbr_indptr, gk.nbr_indices
    heads = rec[:, 0]
    # check the words of a sample of records against their head's full row
    pick = np.random.default_rng(0).choice(rec.shape[0], size=20000, replace=False)
    for i in pick[:2000]:
        u = heads[i]
        row = ix[ip[u]:ip[u + 1]]
        _bloom_covers(np.repeat(words[i:i + 1], row.shape[0], axis=0), row,
                      (0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D), 25)


def test_sgd_range_records_rgg(gu):
    """GPU-filling epochs on a geometric graph run in a BFS locality order
    (csrc/order.cu) with each record carrying the head's neighbour-id window
    and 64-bit word (REC_RANGE): the records map back to the sym edges, the
    window and the word cover every neighbour, the order is a permutation, and
    the layout quality matches the unrelabelled 128-bit-Bloom epochs."""
    import os

    import torch
    from paper_2509_19703_b200 import fixtures
    from paper_2509_19703_b200.layout import REC_BLOOM, REC_RANGE, SgdPlan

    g = fixtures.rgg(700_000, 12.0, seed=5)
    _, knn = gu.partial_bfs(g, 15, seed=1)
    gk = gu.smooth_knn_weights(knn)
    plan = SgdPlan(gk, 0, torch.device("cuda"))
    assert plan.record_mode == REC_RANGE, plan.mean_window
    order = plan.order.cpu().numpy()
    relabel = plan.relabel.cpu().numpy()
    assert np.array_equal(np.sort(order), np.arange(g.n))
    assert np.array_equal(relabel[order], np.arange(g.n))
    rec = plan.edges.cpu().numpy()
    perm = plan.perm.cpu().numpy()
    assert np.array_equal(order[rec[:, 0]], gk.sym_src[perm])
    assert np.array_equal(order[rec[:, 1]], gk.sym_dst[perm])
    ip = plan.nbr_indptr.cpu().numpy().astype(np.int64)
    ix = plan.nbr_indices.cpu().numpy()
    pick = np.random.default_rng(0).choice(rec.shape[0], size=3000, replace=False)
    for i in pick:
        u = rec[i, 0]
        row = ix[ip[u]:ip[u + 1]]
        assert np.array_equal(np.sort(row), row)
        assert np.array_equal(np.sort(relabel[gk.nbr_indices[gk.nbr_indptr[order[u]]:
                                                             gk.nbr_indptr[order[u] + 1]]]), row)
        assert rec[i, 4] <= row.min() and row.max() <= rec[i, 5]
        _bloom_covers(np.repeat(rec[i:i + 1, 6:8].view(np.uint32), row.shape[0], axis=0), row,
                      (0x9E3779B1, 0x85EBCA77), 26)
    # same quality with and without the relabelling (statistically equal runs)
    from paper_2509_19703_b200 import metrics as M
    src = np.random.default_rng(1).choice(g.n, size=2000, replace=False)
    vals = {"1": [], "0": []}
    for relab in ("1", "0"):
        os.environ["GU_SGD_RELABEL"] = relab
        try:
            gk2 = gu.smooth_knn_weights(knn)
            for seed in (3, 4, 5):
                lay = gu.optimize_full(gk2, gu.random_init(g, seed, 10.0),
                                       gu.OptimizerConfig(iterations=100, k=15, seed=seed))
                vals[relab].append(M.neighborhood_preservation(g, lay, sources=src))
        finally:
            os.environ.pop("GU_SGD_RELABEL", None)
    ratio = np.mean(vals["1"]) / np.mean(vals["0"])
    print("NP relabelled / plain:", vals, ratio)
    # Hogwild runs of one seed differ by ~1-2% NP between repeats at this size
    assert abs(ratio - 1.0) < 0.025


@pytest.mark.parametrize("n", [(1 << 23) + 5, (1 << 24) + 7])
def test_partial_bfs_large_ids_unpacked_path(gu, oracle, n):
    """Large ids: from n >= 2^23 - 1 big balls leave the CTA tier (23-bit
    packed keys) for the 1024-id warp tier, and from n >= 2^24 - 1 tiers F /
    1a / 1b switch from packed (tag << 24 | id) keys to the MATCH election.
    A scale-free graph relabelled onto the top ids of an n-vertex space (the
    rest isolated); its sources' rows must equal the oracle's
    (_kernels.py:60-131)."""
    import torch

    from paper_2509_19703_b200.device import device_csr
    from paper_2509_19703_b200.fixtures import canonical_edges, graph_from_edges
    from paper_2509_19703_b200.neighbors import partial_bfs_records

    base = gu.synth_graph("scale_free", 20000, seed=5, m0=3)
    off = n - base.n
    src = np.repeat(np.arange(base.n), np.diff(base.adj_indptr))
    pairs = np.stack([src + off, base.adj_indices.astype(np.int64) + off], axis=1)
    pairs = pairs[pairs[:, 0] < pairs[:, 1]]
    g = graph_from_edges(n, canonical_edges(n, pairs))
    csr = device_csr(g)
    nb, dd, cnt = partial_bfs_records(csr, 15, 9, off, n, tier2_warps=1)
    torch.cuda.synchronize()
    o_n, o_d, o_c = oracle.partial_bfs_raw(g, 15, 9, src_begin=off, src_end=n,
                                           nthreads=oracle.max_threads())
    assert np.array_equal(cnt.cpu().numpy(), o_c)
    assert np.array_equal(nb.cpu().numpy().reshape(-1), o_n)
    assert np.array_equal(dd.cpu().numpy().reshape(-1), o_d)


def test_sgd_hash_fallback_for_huge_rows(gu):
    """A row above 8192 neighbour ids (a star's hub) cannot use the exact
    neighbour sets: the small-cap plan falls back to the gathered Bloom
    table (REC_TABLE) and the epochs still run."""
    from paper_2509_19703_b200.fixtures import canonical_edges, graph_from_edges
    from paper_2509_19703_b200.layout import REC_TABLE, _plan_for
    import torch

    n = 10000
    pairs = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], axis=1)
    g = graph_from_edges(n, canonical_edges(n, pairs))
    _, knn = gu.partial_bfs(g, 15, seed=0)
    gk = gu.smooth_knn_weights(knn)
    assert int(np.diff(gk.nbr_indptr).max()) > 8192
    plan = _plan_for(gk, 0, torch.device("cuda"))
    assert plan.record_mode == REC_TABLE
    lay = gu.optimize_full(gk, gu.random_init(g, 0), gu.OptimizerConfig(iterations=5, k=15, seed=0))
    assert np.all(np.isfinite(lay.coords))


def test_random_uniform_matches_numpy(gu):
    """gu_random_uniform == numpy default_rng(seed).uniform(low, high, count)
    bit for bit (PCG64 jump-ahead per thread run), and random_init's GPU path
    equals the reference's numpy draws."""
    import torch

    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import stream_ptr

    for seed, count, lo, hi in ((0, 1, -10.0, 10.0), (2, 200_003, -10.0, 10.0),
                                (2**40 + 3, 4097, -1.5, 3.25), (2**64 - 1, 777, 0.0, 1.0)):
        out = torch.empty(count, dtype=torch.float64, device="cuda")
        _lib.call("gu_random_uniform", count, seed, lo, hi, _lib.ptr(out), stream_ptr())
        ref = np.random.default_rng(seed).uniform(lo, hi, count)
        assert np.array_equal(out.cpu().numpy(), ref), seed
    g = gu.synth_graph("scale_free", 100_000, seed=2, m0=3)
    lay = gu.random_init(g, 7, 10.0)
    assert np.array_equal(lay.coords, np.random.default_rng(7).uniform(-10.0, 10.0, (g.n, 2)))


def test_sgd_negative_counts_small_cap(gu):
    """Small-cap epochs (exact neighbour sets, one visit on four lanes) with
    0, 7 and 11 negatives per visit: finite layouts; 0 negatives moves the
    layout by attraction only (the points contract)."""
    g = gu.synth_graph("grid", 2500)
    gk = gu.smooth_knn_weights(gu.knn_from_full_distances(gu.all_pairs_bfs(g), 15, seed=0))
    init = gu.random_init(g, 0, 10.0)
    for nn in (0, 7, 11):  # 11: the quad kernel's third slot round (slots 8..10)
        cfg = gu.OptimizerConfig(iterations=20, k=15, seed=0, negative_sample_count=nn)
        lay = gu.optimize_full(gk, init, cfg)
        assert np.all(np.isfinite(lay.coords))
        if nn == 0:
            assert np.std(lay.coords) < np.std(init.coords)


@pytest.mark.parametrize("case", ["n1", "n2", "k20_1", "k20_15", "k20_19", "k20_25", "star_15",
                                  "star_32", "star_33", "path_15"])
def test_partial_bfs_edge_shapes(gu, oracle, case):
    """Degenerate shapes against the oracle: a single vertex, no edges, a
    clique at k up to and beyond n - 1 (level-1 crossings of every size), a
    1000-leaf star around k = 32 (hub rows: tier C / tier 2) and a path."""
    from paper_2509_19703_b200.fixtures import canonical_edges, graph_from_edges

    def g_of(n, pairs):
        return graph_from_edges(n, canonical_edges(n, np.asarray(pairs, np.int64).reshape(-1, 2)))

    kind, _, kk = case.partition("_")
    if kind == "n1":
        g, k = g_of(1, []), 5
    elif kind == "n2":
        g, k = g_of(2, []), 1
    elif kind == "k20":
        g = g_of(20, [(i, j) for i in range(20) for j in range(i + 1, 20)])
        k = int(kk)
    elif kind == "star":
        g = g_of(1000, [(0, j) for j in range(1, 1000)])
        k = int(kk)
    else:
        g = g_of(300, [(i, i + 1) for i in range(299)])
        k = int(kk)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, knn = gu.partial_bfs(g, k, seed=3)
        ip, dst, dist = oracle.partial_bfs(g, k, seed=3)
    assert np.array_equal(knn.indptr, ip) and np.array_equal(knn.dst, dst)
    assert np.array_equal(knn.dist, dist)


@pytest.mark.parametrize("k", [2, 5, 15, 31])
@pytest.mark.parametrize("hub_pos", ["low", "mid", "high"])
def test_partial_bfs_hub_tier(gu, oracle, k, hub_pos):
    """Tier H (csrc/partial_bfs.cu): sources next to one high-degree vertex,
    whose row is handled implicitly.  Hubs with low / middle / high ids (the
    hub before, between and after the other parents in queue order), hubs
    adjacent to each other (members of N(H) among N(s)), leaves shared by two
    hubs (explicit second hub), and a sparse background -- every row against
    the oracle, and the tier is checked to have run."""
    import ctypes
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import device_csr, workspace
    from paper_2509_19703_b200.fixtures import canonical_edges, graph_from_edges
    from paper_2509_19703_b200.neighbors import _tier2_warps, partial_bfs_records

    rng = np.random.default_rng(100 + k)
    n = 6000
    hubs = {"low": np.arange(4), "mid": np.arange(3000, 3004),
            "high": np.arange(n - 4, n)}[hub_pos]
    pairs = []
    others = np.setdiff1d(np.arange(n), hubs)
    # a sparse background (ring + random chords)
    pairs += [(int(others[i]), int(others[(i + 1) % len(others)])) for i in range(len(others))]
    pairs += [tuple(int(x) for x in rng.choice(others, 2, replace=False)) for _ in range(4000)]
    # hubs of degree ~700, ~400, ~150, ~80; the first two share 60 leaves
    for h, d in zip(hubs, (700, 400, 150, 80)):
        pairs += [(int(h), int(x)) for x in rng.choice(others, d, replace=False)]
    shared = rng.choice(others, 60, replace=False)
    pairs += [(int(hubs[0]), int(x)) for x in shared] + [(int(hubs[1]), int(x)) for x in shared]
    pairs += [(int(hubs[0]), int(hubs[1])), (int(hubs[1]), int(hubs[2]))]
    g = graph_from_edges(n, canonical_edges(n, np.asarray(pairs, np.int64)))
    csr = device_csr(g)
    t2 = _tier2_warps(g.n)
    lib = _lib.load()
    ws = workspace(lib.gu_partial_bfs_workspace_size(g.n, g.n, t2), csr.device)
    nbr, dist, cnt = partial_bfs_records(csr, k, 9, 0, g.n, tier2_warps=t2, ws=ws)
    tiers = (ctypes.c_int32 * 4)()
    assert lib.gu_partial_bfs_tier_counts(ctypes.c_void_p(ws.data_ptr()), g.n, tiers) == 0
    o_n, o_d, o_c = oracle.partial_bfs_raw(g, k, 9, nthreads=4)
    assert np.array_equal(cnt.cpu().numpy(), o_c)
    assert np.array_equal(nbr.cpu().numpy().reshape(-1), o_n)
    assert np.array_equal(dist.cpu().numpy().reshape(-1), o_d)
    entered_h, entered_big = int(tiers[1]), int(tiers[2])
    print(f"k={k} hubs {hub_pos}: left F {tiers[0]}, entered H {entered_h}, big-ball tier {entered_big}")
    if k >= 5:  # (k = 2: only degree-1 sources stop at level 2, the tier has nothing to do)
        assert entered_h > 0 and entered_big < entered_h  # tier H ran and finished sources


def test_symmetrize_memo_matches_plain(gu):
    """gu_symmetrize_memo (backward weights read from K5's profile table, the
    path smooth_knn_weights takes) against plain gu_symmetrize (weights
    gathered from w) on the same kNN rows: identical arrays, including rows
    that have no profile (> 4 distance runs) and therefore gather."""
    import ctypes
    import torch
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import stream_ptr, workspace

    rng = np.random.default_rng(5)
    n, k = 20000, 15
    dist = np.empty((n, k), np.int32)
    for v in range(n):
        if v % 9 == 0:   # six runs: no profile key, solved and gathered directly
            dist[v] = np.sort(rng.integers(1, 7, size=k))
        else:
            t0 = int(rng.integers(1, k))
            dist[v] = [1] * t0 + [2] * (k - t0)
    dst = np.stack([rng.choice(n - 1, size=k, replace=False) for _ in range(n)]).astype(np.int32)
    dst += dst >= np.arange(n)[:, None]  # no self entries
    order = np.lexsort((dst, dist), axis=1)
    dst = np.take_along_axis(dst, order, 1)
    dist = np.take_along_axis(dist, order, 1)
    indptr = (k * np.arange(n + 1)).astype(np.int64)
    knn = gu.DirectedKnn(n=n, k=k, indptr=indptr, dst=dst.reshape(-1), dist=dist.reshape(-1))
    gk = gu.smooth_knn_weights(knn)  # memo path
    dev = torch.device("cuda")
    lib = _lib.load()
    nnz = n * k
    d_ip = torch.from_numpy(indptr).to(dev)
    d_dst = torch.from_numpy(dst.reshape(-1)).to(dev)
    d_w = gk._dev["w"]  # the directed weights K5 produced (device-resident)
    ws = workspace(lib.gu_symmetrize_workspace_size(n, nnz), dev)
    s_src = torch.empty(2 * nnz, dtype=torch.int32, device=dev)
    s_dst = torch.empty(2 * nnz, dtype=torch.int32, device=dev)
    s_w = torch.empty(2 * nnz, dtype=torch.float64, device=dev)
    nip = torch.empty(n + 1, dtype=torch.int64, device=dev)
    E = ctypes.c_int64(0)
    _lib.call("gu_symmetrize", n, nnz, _lib.ptr(d_ip), _lib.ptr(d_dst), _lib.ptr(d_w), _lib.ptr(s_src),
              _lib.ptr(s_dst), _lib.ptr(s_w), _lib.ptr(nip), ctypes.byref(E), _lib.ptr(ws), ws.numel(),
              stream_ptr(dev))
    E = int(E.value)
    assert E == gk.edge_count
    assert np.array_equal(s_src[:E].cpu().numpy(), gk.sym_src)
    assert np.array_equal(s_dst[:E].cpu().numpy(), gk.sym_dst)
    assert np.array_equal(s_w[:E].cpu().numpy(), gk.sym_w)  # bit-identical
    assert np.array_equal(nip.cpu().numpy(), gk.nbr_indptr)
