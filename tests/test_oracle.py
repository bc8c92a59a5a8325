"""Pin the CPU oracle (oracle/) to the reference's golden vectors (CPU only).

The fixtures were produced by the live reference (tests/golden/make_golden.py);
every check here is bit-exact.
"""

import math

import numpy as np
import pytest

from conftest import golden_graphs, load_golden, sha, split
from paper_2509_19703_b200 import fixtures as F


def test_partial_bfs_small_graphs(oracle):
    for g, k, seed, exp in golden_graphs("partial_small.npz"):
        ip, dst, dist = oracle.partial_bfs(g, k, seed=seed, nthreads=2)
        assert np.array_equal(ip, exp["indptr"])
        assert np.array_equal(dst, exp["dst"])
        assert np.array_equal(dist, exp["dist"])


def test_full_knn_small_graphs(oracle):
    for g, k, seed, exp in golden_graphs("full_small.npz"):
        m = oracle.all_pairs_bfs(g)
        assert sha(m) == exp["apsp_sha"]
        for res in (oracle.knn_from_full_distances(m, k, seed=seed),
                    oracle.full_knn(g, k, seed=seed, nthreads=2)):
            assert np.array_equal(res[0], exp["indptr"])
            assert np.array_equal(res[1], exp["dst"])
            assert np.array_equal(res[2], exp["dist"])


def test_numpy_permutation_restatement(oracle):
    for seed in (0, 1, 7, 2**32 + 5, 2**40 + 3):
        for key in (0, 3, 2**31 + 1, 2**33):
            for T in (1, 2, 13, 200):
                want = np.random.default_rng(
                    np.random.SeedSequence(entropy=seed, spawn_key=(key,))).permutation(T)
                assert np.array_equal(oracle.numpy_permutation(seed, key, T), want)


def test_smooth_cases(oracle):
    z = load_golden("smooth_cases.npz")
    for i in range(z["n"].shape[0]):
        n, k = int(z["n"][i]), int(z["k"][i])
        ip = split(z["indptr"], z["indptr_off"], i)
        dst = split(z["dst"], z["dst_off"], i)
        dist = split(z["dist"], z["dist_off"], i)
        o = oracle.smooth_knn_weights(n, ip, dst, dist, k)
        assert np.array_equal(o["rho"], split(z["rho"], z["rho_off"], i))
        assert np.array_equal(o["sigma"], split(z["sigma"], z["sigma_off"], i))
        assert np.array_equal(o["sym_src"], split(z["sym_src"], z["sym_src_off"], i))
        assert np.array_equal(o["sym_dst"], split(z["sym_dst"], z["sym_dst_off"], i))
        assert np.array_equal(o["sym_w"], split(z["sym_w"], z["sym_w_off"], i))
        assert np.array_equal(o["nbr_indptr"], split(z["nbr_indptr"], z["nbr_indptr_off"], i))


def test_c1_grid_pipeline(oracle):
    z = load_golden("c1.npz")
    g = F.grid(2500)
    m = oracle.all_pairs_bfs(g, nthreads=4)
    assert sha(m) == str(z["apsp_sha"])
    ip, dst, dist = oracle.full_knn(g, 15, seed=0, nthreads=4)
    assert np.array_equal(ip, z["knn_indptr"]) and np.array_equal(dst, z["knn_dst"])
    assert np.array_equal(dist, z["knn_dist"])
    ip7, dst7, dist7 = oracle.full_knn(g, 5, seed=7, nthreads=4)
    assert np.array_equal(dst7, z["knn7_dst"]) and np.array_equal(dist7, z["knn7_dist"])
    o = oracle.smooth_knn_weights(g.n, ip, dst, dist, 15)
    for key in ("rho", "sigma", "sym_src", "sym_dst", "sym_w", "nbr_indptr", "nbr_indices"):
        assert np.array_equal(o[key], z[key]), key
    # two full epochs of the reference schedule, bit-exact
    a, b = float(z["a"]), float(z["b"])
    gk = o
    c = np.array(z["init"], copy=True)
    rng = np.random.default_rng(np.random.SeedSequence(entropy=0, spawn_key=(29,)))
    state = (0 ^ oracle.SPLIT_GAMMA)
    for it, key in ((0, "after1"), (1, "after2")):
        order = rng.permutation(gk["sym_src"].shape[0])
        assert np.array_equal(order, z["order%d" % it])
        lr = 1.0 * (1.0 - it / 200)
        state, _, _ = oracle.sgd_sweep(c, gk["sym_src"], gk["sym_dst"], gk["sym_w"], order,
                                       gk["nbr_indptr"], gk["nbr_indices"], a, b, lr, 5, state)
        assert np.array_equal(c, z[key]), key


def test_c1_full_run_matches_reference_final(oracle):
    z = load_golden("c1.npz")
    gk = dict(sym_src=z["sym_src"], sym_dst=z["sym_dst"], sym_w=z["sym_w"],
              nbr_indptr=z["nbr_indptr"], nbr_indices=z["nbr_indices"])
    coords, _ = oracle.run_sgd(gk, z["init"], 200, float(z["a"]), float(z["b"]), 1.0, 5, 0,
                               windowed=False)
    assert np.array_equal(coords, z["final"])


def test_c3_scale_free_pipeline(oracle):
    z = load_golden("c3.npz")
    g = F.scale_free(100000, seed=2, m0=3)
    ip, dst, dist = oracle.partial_bfs(g, 15, seed=2, nthreads=8)
    assert sha(ip) == str(z["knn_indptr_sha"])
    assert sha(dst) == str(z["knn_dst_sha"])
    assert sha(dist) == str(z["knn_dist_sha"])
    o = oracle.smooth_knn_weights(g.n, ip, dst, dist, 15, nthreads=8)
    assert sha(o["rho"]) == str(z["rho_sha"])
    assert sha(o["sigma"]) == str(z["sigma_sha"])
    assert sha(o["sym_src"]) == str(z["sym_src_sha"])
    assert sha(o["sym_dst"]) == str(z["sym_dst_sha"])
    assert sha(o["sym_w"]) == str(z["sym_w_sha"])
    E = o["sym_src"].shape[0]
    assert E == int(z["E"])
    samp = math.log(0.1 * E) / math.log(E)
    init = np.random.default_rng(2).uniform(-10.0, 10.0, size=(g.n, 2))
    coords, logs = oracle.run_sgd(o, init, 3, float(z["a"]), float(z["b"]), 1.0, 5, 2,
                                  samp=samp, windowed=True, epochs_to_log=(0, 1, 2))
    # run_sgd(t=3) has a different lr schedule than the t=200 reference run:
    # replay the logged orders with the t=200 learning rates instead
    c = np.array(init, copy=True)
    st = (2 ^ oracle.SPLIT_GAMMA)
    for it in range(3):
        order = logs[it][1]
        st, _, _ = oracle.sgd_sweep(c, o["sym_src"], o["sym_dst"], o["sym_w"], order,
                                    o["nbr_indptr"], o["nbr_indices"], float(z["a"]),
                                    float(z["b"]), 1.0 * (1.0 - it / 200), 5, st)
        if it == 0:
            assert sha(c) == str(z["after1_sha"])
            assert np.array_equal(c[z["sample"]], z["after1_sample"])
        if it == 1:
            assert np.array_equal(c[z["sample"]], z["after2_sample"])
    assert sha(c) == str(z["after3_sha"])


def test_fuzzy_union_c_matches_numpy_restatement(oracle):
    """oracle.c or_fuzzy_union (used by the full-size C1 parity tests) gives
    the same arrays as the numpy restatement pinned above: the golden smooth
    cases, c1, and random rows with duplicates, unsorted ids, exact-zero
    weights and one-sided pairs."""
    z = load_golden("smooth_cases.npz")
    for i in range(z["n"].shape[0]):
        n, k = int(z["n"][i]), int(z["k"][i])
        ip = split(z["indptr"], z["indptr_off"], i)
        dst = split(z["dst"], z["dst_off"], i)
        dist = split(z["dist"], z["dist_off"], i)
        a = oracle.smooth_knn_weights(n, ip, dst, dist, k)
        b = oracle.smooth_knn_weights(n, ip, dst, dist, k, union="c")
        for key in ("sym_src", "sym_dst", "sym_w", "nbr_indptr", "nbr_indices"):
            assert np.array_equal(a[key], b[key]), (i, key)
    z = load_golden("c1.npz")
    o = oracle.smooth_knn_weights(2500, z["knn_indptr"], z["knn_dst"], z["knn_dist"], 15,
                                  union="c")
    for key in ("sym_src", "sym_dst", "sym_w", "nbr_indptr", "nbr_indices"):
        assert np.array_equal(o[key], z[key]), key
    rng = np.random.default_rng(5)
    for trial in range(20):
        n = int(rng.integers(2, 300))
        counts = rng.integers(0, 12, size=n)
        ip = np.zeros(n + 1, np.int64)
        ip[1:] = np.cumsum(counts)
        dst = rng.integers(0, n, size=int(ip[-1])).astype(np.int32)
        w = rng.random(int(ip[-1]))
        w[rng.random(w.shape[0]) < 0.2] = 0.0
        a = oracle.fuzzy_union_symmetrize(n, ip, dst, w)
        b = oracle.fuzzy_union_c(n, ip, dst, w, nthreads=2)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), trial
