"""Freeze golden vectors from the LIVE reference (run in the build container).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Imports graph_umap read-only from /root/reference/pkg/src and writes small
.npz fixtures next to this file.  The reference does not exist on the GPU box:
tests only ever read the committed .npz files.  Large arrays are stored as
SHA-256 digests plus explicit samples.

Fixture inputs come from paper_2509_19703_b200.fixtures, whose grid /
scale_free / random_connected_graph are draw-for-draw restatements of the
reference generators (checked here: the reference's own synth_graph output is
asserted equal before anything is frozen).
"""

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import graph_umap as gu  # noqa: E402
import numba  # noqa: E402
import scipy  # noqa: E402

from paper_2509_19703_b200 import fixtures as F  # noqa: E402


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def flat(lists, dtype):
    if not lists:
        return np.zeros(0, dtype), np.zeros(1, np.int64)
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in lists])
    return np.concatenate([np.asarray(x, dtype) for x in lists]), off


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def gen_partial_small():
    """Acceptance-criterion-1 style graphs (test_acceptance.py:45-63)."""
    rng = np.random.default_rng(101)
    edges_l, n_l, k_l, seed_l, ip_l, dst_l, dist_l = [], [], [], [], [], [], []
    graphs = []
    for trial in range(100):  # all 100 graphs of criterion 1
        n, e = F.random_connected_graph(rng, n_max=200)
        k = int(rng.integers(1, 21))
        graphs.append((np.array(e, np.int64), k, trial))
    # special shapes: star tie-break, path, small components, complete graph
    graphs.append((np.array([(0, i) for i in range(1, 6)]), 3, 5))
    graphs.append((np.array([(i, i + 1) for i in range(4)]), 2, 0))
    graphs.append((np.array([(0, 1), (1, 2), (3, 4)]), 3, 0))
    graphs.append((np.array([(i, j) for i in range(6) for j in range(i + 1, 6)]), 10, 1))
    graphs.append((np.array([(0, i) for i in range(1, 300)] + [(i, i + 300) for i in range(1, 300)]), 15, 9))
    import warnings
    for e, k, seed in graphs:
        g = gu.build_graph([tuple(map(int, x)) for x in e])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            _, kn = gu.partial_bfs(g, k, seed=seed)
        edges_l.append(np.asarray(g.edges, np.int64).reshape(-1))
        n_l.append(g.n)
        k_l.append(k)
        seed_l.append(seed)
        ip_l.append(kn.indptr)
        dst_l.append(kn.dst)
        dist_l.append(kn.dist)
    E, Eo = flat(edges_l, np.int64)
    IP, IPo = flat(ip_l, np.int64)
    D, Do = flat(dst_l, np.int32)
    DD, _ = flat(dist_l, np.int32)
    save("partial_small.npz", edges=E, edges_off=Eo, n=np.array(n_l), k=np.array(k_l),
         seed=np.array(seed_l, np.uint64), indptr=IP, indptr_off=IPo, dst=D, dst_off=Do,
         dist=DD)


def gen_full_small():
    rng = np.random.default_rng(202)
    cases = []
    for t in range(12):
        n, e = F.random_connected_graph(rng, n_max=120)
        cases.append((np.array(e, np.int64), [1, 5, 15][t % 3], [0, 7, 2**40 + 3][t % 3]))
    cases.append((np.array([(0, 1), (2, 3), (3, 4), (4, 5)]), 3, 0))   # disconnected
    cases.append((np.array([(0, i) for i in range(1, 40)]), 5, 11))     # star: big tie set
    import warnings
    out = dict(edges=[], n=[], k=[], seed=[], indptr=[], dst=[], dist=[], apsp_sha=[])
    for e, k, seed in cases:
        g = gu.build_graph([tuple(map(int, x)) for x in e])
        ds = gu.all_pairs_bfs(g)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            kn = gu.knn_from_full_distances(ds, k, seed=seed)
        out["edges"].append(np.asarray(g.edges, np.int64).reshape(-1))
        out["n"].append(g.n)
        out["k"].append(k)
        out["seed"].append(seed)
        out["indptr"].append(kn.indptr)
        out["dst"].append(kn.dst)
        out["dist"].append(kn.dist)
        out["apsp_sha"].append(sha(ds.matrix.astype(np.int32)))
    E, Eo = flat(out["edges"], np.int64)
    IP, IPo = flat(out["indptr"], np.int64)
    D, Do = flat(out["dst"], np.int32)
    DD, _ = flat(out["dist"], np.int32)
    save("full_small.npz", edges=E, edges_off=Eo, n=np.array(out["n"]), k=np.array(out["k"]),
         seed=np.array(out["seed"], np.uint64), indptr=IP, indptr_off=IPo, dst=D, dst_off=Do,
         dist=DD, apsp_sha=np.array(out["apsp_sha"]))


def gen_smooth_cases():
    """DirectedKnn inputs straight into smooth_knn_weights (neighbors.py:245)."""
    rng = np.random.default_rng(303)
    cases = [
        # test_neighbors.py:169-189 two-neighbour example
        (3, 2, [0, 2, 4, 6], [1, 2, 0, 2, 0, 1], [1, 2, 1, 2, 1, 2]),
        # test_neighbors.py:192-202 all identical -> sigma max
        (2, 2, [0, 1, 2], [1, 0], [1, 1]),
        # duplicate directed pair inside a row (first occurrence wins)
        (3, 3, [0, 3, 4, 6], [1, 1, 2, 0, 0, 1], [1, 2, 2, 1, 1, 1]),
    ]
    for t in range(25):
        n = int(rng.integers(3, 60))
        k = int(rng.integers(1, 20))
        counts = rng.integers(1, k + 1, n) if t % 2 else np.full(n, k)
        ip = np.concatenate([[0], np.cumsum(counts)])
        dst, dist = [], []
        for v in range(n):
            others = np.setdiff1d(np.arange(n), [v])
            c = int(counts[v])
            pick = rng.choice(others, size=min(c, others.shape[0]), replace=others.shape[0] < c)
            d = np.sort(rng.integers(1, 1 + int(rng.integers(1, 7)), pick.shape[0]))
            dst.extend(pick.tolist())
            dist.extend(d.tolist())
        cases.append((n, k, ip.tolist(), dst, dist))
    rec = dict(n=[], k=[], indptr=[], dst=[], dist=[], rho=[], sigma=[], sym_src=[],
               sym_dst=[], sym_w=[], nbr_indptr=[])
    for n, k, ip, dst, dist in cases:
        ip = np.array(ip, np.int64)
        counts = np.diff(ip)
        dst = np.array(dst, np.int32)[: ip[-1]]
        dist = np.array(dist, np.int32)[: ip[-1]]
        if dst.shape[0] < ip[-1]:
            continue
        kn = gu.DirectedKnn(n=n, k=k, indptr=ip, dst=dst, dist=dist)
        gk = gu.smooth_knn_weights(kn)
        rec["n"].append(n)
        rec["k"].append(k)
        rec["indptr"].append(ip)
        rec["dst"].append(dst)
        rec["dist"].append(dist)
        rec["rho"].append(gk.rho)
        rec["sigma"].append(gk.sigma)
        rec["sym_src"].append(gk.sym_src)
        rec["sym_dst"].append(gk.sym_dst)
        rec["sym_w"].append(gk.sym_w)
        rec["nbr_indptr"].append(gk.nbr_indptr)
        del counts
    arrays = dict(n=np.array(rec["n"]), k=np.array(rec["k"]))
    for key, dt in (("indptr", np.int64), ("dst", np.int32), ("dist", np.int32),
                    ("rho", np.float64), ("sigma", np.float64), ("sym_src", np.int32),
                    ("sym_dst", np.int32), ("sym_w", np.float64), ("nbr_indptr", np.int64)):
        a, off = flat(rec[key], dt)
        arrays[key] = a
        arrays[key + "_off"] = off
    save("smooth_cases.npz", **arrays)


def gen_c1():
    g = F.grid(2500)
    rg = gu.synth_graph("grid", 2500)
    assert np.array_equal(g.adj_indices, rg.adj_indices) and np.array_equal(g.adj_indptr, rg.adj_indptr)
    ds = gu.all_pairs_bfs(rg)
    kn = gu.knn_from_full_distances(ds, 15, seed=0)
    kn7 = gu.knn_from_full_distances(ds, 5, seed=7)
    gk = gu.smooth_knn_weights(kn)
    init = gu.random_init(rg, 0, 10.0)
    cfg = gu.OptimizerConfig(iterations=200, k=15, seed=0, learning_rate=1.0,
                             negative_sample_count=5, min_dist=0.1)
    a, b = cfg.curve()
    snaps = {}

    def cb(it, coords):
        snaps[it] = coords
    log = []
    final = gu.optimize_full(gk, init, cfg, visit_log=log, callback=cb, callback_every=1)
    # instrumented epochs: negatives + thetas of epochs 0 and 1, from the oracle
    # restatement, which tests/test_oracle.py pins bit-exact against snaps[1], [2]
    save("c1.npz", apsp_sha=np.array(sha(ds.matrix)), knn_indptr=kn.indptr, knn_dst=kn.dst,
         knn_dist=kn.dist, knn7_indptr=kn7.indptr, knn7_dst=kn7.dst, knn7_dist=kn7.dist,
         rho=gk.rho, sigma=gk.sigma, sym_src=gk.sym_src, sym_dst=gk.sym_dst, sym_w=gk.sym_w,
         nbr_indptr=gk.nbr_indptr, nbr_indices=gk.nbr_indices, a=a, b=b,
         init=init.coords, order0=log[0], order1=log[1], after1=snaps[1], after2=snaps[2],
         after10=snaps[10], final=final.coords)


def gen_c3():
    g = F.scale_free(100000, seed=2, m0=3)
    rg = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    assert np.array_equal(g.adj_indices, rg.adj_indices) and np.array_equal(g.adj_indptr, rg.adj_indptr)
    _, kn = gu.partial_bfs(rg, 15, seed=2)
    gk = gu.smooth_knn_weights(kn)
    E = gk.edge_count
    samp = math.log(0.1 * E) / math.log(E)
    init = gu.random_init(rg, 2, 10.0)
    cfg = gu.OptimizerConfig(iterations=200, k=15, seed=2, samp=samp)
    a, b = cfg.curve()
    snaps = {}

    # only the first 3 epochs are needed: run the 200-iteration schedule and
    # stop it from the callback after epoch 3
    class Stop(Exception):
        pass

    def cb2(it, coords):
        snaps[it] = coords
        if it >= 3:
            raise Stop()
    try:
        gu.optimize_sampled(gk, init, cfg, callback=cb2, callback_every=1)
    except Stop:
        pass
    sample = np.arange(0, g.n, 97)
    save("c3.npz", knn_indptr_sha=np.array(sha(kn.indptr)), knn_dst_sha=np.array(sha(kn.dst)),
         knn_dist_sha=np.array(sha(kn.dist)), knn_indptr_head=kn.indptr[:2001],
         knn_dst_head=kn.dst[:30000], knn_dist_head=kn.dist[:30000],
         rho_sha=np.array(sha(gk.rho)), sigma_sha=np.array(sha(gk.sigma)),
         sigma_sample=gk.sigma[sample], sample=sample, E=np.array(E),
         sym_src_sha=np.array(sha(gk.sym_src)), sym_dst_sha=np.array(sha(gk.sym_dst)),
         sym_w_sha=np.array(sha(gk.sym_w)), sym_w_head=gk.sym_w[:20000], samp=samp, a=a, b=b,
         after1_sha=np.array(sha(snaps[1])), after1_sample=snaps[1][sample],
         after2_sample=snaps[2][sample], after3_sha=np.array(sha(snaps[3])))


def gen_quality_c1(nseeds=20):
    """Check (c) reference statistics: c1 pipeline with random init per seed."""
    rg = gu.synth_graph("grid", 2500)
    ds = gu.all_pairs_bfs(rg)
    vals = []
    layouts = []
    for seed in range(nseeds):
        kn = gu.knn_from_full_distances(ds, 15, seed=seed)
        gk = gu.smooth_knn_weights(kn)
        init = gu.random_init(rg, seed, 10.0)
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed)
        lay = gu.optimize_full(gk, init, cfg, tag="GUMAP")
        npv = gu.neighborhood_preservation(rg, lay)
        st = gu.stress(rg, lay)
        cr = gu.count_crossings(rg, lay)
        vals.append((npv, st, cr))
        if seed < 2:
            layouts.append(lay.coords)
        print("quality seed", seed, vals[-1], flush=True)
    v = np.array(vals, np.float64)
    save("quality_c1.npz", np_=v[:, 0], stress=v[:, 1], crossings=v[:, 2],
         layout0=layouts[0], layout1=layouts[1])


def gen_quality_c3(nseeds=5):
    """Check (c) at SL scale: the reference's c3 SL pipeline (BA 100k, random
    init, 200 epochs, 10% window) for seeds 0..nseeds-1; sampled NP / stress
    over a fixed 2000-source sample (oracle/metrics.py estimators)."""
    import time
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from oracle.metrics import (sample_sources, sampled_neighborhood_preservation,
                                sampled_stress)
    rg = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    src = sample_sources(rg.n)
    rows = np.empty((len(src), rg.n), np.int32)
    O.lib().or_apsp_rows(rg.n, rg.adj_indptr.ctypes.data_as(O._i64p),
                         np.ascontiguousarray(rg.adj_indices, np.int32).ctypes.data_as(O._i32p),
                         src.astype(np.int64).ctypes.data_as(O._i64p), len(src),
                         rows.ctypes.data_as(O._i32p), 8)
    vals = []
    for seed in range(nseeds):
        t = time.time()
        _, kn = gu.partial_bfs(rg, 15, seed=seed)
        gk = gu.smooth_knn_weights(kn)
        E = gk.edge_count
        samp = math.log(0.1 * E) / math.log(E)
        lay = gu.optimize_sampled(gk, gu.random_init(rg, seed, 10.0),
                                  gu.OptimizerConfig(iterations=200, k=15, seed=seed, samp=samp))
        npv = sampled_neighborhood_preservation(lay.coords, rows, src)
        st = sampled_stress(lay.coords, rows, src)
        vals.append((npv, st))
        print("quality c3 seed", seed, vals[-1], f"{time.time() - t:.1f}s", flush=True)
    v = np.array(vals)
    save("quality_c3.npz", np_=v[:, 0], stress=v[:, 1], sources=src)



# ---- exact check (c) values at c3: workers for a process pool (top level)
_Q = {}


def _q_init(indptr, indices, coords, edges):
    from oracle import oracle as O
    _Q.update(indptr=indptr, indices=indices, coords=coords, edges=edges, O=O)


def _q_rows(lo, hi):
    O = _Q["O"]
    n = _Q["indptr"].shape[0] - 1
    src = np.arange(lo, hi, dtype=np.int64)
    rows = np.empty((hi - lo, n), np.int32)
    O.lib().or_apsp_rows(n, _Q["indptr"].ctypes.data_as(O._i64p),
                         _Q["indices"].ctypes.data_as(O._i32p), src.ctypes.data_as(O._i64p),
                         hi - lo, rows.ctypes.data_as(O._i32p), 1)
    return rows


def _q_chunk(args):
    """metrics.py:41-79 (NP terms) and metrics.py:106-113 (stress scale sums)
    for sources [lo, hi), restated chunk-wise as oracle/metrics.py does."""
    from scipy.spatial.distance import cdist
    lo, hi = args
    c = _Q["coords"]
    rows = _q_rows(lo, hi)
    delta = cdist(c[lo:hi], c)
    d = rows.astype(np.float64)
    np.fill_diagonal(d[:, lo:hi], np.inf)
    s_num = float((delta / d).sum())
    s_den = float((delta * delta / (d * d)).sum())
    jac = 0.0
    for i in range(hi - lo):
        v = lo + i
        hv = rows[i]
        hood = np.flatnonzero((hv >= 1) & (hv <= 2))
        q = hood.shape[0]
        if q == 0:
            jac += 1.0
            continue
        row = delta[i].copy()
        row[v] = np.inf
        nearest = np.argsort(row, kind="stable")[:q]
        inter = np.intersect1d(hood, nearest, assume_unique=True).shape[0]
        jac += inter / (2 * q - inter)
    return s_num, s_den, jac


def _q_chunk2(args):
    """metrics.py:115-131 (stress terms) for sources [lo, hi)."""
    from scipy.spatial.distance import cdist
    lo, hi, scale = args
    c = _Q["coords"]
    rows = _q_rows(lo, hi)
    delta = cdist(c[lo:hi], c) * scale
    d = rows.astype(np.float64)
    np.fill_diagonal(d[:, lo:hi], np.inf)
    term = (1.0 - delta / d) ** 2
    np.fill_diagonal(term[:, lo:hi], 0.0)
    return float(term.sum())


def _q_cross(args):
    """oracle.metrics.count_crossings (float filter + exact Fractions) for the
    pairs whose first edge lies in [i0, i1)."""
    from types import SimpleNamespace
    from oracle import metrics as OM
    return OM.count_crossings(SimpleNamespace(edges=_Q["edges"]), _Q["coords"], rows=args)


def gen_quality_c3_full(nseeds=5, procs=8):
    """Exact NP, stress and crossings (metrics.py:41-190 restated in
    oracle/metrics.py, chunked) of the reference's own c3 SL layouts, seeds
    0..nseeds-1 -- the reference side of the exact check (c) at c3.  Only the
    scalars are frozen."""
    import multiprocessing as mp
    import time
    sys.path.insert(0, ROOT)
    rg = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    n = rg.n
    indptr = np.ascontiguousarray(rg.adj_indptr, np.int64)
    indices = np.ascontiguousarray(rg.adj_indices, np.int32)
    edges = np.ascontiguousarray(rg.edges, np.int64)
    out = {"np_": [], "stress": [], "crossings": []}
    for seed in range(nseeds):
        t = time.time()
        _, kn = gu.partial_bfs(rg, 15, seed=seed)
        gk = gu.smooth_knn_weights(kn)
        E = gk.edge_count
        samp = math.log(0.1 * E) / math.log(E)
        lay = gu.optimize_sampled(gk, gu.random_init(rg, seed, 10.0),
                                  gu.OptimizerConfig(iterations=200, k=15, seed=seed, samp=samp))
        coords = np.ascontiguousarray(lay.coords, np.float64)
        chunks = [(lo, min(lo + 512, n)) for lo in range(0, n, 512)]
        with mp.get_context("fork").Pool(procs, _q_init, (indptr, indices, coords, edges)) as pool:
            parts = pool.map(_q_chunk, chunks)
            s_num = sum(p[0] for p in parts)
            s_den = sum(p[1] for p in parts)
            scale = s_num / s_den if s_den > 0 else 1.0
            st = sum(pool.map(_q_chunk2, [(lo, hi, scale) for lo, hi in chunks])) / (n * n - n)
            npv = sum(p[2] for p in parts) / n
            m = edges.shape[0]
            bounds = np.linspace(0, m, 4 * procs + 1).astype(int)
            cr = sum(pool.map(_q_cross, list(zip(bounds[:-1], bounds[1:]))))
        out["np_"].append(npv)
        out["stress"].append(st)
        out["crossings"].append(cr)
        print("quality c3 full seed", seed, npv, st, cr, f"{time.time() - t:.1f}s", flush=True)
        save("quality_c3_full.npz", np_=np.array(out["np_"]), stress=np.array(out["stress"]),
             crossings=np.array(out["crossings"], np.int64))


def gen_spectral():
    """spectral_init (layout.py:221-304) of the reference on graphs with n >
    512 (the Lanczos path): BA graphs (simple spectra: coordinates compared)
    and a grid (degenerate pairs: eigen-residual properties only)."""
    out = {}
    cases = [("ba700", F.scale_free(700, seed=5, m0=2), 0), ("ba1500", F.scale_free(1500, seed=6, m0=3), 3),
             ("grid900", F.grid(900), 1)]
    for name, g, seed in cases:
        n = g.n
        rg = gu.build_graph([tuple(map(int, e)) for e in g.edges])
        assert rg.n == n
        lay = gu.spectral_init(rg, seed=seed)
        out[name + "_coords"] = np.asarray(lay.coords)
        out[name + "_seed"] = np.array(seed)
        # reference eigenvalues of L_sym (dense) for the gap
        import scipy.sparse as sp
        deg = np.diff(rg.adj_indptr).astype(np.float64)
        A = sp.csr_matrix((np.ones(rg.adj_indices.shape[0]), rg.adj_indices, rg.adj_indptr), shape=(n, n))
        isq = 1.0 / np.sqrt(deg)
        lam = np.linalg.eigvalsh(np.eye(n) - (isq[:, None] * A.toarray()) * isq[None, :])
        out[name + "_lam"] = lam[:6]
        print(name, "lam", lam[:4])
    save("spectral.npz", **out)


def gen_spectral_c3():
    """spectral_init of the reference on BASELINE c3 (BA n=100k, m0=3, seed
    2; ARPACK, ~15 s here): coordinates (float32) and the three smallest
    eigenvalues of L_sym (eigsh on 2I - L, the reference's own operator), so
    the test can bound the coordinate difference by residual / gap."""
    import scipy.sparse as sp
    from scipy.sparse.linalg import eigsh
    g = F.scale_free(100000, seed=2, m0=3)
    rg = gu.build_graph([tuple(map(int, e)) for e in g.edges])
    assert rg.n == g.n
    lay = gu.spectral_init(rg, seed=2)
    n = rg.n
    deg = np.diff(rg.adj_indptr).astype(np.float64)
    A = sp.csr_matrix((np.ones(rg.adj_indices.shape[0]), rg.adj_indices, rg.adj_indptr), shape=(n, n))
    isq = sp.diags(1.0 / np.sqrt(deg))
    M = sp.identity(n) + isq @ A @ isq   # 2I - L_sym
    vals = eigsh(M, k=4, which="LM", tol=1e-10, return_eigenvectors=False)
    lam = np.sort(2.0 - vals)
    print("c3 lam", lam)
    save("spectral_c3.npz", coords=np.asarray(lay.coords, np.float32), seed=np.array(2), lam=lam)


def gen_sparsify():
    """sparsify.py:49-205 on dense graphs (m > n log2 n): the reference's exact
    resistances, its sparsifier's kept-edge mask, and its sketch resistances
    (numpy signs, for the statistical comparison)."""
    import importlib
    S = importlib.import_module("graph_umap.sparsify")
    out = {}
    cases = [("er300", F.erdos_renyi(300, avg_degree=30, seed=11)),
             ("er800", F.erdos_renyi(800, avg_degree=30, seed=12)),
             ("ba600", F.scale_free(600, seed=13, m0=12))]
    for name, g in cases:
        rg = gu.build_graph([tuple(map(int, e)) for e in g.edges])
        assert rg.n == g.n and rg.m == g.m and np.array_equal(rg.edges, g.edges)
        r = S.effective_resistance_exact(rg)
        sp_g = S.sparsify(rg, r)
        keys = set(map(tuple, sp_g.edges.tolist()))
        mask = np.array([tuple(e) in keys for e in rg.edges.tolist()])
        ra = S.effective_resistance_approx(rg, epsilon=0.5, seed=0)
        out[name + "_r"] = np.asarray(r.values)
        out[name + "_keep"] = mask
        out[name + "_r_approx"] = np.asarray(ra.values)
        print(name, rg.n, rg.m, "kept", mask.sum(), "target", S.sparsifier_target(rg.n, rg.m))
    save("sparsify.npz", **out)


def _c4_seed(args):
    """One reference c4 SSSL-style layout (random init, partial BFS kNN k=15,
    smooth weights, 200 windowed epochs at the default samp=0.9) and its
    sampled NP / stress over the fixed sources."""
    seed, edges_path, rows_path, src_path = args
    import time
    sys.path.insert(0, ROOT)
    from oracle.metrics import sampled_neighborhood_preservation, sampled_stress
    t = time.time()
    e = np.load(edges_path)
    rg = gu.build_graph([tuple(map(int, x)) for x in e])
    _, kn = gu.partial_bfs(rg, 15, seed=seed)
    gk = gu.smooth_knn_weights(kn)
    lay = gu.optimize_sampled(gk, gu.random_init(rg, seed, 10.0),
                              gu.OptimizerConfig(iterations=200, k=15, seed=seed))
    rows = np.load(rows_path, mmap_mode="r")  # 8 GB at c4: one page-cache copy for all workers
    src = np.load(src_path)
    out = (sampled_neighborhood_preservation(lay.coords, rows, src),
           sampled_stress(lay.coords, rows, src))
    print("quality c4 seed", seed, out, f"{time.time() - t:.0f}s", flush=True)
    return out


def gen_quality_c4(nseeds=5):
    """Check (c) at 1M scale: the reference's own c4 layouts (SBM 1M fixture,
    random init, partial BFS kNN, 200 epochs at samp 0.9), one process per
    seed; sampled NP / stress over 2000 fixed sources (oracle/metrics.py
    estimators, exact per-source terms).  Only the scalars are frozen."""
    import multiprocessing as mp
    import tempfile
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from oracle.metrics import sample_sources
    g = F.config_graph("c4")
    src = sample_sources(g.n)
    rows = O.all_pairs_bfs_rows(g, src)
    tmp = tempfile.mkdtemp()
    ep, rp, sp = (os.path.join(tmp, f) for f in ("edges.npy", "rows.npy", "src.npy"))
    np.save(ep, np.asarray(g.edges))
    np.save(rp, rows)
    np.save(sp, src)
    del rows, g
    with mp.get_context("spawn").Pool(nseeds) as pool:
        vals = pool.map(_c4_seed, [(s, ep, rp, sp) for s in range(nseeds)])
    v = np.array(vals)
    save("quality_c4.npz", np_=v[:, 0], stress=v[:, 1], sources=src)


def _c2_seed(args):
    """One reference c2 SS-GUMAP layout on the shared G' fixture (random
    init, all-pairs BFS kNN k=15, 200 full epochs)."""
    seed, edges_path, n = args
    import time
    t = time.time()
    e = np.load(edges_path)
    rg = gu.build_graph([tuple(map(int, x)) for x in e])
    assert rg.n == n
    dset = gu.all_pairs_bfs(rg)
    kn = gu.knn_from_full_distances(dset, 15, seed=seed)
    gk = gu.smooth_knn_weights(kn)
    lay = gu.optimize_full(gk, gu.random_init(rg, seed, 10.0),
                           gu.OptimizerConfig(iterations=200, k=15, seed=seed))
    print("quality c2 seed", seed, f"{time.time() - t:.0f}s", flush=True)
    return np.asarray(lay.coords, np.float64)


def gen_quality_c2(nseeds=5):
    """Check (c) at SS-GUMAP scale: the reference's own final layouts of c2
    (the G' fixture of ER(20000, 200), random init, 200 full epochs), seeds
    0..nseeds-1, one process each.  The layouts themselves are frozen (20k x 2
    float64 each): the GPU metrics -- pinned to the reference's own metric
    values on c1 -- then evaluate NP, stress and crossings on both sides."""
    import multiprocessing as mp
    import tempfile
    g = F.config_graph("c2")
    tmp = tempfile.mkdtemp()
    ep = os.path.join(tmp, "edges.npy")
    np.save(ep, np.asarray(g.edges))
    with mp.get_context("spawn").Pool(nseeds) as pool:
        lays = pool.map(_c2_seed, [(s, ep, g.n) for s in range(nseeds)])
    save("quality_c2.npz", layouts=np.stack(lays), n=np.array(g.n), m=np.array(g.m))

def _ingest_cases():
    """Inputs of the build_graph / largest_connected_component goldens
    (graph.py:132-232): the recipe is shared with tests/test_ingest.py."""
    rng = np.random.default_rng(303)
    cases = []
    # integers: non-contiguous ids, duplicates (both orientations), self loops
    ids = rng.choice(10**9, size=300, replace=False)
    pairs = [(int(ids[a]), int(ids[b])) for a, b in rng.integers(0, 300, size=(900, 2))]
    cases.append(("ints", pairs))
    cases.append(("strings", [("b", "a"), ("c", "b"), ("a", "b"), ("d", "d"), ("e", "f"),
                              ("f", "e"), ("zz", "a")]))
    # numeric strings sort as strings ("10" < "8" < "9")
    cases.append(("numeric_strings", [("10", "9"), ("9", "8"), ("8", "10"), ("100", "7"),
                                      ("7", "8")]))
    # floats keep their values: (1.5, 1.7) is an edge, not a self loop
    cases.append(("floats", [(1.5, 1.7), (1.7, 2.5), (2.5, 1.5), (0.25, 3.0), (3.0, 3.0)]))
    # several components of different sizes, a size tie for the runner-up
    comp = [(i, i + 1) for i in range(0, 9)] + [(20, 21), (21, 22), (30, 31), (31, 32),
                                                 (40, 41)]
    cases.append(("components", comp))
    return cases


def _ingest_tie_graph(gu_mod):
    """Two equal-size components whose smallest labels are NOT in vertex
    order: the reference's tie rule (graph.py:211-214) takes the component
    holding the smallest label (vertices 3..5, labels 10..12)."""
    edges = np.array([(0, 1), (1, 2), (3, 4), (4, 5)], np.int64)
    labels = (50, 51, 52, 10, 11, 12)
    if hasattr(gu_mod, "graph_from_edges"):
        return gu_mod.graph_from_edges(6, edges, labels=labels)
    from graph_umap.graph import _from_canonical, Graph
    n, m, ip, ix, e = _from_canonical(6, edges, labels)
    return Graph(n=n, m=m, adj_indptr=ip, adj_indices=ix, edges=e, labels=labels)


def _graph_json(g):
    return dict(n=int(g.n), m=int(g.m), edges=np.asarray(g.edges).tolist(),
                labels=list(g.labels), dropped_self_loops=int(g.dropped_self_loops),
                dropped_duplicates=int(g.dropped_duplicates),
                indptr=np.asarray(g.adj_indptr).tolist(),
                indices=np.asarray(g.adj_indices).tolist())


def gen_ingest():
    """build_graph / largest_connected_component outputs of the live
    reference (graph.py:132-232) for small label-typed inputs, a large
    integer input (the GPU build path; digests only) and the label tie."""
    from graph_umap.graph import largest_connected_component as ref_lcc
    out = {"cases": []}
    for name, pairs in _ingest_cases():
        g = gu.build_graph(pairs)
        out["cases"].append(dict(name=name, pairs=[list(p) for p in pairs], graph=_graph_json(g),
                                 lcc=_graph_json(ref_lcc(g))))
    tie = _ingest_tie_graph(gu)
    out["tie"] = dict(graph=_graph_json(tie), lcc=_graph_json(ref_lcc(tie)))
    # large integer input: 200k random pairs over 60k ids below 2^40 (many
    # components); the GPU build and LCC paths engage at this size
    rng = np.random.default_rng(404)
    idv = rng.choice(2**40, size=60000, replace=False)
    pairs = idv[rng.integers(0, 60000, size=(200000, 2))]
    g = gu.build_graph([(int(a), int(b)) for a, b in pairs])
    h = ref_lcc(g)
    out["large"] = dict(seed=404, nids=60000, npairs=200000, n=int(g.n), m=int(g.m),
                        dropped_self_loops=int(g.dropped_self_loops),
                        dropped_duplicates=int(g.dropped_duplicates),
                        edges_sha=sha(np.asarray(g.edges, np.int64)),
                        labels_sha=sha(np.asarray(g.labels, np.int64)),
                        lcc_n=int(h.n), lcc_m=int(h.m),
                        lcc_edges_sha=sha(np.asarray(h.edges, np.int64)),
                        lcc_labels_sha=sha(np.asarray(h.labels, np.int64)))
    path = os.path.join(HERE, "ingest.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, os.path.getsize(path), "bytes")


def main():
    # quality_c3_full (~1.5 h on 8 cores) runs only when named
    which = sys.argv[1:] or ["partial_small", "full_small", "smooth_cases", "c1", "c3", "quality_c1",
                             "quality_c3", "spectral", "sparsify"]
    for w in which:
        globals()["gen_" + w]()
    manifest = dict(numpy=np.__version__, scipy=scipy.__version__, numba=numba.__version__,
                    python=sys.version.split()[0], reference="/root/reference/pkg (graph_umap 0.1.0)")
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main()
