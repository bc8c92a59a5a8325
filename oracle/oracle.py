"""CPU oracle for the graph_umap hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / CPU baseline.  The product package
``paper_2509_19703_b200`` never imports it.

The integer / RNG work runs in ``oracle.c`` (compiled by ``oracle/Makefile``
into ``oracle/_build/liboracle.so``); the float64 weight formula and the fuzzy
union are restated here in numpy so that ``exp`` is numpy's own (bit-identical
weights to the reference).  Each function cites the reference routine it
restates (paths relative to /root/reference/pkg/src/graph_umap).

Pinning: tests/test_oracle.py checks every function here against golden
vectors produced by the live reference (tests/golden/make_golden.py).
"""

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

INF32 = 2**31 - 1
SPLIT_GAMMA = 0x9E3779B97F4A7C15

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, u64, f64, cint = (ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                                    ctypes.c_double, ctypes.c_int)
        L.or_apsp_rows.argtypes = [i64, _i64p, _i32p, _i64p, i64, _i32p, cint]
        L.or_partial_bfs_all.argtypes = [i64, _i64p, _i32p, i32, u64, i64, i64,
                                         _i32p, _i32p, _i32p, _i64p, _i64p, cint]
        L.or_numpy_permutation.argtypes = [u64, u64, i64, _i64p]
        L.or_knn_from_matrix.argtypes = [i64, _i32p, i32, u64, _i32p, _i32p, _i32p, cint]
        L.or_full_knn.argtypes = [i64, _i64p, _i32p, i32, u64, i64, i64, _i32p,
                                  _i32p, _i32p, cint]
        L.or_smooth_rows.argtypes = [i64, _i64p, _i32p, i64, f64, _f64p, _f64p,
                                     _f64p, cint]
        L.or_sgd_sweep.argtypes = [_f64p, i64, _i32p, _i32p, _f64p, _i64p, i64,
                                   _i64p, _i32p, f64, f64, f64, i32, _u64p,
                                   _i32p, _f64p]
        L.or_sgd_replay.argtypes = [_f64p, _i32p, _i32p, _f64p, _i64p, i64, _i32p,
                                    _f64p, f64, f64, f64, i32]
        L.or_fuzzy_union.argtypes = [i64, _i64p, _i32p, _f64p, _i32p, _i32p, _f64p,
                                     _i64p, cint]
        L.or_fuzzy_union.restype = i64
        L.or_max_threads.restype = cint
        _lib = L
    return _lib


def _p(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def max_threads():
    return int(lib().or_max_threads())


def _csr(g):
    ip = np.ascontiguousarray(g.adj_indptr, dtype=np.int64)
    ix = np.ascontiguousarray(g.adj_indices, dtype=np.int32)
    return ip, ix


# ----------------------------------------------------------------- C0 full
def all_pairs_bfs(g, nthreads=1):
    """neighbors.py:120-134 / _kernels.py:33-57 -> int32 (n, n) matrix."""
    return all_pairs_bfs_rows(g, np.arange(int(g.n)), nthreads)


def all_pairs_bfs_rows(g, sources, nthreads=None):
    """The rows of all_pairs_bfs for ``sources`` only (int32, INF32 unreachable)."""
    ip, ix = _csr(g)
    n = int(g.n)
    src = np.ascontiguousarray(sources, dtype=np.int64)
    out = np.empty((len(src), n), dtype=np.int32)
    lib().or_apsp_rows(n, _p(ip, _i64p), _p(ix, _i32p), _p(src, _i64p), len(src),
                       _p(out, _i32p), max_threads() if nthreads is None else nthreads)
    return out


def numpy_permutation(seed, key, T):
    """default_rng(SeedSequence(entropy=seed, spawn_key=(key,))).permutation(T)."""
    out = np.empty(T, dtype=np.int64)
    lib().or_numpy_permutation(int(seed), int(key), int(T), _p(out, _i64p))
    return out


def _pack(n, k, dst, dist, counts):
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    if k == 0:
        return indptr, np.empty(0, np.int32), np.empty(0, np.int32)
    mask = np.arange(k)[None, :] < counts[:, None]
    return indptr, dst.reshape(n, k)[mask], dist.reshape(n, k)[mask]


def knn_from_full_distances(matrix, k, seed=0, nthreads=1):
    """neighbors.py:183-237 -> (indptr int64, dst int32, dist int32)."""
    n = matrix.shape[0]
    m = np.ascontiguousarray(matrix, dtype=np.int32)
    dst = np.zeros(n * k, np.int32)
    dist = np.zeros(n * k, np.int32)
    cnt = np.zeros(n, np.int32)
    lib().or_knn_from_matrix(n, _p(m, _i32p), k, int(seed), _p(dst, _i32p),
                             _p(dist, _i32p), _p(cnt, _i32p), nthreads)
    return _pack(n, k, dst, dist, cnt)


def full_knn(g, k, seed=0, src_begin=0, src_end=None, nthreads=1, packed=True):
    """all_pairs_bfs + knn_from_full_distances fused per source (no n x n)."""
    ip, ix = _csr(g)
    n = int(g.n)
    src_end = n if src_end is None else src_end
    ns = src_end - src_begin
    dst = np.zeros(ns * k, np.int32)
    dist = np.zeros(ns * k, np.int32)
    cnt = np.zeros(ns, np.int32)
    lib().or_full_knn(n, _p(ip, _i64p), _p(ix, _i32p), k, int(seed), src_begin,
                      src_end, _p(dst, _i32p), _p(dist, _i32p), _p(cnt, _i32p),
                      nthreads)
    if not packed:
        return dst, dist, cnt
    return _pack(ns, k, dst, dist, cnt)


# -------------------------------------------------------------- C0 partial
def partial_bfs_raw(g, k_eff, seed=0, src_begin=0, src_end=None, nthreads=1,
                    work=False):
    """_kernels.py:60-131 on sources [src_begin, src_end): fixed-stride rows."""
    ip, ix = _csr(g)
    n = int(g.n)
    src_end = n if src_end is None else src_end
    ns = src_end - src_begin
    kk = max(k_eff, 1)
    nbr = np.zeros(ns * kk, np.int32)
    dist = np.zeros(ns * kk, np.int32)
    cnt = np.zeros(ns, np.int32)
    sc = np.zeros(ns, np.int64) if work else None
    ex = np.zeros(ns, np.int64) if work else None
    if k_eff > 0:
        lib().or_partial_bfs_all(n, _p(ip, _i64p), _p(ix, _i32p), k_eff,
                                 int(seed) & (2**64 - 1), src_begin, src_end,
                                 _p(nbr, _i32p), _p(dist, _i32p), _p(cnt, _i32p),
                                 _p(sc, _i64p), _p(ex, _i64p), nthreads)
    if work:
        return nbr, dist, cnt, sc, ex
    return nbr, dist, cnt


def partial_bfs(g, k, seed=0, nthreads=1):
    """neighbors.py:137-180 -> (indptr, dst, dist), k_eff = min(k, n-1)."""
    n = int(g.n)
    k_eff = min(k, n - 1) if n > 1 else 0
    nbr, dist, cnt = partial_bfs_raw(g, k_eff, seed, nthreads=nthreads)
    return _pack(n, k_eff, nbr, dist, cnt)


# ------------------------------------------------------------------- C1
def smooth_rho_sigma(indptr, dist, k, nthreads=1):
    """neighbors.py:261-307: rho, sigma (float64, bisection restated in C)."""
    n = indptr.shape[0] - 1
    counts = np.diff(indptr)
    if np.any(counts < 1):
        raise ValueError("every vertex needs at least one outgoing kNN edge")
    kmax = int(counts.max())
    rho = np.empty(n)
    sigma = np.empty(n)
    ip = np.ascontiguousarray(indptr, np.int64)
    dd = np.ascontiguousarray(dist, np.int32)
    lib().or_smooth_rows(n, _p(ip, _i64p), _p(dd, _i32p), kmax, float(np.log2(k)),
                         _p(rho, _f64p), _p(sigma, _f64p), None, nthreads)
    return rho, sigma


def directed_weights(indptr, dist, rho, sigma):
    """neighbors.py:309-318 with numpy's exp: w = exp(-(d - rho) / sigma)."""
    counts = np.diff(indptr)
    rows = np.repeat(np.arange(indptr.shape[0] - 1), counts)
    d = dist.astype(np.float64)
    return np.exp(-(d - rho[rows]) / sigma[rows])


def fuzzy_union_symmetrize(n, indptr, dst, w):
    """neighbors.py:320-350 as a sort-based union (no scipy).

    Dedupe (first occurrence), h = (a + b) - a*b over both orientations with a
    missing orientation counted as 0, drop exact zeros, lexsort by (src, dst).
    """
    counts = np.diff(indptr)
    rows = np.repeat(np.arange(n, dtype=np.int64), counts)
    cols = dst.astype(np.int64)
    keys = rows * n + cols
    _, first = np.unique(keys, return_index=True)
    rows, cols, vals = rows[first], cols[first], w[first]
    fk = rows * n + cols          # forward keys (sorted, unique)
    bk = cols * n + rows          # the same weights seen from the other end
    allk = np.union1d(fk, bk)
    a = np.zeros(allk.shape[0])
    b = np.zeros(allk.shape[0])
    a[np.searchsorted(allk, fk)] = vals
    b[np.searchsorted(allk, bk)] = vals
    h = (a + b) - a * b
    keep = h != 0.0
    allk, h = allk[keep], h[keep]
    src = (allk // n).astype(np.int32)
    dstc = (allk % n).astype(np.int32)
    nbr_indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=nbr_indptr[1:])
    return src, dstc, h.astype(np.float64), nbr_indptr, dstc.copy()


def fuzzy_union_c(n, indptr, dst, w, nthreads=None):
    """neighbors.py:320-350 in C (oracle.c or_fuzzy_union): the same result as
    fuzzy_union_symmetrize (pinned against it in tests/test_oracle.py), in
    O(nnz) per-vertex merges instead of global numpy sorts -- what makes the
    full-size C1 parity tests (c4, c5) affordable."""
    ip = np.ascontiguousarray(indptr, np.int64)
    dd = np.ascontiguousarray(dst, np.int32)
    ww = np.ascontiguousarray(w, np.float64)
    nt = max_threads() if nthreads is None else nthreads
    E = lib().or_fuzzy_union(n, _p(ip, _i64p), _p(dd, _i32p), _p(ww, _f64p), None, None,
                             None, None, nt)
    src = np.empty(E, np.int32)
    dstc = np.empty(E, np.int32)
    h = np.empty(E, np.float64)
    nip = np.empty(n + 1, np.int64)
    lib().or_fuzzy_union(n, _p(ip, _i64p), _p(dd, _i32p), _p(ww, _f64p), _p(src, _i32p),
                         _p(dstc, _i32p), _p(h, _f64p), _p(nip, _i64p), nt)
    return src, dstc, h, nip, dstc.copy()


def smooth_knn_weights(n, indptr, dst, dist, k, nthreads=1, union="numpy"):
    """neighbors.py:245-350 -> dict of the KnnGraph arrays.  union="c" takes
    the C restatement of the fuzzy union (same arrays, much faster)."""
    rho, sigma = smooth_rho_sigma(indptr, dist, k, nthreads)
    w = directed_weights(indptr, dist, rho, sigma)
    if union == "c":
        s, d, h, nip, nix = fuzzy_union_c(n, indptr, dst, w, nthreads)
    else:
        s, d, h, nip, nix = fuzzy_union_symmetrize(n, indptr, dst, w)
    return dict(rho=rho, sigma=sigma, w=w, sym_src=s, sym_dst=d, sym_w=h,
                nbr_indptr=nip, nbr_indices=nix)


# ------------------------------------------------------------------- C2
def sgd_sweep(coords, sym_src, sym_dst, sym_w, order, nbr_indptr, nbr_indices,
              a, b, lr, n_neg, state, log=True):
    """_kernels.py:158-223 in place on float64 coords; returns (state, negs, thetas)."""
    n = coords.shape[0]
    order = np.ascontiguousarray(order, np.int64)
    st = np.array([state], dtype=np.uint64)
    negs = np.empty(order.shape[0] * n_neg, np.int32) if log else None
    th = np.empty(order.shape[0] * n_neg, np.float64) if log else None
    lib().or_sgd_sweep(_p(coords, _f64p), n, _p(sym_src, _i32p), _p(sym_dst, _i32p),
                       _p(sym_w, _f64p), _p(order, _i64p), order.shape[0],
                       _p(nbr_indptr, _i64p), _p(nbr_indices, _i32p), a, b, lr,
                       n_neg, _p(st, _u64p), _p(negs, _i32p), _p(th, _f64p))
    return int(st[0]), negs, th


def sgd_replay(coords, sym_src, sym_dst, sym_w, order, negs, thetas, a, b, lr,
               n_neg):
    order = np.ascontiguousarray(order, np.int64)
    lib().or_sgd_replay(_p(coords, _f64p), _p(sym_src, _i32p), _p(sym_dst, _i32p),
                        _p(sym_w, _f64p), _p(order, _i64p), order.shape[0],
                        _p(negs, _i32p), _p(thetas, _f64p), a, b, lr, n_neg)


def run_sgd(gk, coords0, iterations, a, b, learning_rate=1.0, n_neg=5, seed=0,
            samp=0.9, windowed=False, epochs_to_log=()):
    """layout.py:314-360 (_run_sgd) with logging of selected epochs.

    gk: dict with sym_src/sym_dst/sym_w/nbr_indptr/nbr_indices.
    Returns (coords, logs) where logs[it] = (coords_before, order, negs, thetas, lr).
    """
    coords = np.array(coords0, dtype=np.float64, copy=True, order="C")
    E = gk["sym_src"].shape[0]
    logs = {}
    t = iterations
    if t == 0 or E == 0:
        return coords, logs
    shuffle_rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(29,)))
    state = (int(seed) ^ SPLIT_GAMMA) & (2**64 - 1)
    if windowed:
        base_order = shuffle_rng.permutation(E)
        window = max(1, int(math.floor(E ** samp)))
        j = 0
    for it in range(t):
        lr = learning_rate * (1.0 - it / t)
        if windowed:
            order = base_order[(j + np.arange(window)) % E]
            j = (j + window) % E
        else:
            order = shuffle_rng.permutation(E)
        before = coords.copy() if it in epochs_to_log else None
        state, negs, th = sgd_sweep(coords, gk["sym_src"], gk["sym_dst"], gk["sym_w"],
                                    order, gk["nbr_indptr"], gk["nbr_indices"], a, b,
                                    lr, n_neg, state, log=it in epochs_to_log)
        if not np.all(np.isfinite(coords)):
            raise FloatingPointError(f"diverged at iteration {it}")
        if it in epochs_to_log:
            logs[it] = (before, order.copy(), negs, th, lr)
    return coords, logs
