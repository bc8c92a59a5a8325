"""C0/C1 drop-in: BFS distances, kNN selection, fuzzy weights (B200 path).

Same names, signatures, return types and error behaviour as
/root/reference/pkg/src/graph_umap/neighbors.py:
  all_pairs_bfs(g, chunk=1024)              neighbors.py:120-134
  partial_bfs(g, k, seed=0)                 neighbors.py:137-180
  knn_from_full_distances(dset, k, seed=0)  neighbors.py:183-237
  smooth_knn_weights(knn, k=None)           neighbors.py:245-350
  fuzzy_union(a, b)                         neighbors.py:240-242
Behind them every array operation runs in libgumap.so on the GPU; results
stay resident as device tensors and are copied to numpy only when a numpy
attribute (``dst``, ``matrix``, ``sym_w`` ...) is first read, so a pipeline
(partial_bfs -> smooth_knn_weights -> optimize_*) never round-trips through
the host.  The full-distance set returned by ``all_pairs_bfs`` is lazy: its
n x n ``matrix`` is only materialised if someone reads it;
``knn_from_full_distances`` on such a set runs the fused bitset BFS-kNN
kernel instead.
"""

import warnings

import numpy as np
import torch

from . import _lib
from .device import to_host_into, device_csr, require_cuda, stream_ptr, to_device, to_host, workspace

#: sentinel hop distance for unreachable pairs (neighbors.py:17-18)
UNREACHABLE = 2**31 - 1
INF32 = UNREACHABLE
SMOOTH_TOLERANCE = 1e-5
SIGMA_MIN = 1e-3
SIGMA_MAX = 1e3
SMOOTH_ITERATIONS = 64

# tier-2 scratch budget of the partial BFS (per-warp n-int slots)
_TIER2_BUDGET_BYTES = 256 << 20


class _LazyArrays:
    """Holds numpy arrays and/or device tensors; converts on first access."""

    _host_dtypes = {}

    def _init_lazy(self, host, dev):
        object.__setattr__(self, "_host", dict(host))
        object.__setattr__(self, "_dev", dict(dev))
        object.__setattr__(self, "_pending", {})  # name -> (pinned tensor, waiter)
        object.__setattr__(self, "_pending_bytes", None)

    def _get_host(self, name):
        h = self._host.get(name)
        if h is None and name in self._pending:
            pinned, ev = self._pending.pop(name)
            ev.synchronize()
            h = pinned.numpy()
            h.setflags(write=False)
            self._host[name] = h
        if h is None:
            d = self._dev.get(name)
            if d is None:
                return None
            h = to_host(d).astype(self._host_dtypes[name], copy=False)
            h.setflags(write=False)
            self._host[name] = h
        return h

    def device(self, name, device=None):
        """Device tensor of array ``name`` (uploads a host array once)."""
        d = self._dev.get(name)
        if d is None:
            h = self._host.get(name)
            if h is None:
                return None
            device = require_cuda(device)
            d = to_device(h, self._host_dtypes[name], device)
            self._dev[name] = d
        return d


class SparseDistanceSet(_LazyArrays):
    """Hop distances from every vertex, full (n x n) or truncated (neighbors.py:26-49)."""

    _host_dtypes = {"matrix": np.int32, "indptr": np.int64, "nbr": np.int32, "dist": np.int32}

    def __init__(self, n, full, matrix=None, indptr=None, nbr=None, dist=None, *, _graph=None,
                 _dev=None, _chunk=1024):
        self.n = int(n)
        self.full = bool(full)
        self._init_lazy(dict(matrix=matrix, indptr=indptr, nbr=nbr, dist=dist), _dev or {})
        object.__setattr__(self, "_graph", _graph)
        object.__setattr__(self, "_chunk", int(_chunk))

    @property
    def matrix(self):
        if not self.full:
            return None
        m = self._host.get("matrix")
        if m is None and self._graph is not None:
            m = _apsp_matrix(self._graph, self._chunk)
            m.setflags(write=False)
            self._host["matrix"] = m
        return m

    @property
    def indptr(self):
        return self._get_host("indptr")

    @property
    def nbr(self):
        return self._get_host("nbr")

    @property
    def dist(self):
        return self._get_host("dist")

    def run_bfs(self, k, seed=0):
        """Run the BFS of a lazy full set now, for a later
        ``knn_from_full_distances(self, k, seed)``: the fused bitset BFS with
        its per-source k-th-distance selection, records kept on the device.
        The drivers call it inside the C0 bracket (reference layout.py:418-420
        times all_pairs_bfs as C0), so C1 is the packing, the weights and the
        union, as in the reference."""
        g = self._graph
        if not self.full or g is None or k < 1:
            return
        dev = require_cuda()
        recs = full_knn_records(device_csr(g, dev), k, seed, 0, self.n)
        self.__dict__.setdefault("_knn_records", {})[(int(k), int(seed))] = recs

    def _take_records(self, k, seed):
        return self.__dict__.get("_knn_records", {}).pop((int(k), int(seed)), None)

    def row(self, v):
        """(neighbor ids, hop distances) for vertex ``v``, excluding ``v``."""
        if self.full:
            d = self.matrix[v]
            ids = np.flatnonzero((d != INF32) & (np.arange(self.n) != v))
            return ids, d[ids]
        lo, hi = self.indptr[v], self.indptr[v + 1]
        return self.nbr[lo:hi], self.dist[lo:hi]


class DirectedKnn(_LazyArrays):
    """Directed kNN edges grouped by source (neighbors.py:52-64)."""

    _host_dtypes = {"indptr": np.int64, "dst": np.int32, "dist": np.int32}

    def __init__(self, n, k, indptr=None, dst=None, dist=None, *, _dev=None):
        self.n = int(n)
        self.k = int(k)
        self._init_lazy(dict(indptr=None if indptr is None else np.asarray(indptr),
                             dst=None if dst is None else np.asarray(dst),
                             dist=None if dist is None else np.asarray(dist)), _dev or {})

    indptr = property(lambda self: self._get_host("indptr"))
    dst = property(lambda self: self._get_host("dst"))
    dist = property(lambda self: self._get_host("dist"))

    @property
    def edge_count(self):
        d = self._dev.get("dst")
        return int(d.shape[0]) if d is not None else int(self.dst.shape[0])

    def __repr__(self):
        return f"DirectedKnn(n={self.n}, k={self.k}, edges={self.edge_count})"


class KnnGraph(_LazyArrays):
    """Raw directed kNN edges plus the symmetrised fuzzy ones (neighbors.py:67-101)."""

    _host_dtypes = {"rho": np.float64, "sigma": np.float64, "sym_src": np.int32,
                    "sym_dst": np.int32, "sym_w": np.float64, "nbr_indptr": np.int64,
                    "nbr_indices": np.int32, "w": np.float64}

    def __init__(self, n, k, directed, rho=None, sigma=None, sym_src=None, sym_dst=None,
                 sym_w=None, nbr_indptr=None, nbr_indices=None, *, _dev=None):
        self.n = int(n)
        self.k = int(k)
        self.directed = directed
        self._init_lazy(dict(rho=rho, sigma=sigma, sym_src=sym_src, sym_dst=sym_dst,
                             sym_w=sym_w, nbr_indptr=nbr_indptr, nbr_indices=nbr_indices),
                        _dev or {})

    rho = property(lambda self: self._get_host("rho"))
    sigma = property(lambda self: self._get_host("sigma"))
    sym_src = property(lambda self: self._get_host("sym_src"))
    sym_dst = property(lambda self: self._get_host("sym_dst"))
    sym_w = property(lambda self: self._get_host("sym_w"))
    nbr_indptr = property(lambda self: self._get_host("nbr_indptr"))
    nbr_indices = property(lambda self: self._get_host("nbr_indices"))

    @property
    def edge_count(self):
        """Number of directed symmetrised edges (what the optimizers see)."""
        d = self._dev.get("sym_src")
        return int(d.shape[0]) if d is not None else int(self.sym_src.shape[0])

    def undirected_edges(self):
        """(u, v, d, h) arrays with u < v, one row per symmetrised pair
        (neighbors.py:94-117; the raw-distance join is vectorised)."""
        mask = self.sym_src < self.sym_dst
        u = self.sym_src[mask]
        v = self.sym_dst[mask]
        h = self.sym_w[mask]
        d = _join_raw_distances(self.directed, u, v)
        return u, v, d, h


def _join_raw_distances(directed, u, v):
    """Raw hop distance for each (u, v) pair from either orientation, the
    first occurrence in (source, position) order winning (neighbors.py:104-117)."""
    n = directed.n
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(directed.indptr))
    dst = directed.dst.astype(np.int64)
    lo, hi = np.minimum(src, dst), np.maximum(src, dst)
    keys = lo * n + hi
    uk, first = np.unique(keys, return_index=True)
    vals = directed.dist[first]
    q = np.asarray(u, np.int64) * n + np.asarray(v, np.int64)
    idx = np.searchsorted(uk, q)
    if np.any(idx >= uk.shape[0]) or np.any(uk[np.minimum(idx, uk.shape[0] - 1)] != q):
        raise KeyError("pair without a raw kNN distance")
    return vals[idx].astype(np.int32)


def fuzzy_union(a, b):
    """Probabilistic t-conorm a + b - a*b used to symmetrise directed weights."""
    return a + b - a * b


# ------------------------------------------------------------------ C0 full
# device row budget of one all_pairs_bfs call (the rows of up to 296 64-source
# batches at once keep every CTA slot busy; the reference's `chunk` is a host
# processing granularity and does not bound the GPU batch)
_APSP_ROW_BUDGET = 8 << 30


def _apsp_matrix(g, chunk=1024):
    """int32 (n, n) hop distances: GPU bitset BFS over as many sources per
    call as the row budget holds, copied back through pinned staging."""
    dev = require_cuda()
    csr = device_csr(g, dev)
    n = csr.n
    out = np.empty((n, n), dtype=np.int32)
    if n == 0:
        return out
    full = ((n + 63) // 64) * 64
    rows_per = min(full, max(64, (_APSP_ROW_BUDGET // (4 * n)) // 64 * 64))
    bif = max(1, min(148 * 2, rows_per // 64))
    ws = workspace(_lib.load().gu_full_bfs_workspace_size(n, 0, bif), dev)
    rows = torch.empty((rows_per, n), dtype=torch.int32, device=dev)
    for start in range(0, n, rows_per):
        stop = min(start + rows_per, n)
        _lib.call("gu_apsp_rows", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), start, stop,
                  _lib.ptr(rows), _lib.ptr(ws), ws.numel(), bif, stream_ptr(dev))
        to_host_into(rows[: stop - start], out[start:stop])
    return out


def all_pairs_bfs(g, chunk=1024):
    """Hop distances between all ordered pairs (the O(nm) baseline C0).

    Unreachable pairs receive the :data:`UNREACHABLE` sentinel.  The n x n
    matrix is produced on first access to ``.matrix`` (GPU bitset BFS, in
    ``chunk``-source slices); ``knn_from_full_distances`` never needs it.
    """
    require_cuda()
    return SparseDistanceSet(n=g.n, full=True, _graph=g, _chunk=chunk)


# --------------------------------------------------------------- records
def _pack(n_rows, k, rec_nbr, rec_dist, rec_cnt, dev, full=None, indptr=None):
    """Fixed-stride records -> (indptr int64, dst int32, dist int32) on device.

    When every row is full (``full``; computed if None) the records already
    are the packed CSR and the indptr is k * arange (``indptr`` when given)."""
    total_max = n_rows * k
    if full is None:
        full = bool(total_max) and bool((rec_cnt == k).all())
    if total_max and full:
        if indptr is None:
            indptr = torch.arange(0, (n_rows + 1) * k, k, dtype=torch.int64, device=dev)
        return indptr, rec_nbr.reshape(-1)[:total_max], rec_dist.reshape(-1)[:total_max]
    indptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    ws = workspace(_lib.load().gu_pack_records_workspace_size(n_rows), dev)
    dst = torch.empty(max(total_max, 1), dtype=torch.int32, device=dev)
    dist = torch.empty(max(total_max, 1), dtype=torch.int32, device=dev)
    _lib.call("gu_pack_records", n_rows, k, _lib.ptr(rec_nbr), _lib.ptr(rec_dist),
              _lib.ptr(rec_cnt), _lib.ptr(indptr), _lib.ptr(dst), _lib.ptr(dist),
              _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    total = int(indptr[-1].item())
    return indptr, dst[:total], dist[:total]


def _warn_short(short, stacklevel=3):
    if short:
        warnings.warn(
            f"{short} vertices live in components smaller than k+1; "
            "returning all reachable vertices for them",
            stacklevel=stacklevel,
        )


def _tier2_warps(n):
    return int(max(1, min(148 * 8, _TIER2_BUDGET_BYTES // max(8 * n, 1))))


def partial_bfs_records(csr, k_eff, seed, src_begin, src_end, work=None, tier2_warps=None,
                        out=None, ws=None):
    """Raw fixed-stride records of sources [src_begin, src_end) (device).

    Returns (nbr int32[ns, k], dist int32[ns, k], count int32[ns]), written
    into ``out`` when given.  ``work``: optional int64[2] device tensor
    receiving (entries scanned, vertices expanded)."""
    dev = csr.device
    ns = src_end - src_begin
    kk = max(k_eff, 1)
    if out is None:
        nbr = torch.empty((ns, kk), dtype=torch.int32, device=dev)
        dist = torch.empty((ns, kk), dtype=torch.int32, device=dev)
        cnt = torch.empty(ns, dtype=torch.int32, device=dev)
    else:
        nbr, dist, cnt = out
    n = csr.n
    if tier2_warps is None:
        tier2_warps = _tier2_warps(n)
    lib = _lib.load()
    if ws is None:
        ws = workspace(lib.gu_partial_bfs_workspace_size(n, ns, tier2_warps), dev)
    _lib.call("gu_partial_bfs_knn", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), k_eff,
              int(seed) & (2**64 - 1), src_begin, src_end, _lib.ptr(nbr), _lib.ptr(dist),
              _lib.ptr(cnt), _lib.ptr(work), _lib.ptr(ws), ws.numel(), tier2_warps,
              stream_ptr(dev))
    return nbr, dist, cnt


def full_knn_records(csr, k, seed, src_begin, src_end, work=None, batches_in_flight=None,
                     out=None):
    """Fused full-BFS kNN records of sources [src_begin, src_end) (device),
    written into ``out`` when given."""
    dev = csr.device
    ns = src_end - src_begin
    kk = max(k, 1)
    if out is None:
        nbr = torch.empty((ns, kk), dtype=torch.int32, device=dev)
        dist = torch.empty((ns, kk), dtype=torch.int32, device=dev)
        cnt = torch.empty(ns, dtype=torch.int32, device=dev)
    else:
        nbr, dist, cnt = out
    n = csr.n
    lib = _lib.load()
    if batches_in_flight is None:
        per = lib.gu_full_bfs_workspace_size(n, k, 1)
        batches_in_flight = int(max(1, min(148 * 2, (1 << 30) // max(per, 1), (ns + 63) // 64)))
    ws = workspace(lib.gu_full_bfs_workspace_size(n, k, batches_in_flight), dev)
    _lib.call("gu_full_bfs_knn", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), k,
              int(seed) & (2**64 - 1), src_begin, src_end, _lib.ptr(nbr), _lib.ptr(dist),
              _lib.ptr(cnt), _lib.ptr(work), _lib.ptr(ws), ws.numel(), batches_in_flight,
              stream_ptr(dev))
    return nbr, dist, cnt


# --------------------------------------------------------------- C0 partial
def partial_bfs(g, k, seed=0):
    """Truncated BFS per vertex: the k hop-nearest others, with distances.

    Bit-identical to neighbors.py:137-180 (ties at the stopping level broken
    by the reference's per-vertex splitmix64 streams).  Returns the partial
    distance set together with the directed kNN edges it implies.  Vertices
    whose component holds fewer than k+1 vertices report everything
    reachable, with a warning.

    The sources run in chunks; each chunk's rows are copied into pinned host
    memory on a side stream while the next chunk computes, so the numpy
    results (``knn.dst`` ...) are ready shortly after the kernel.
    """
    if k < 1:
        raise ValueError("k must be >= 1")
    dev = require_cuda()
    n = int(g.n)
    k_eff = min(k, n - 1) if n > 1 else 0
    csr = device_csr(g, dev)
    kk = max(k_eff, 1)
    nbr = torch.empty((n, kk), dtype=torch.int32, device=dev)
    dist = torch.empty((n, kk), dtype=torch.int32, device=dev)
    cnt = torch.empty(n, dtype=torch.int32, device=dev)
    # rows cross PCIe as int32 ids and (hop distances <= k) uint8 distances
    prefetch = (_HostPrefetch(dev, n * kk, ("dst", "dist"), narrow=("dist",) if kk <= 255 else ())
                if n * kk * 8 >= (64 << 20) else None)
    ip_full = None
    if prefetch is not None:
        # small first chunks, so the row copies start early; the indptr of
        # the all-rows-full outcome goes down during the first kernel and is
        # used when no row turns out short
        bounds = sorted({0, n // 16, n // 4, n // 2, (3 * n) // 4, (15 * n) // 16, n})
        ip_full = torch.arange(0, (n + 1) * kk, kk, dtype=torch.int64, device=dev)
        prefetch.copy_extra("indptr", ip_full)
    else:
        bounds = [0, n]
    tw = _tier2_warps(n)
    most = max(e - b for b, e in zip(bounds[:-1], bounds[1:]))
    ws = workspace(_lib.load().gu_partial_bfs_workspace_size(n, most + 1, tw), dev)
    for b, e in zip(bounds[:-1], bounds[1:]):
        partial_bfs_records(csr, k_eff, seed, b, e, tier2_warps=tw, out=(nbr[b:e], dist[b:e], cnt[b:e]),
                            ws=ws)
        if prefetch is not None:
            prefetch.copy_rows(dict(dst=nbr, dist=dist), b * kk, e * kk)
    short = int((cnt < k_eff).sum().item()) if n else 0
    _warn_short(short)
    full = short == 0 and k_eff > 0
    indptr, dst, dd = _pack(n, k_eff, nbr, dist, cnt, dev, full=full,
                            indptr=ip_full if full else None)
    host = {}
    if prefetch is not None and short == 0:
        host = prefetch.finish()  # rows are the packed arrays: host copies are valid
    devd = dict(indptr=indptr, nbr=dst, dist=dd)
    dset = SparseDistanceSet(n=n, full=False, _dev=devd)
    knn = DirectedKnn(n=n, k=k, _dev=dict(indptr=indptr, dst=dst, dist=dd))
    for name, pend in host.items():
        knn._pending[name] = pend
        dset._pending["nbr" if name == "dst" else name] = pend
    if host:
        # bytes that crossed PCIe for the host arrays (narrowed rows count as
        # sent); reported by bench.py's e2e line
        object.__setattr__(knn, "_pending_bytes", sum(
            t.numel() * (1 if nm in prefetch.narrow else t.element_size()) for nm, (t, _) in host.items()))
    return dset, knn


_WIDEN_POOL = None


def _widen_pool():
    """Host threads that widen narrowed row copies (numpy releases the GIL in
    casting copies; torch releases it in Event.synchronize)."""
    global _WIDEN_POOL
    if _WIDEN_POOL is None:
        import concurrent.futures
        import os
        workers = int(os.environ.get("GU_WIDEN_THREADS", 0)) or max(1, (os.cpu_count() or 1) - 2)
        _WIDEN_POOL = concurrent.futures.ThreadPoolExecutor(max_workers=workers)
    return _WIDEN_POOL


class _Waiter:
    """Completion of a pending host array: a CUDA event and/or host futures."""

    def __init__(self, event=None, futures=()):
        self.event = event
        self.futures = list(futures)

    def synchronize(self):
        if self.event is not None:
            self.event.synchronize()
        for f in self.futures:
            f.result()


class _HostPrefetch:
    """Asynchronous device -> pinned-host copies of row ranges on a side
    stream, ordered after the compute stream's work so far.

    Arrays named in ``narrow`` (small non-negative ints, e.g. hop distances
    <= k <= 255) cross PCIe as uint8 -- a quarter of the bytes -- and are
    widened back to int32 by host threads as each range lands, overlapping
    the remaining copies."""

    _streams = {}

    def __init__(self, dev, numel, names, narrow=()):
        self.dev = dev
        self.stream = self._streams.setdefault(str(dev), torch.cuda.Stream(device=dev))
        self.host = {nm: torch.empty(numel, dtype=torch.int32, pin_memory=True) for nm in names}
        self.narrow = {nm: (torch.empty(numel, dtype=torch.uint8, device=dev),
                            torch.empty(numel, dtype=torch.uint8, pin_memory=True))
                       for nm in narrow if nm in names}
        self.futures = {nm: [] for nm in self.narrow}
        self.done = None

    def copy_rows(self, srcs, lo, hi):
        for nm, (stage, _) in self.narrow.items():
            stage[lo:hi].copy_(srcs[nm].reshape(-1)[lo:hi])  # int32 -> uint8 on the device
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ev)
            for nm, t in srcs.items():
                if nm in self.narrow:
                    stage, pin8 = self.narrow[nm]
                    pin8[lo:hi].copy_(stage[lo:hi], non_blocking=True)
                    stage.record_stream(self.stream)
                else:
                    self.host[nm][lo:hi].copy_(t.reshape(-1)[lo:hi], non_blocking=True)
        self.done = torch.cuda.Event()
        self.done.record(self.stream)
        if self.narrow:
            pool = _widen_pool()
            parts = pool._max_workers
            bounds = np.linspace(lo, hi, parts + 1).astype(np.int64)
            for nm, (_, pin8) in self.narrow.items():
                src = pin8.numpy()
                dst = self.host[nm].numpy()
                for a, b in zip(bounds[:-1], bounds[1:]):
                    if b > a:
                        self.futures[nm].append(pool.submit(_widen, self.done, dst[a:b], src[a:b]))

    def copy_extra(self, name, t):
        """Whole-tensor copy of ``t`` (ordered after the compute stream's work
        so far) into a pinned buffer delivered by finish() under ``name``."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        buf = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ev)
            buf.copy_(t, non_blocking=True)
        t.record_stream(self.stream)
        self.host[name] = buf

    def finish(self):
        return {nm: (h, _Waiter(self.done, self.futures.get(nm, ())))
                for nm, h in self.host.items()}


def _widen(event, dst, src):
    event.synchronize()
    np.copyto(dst, src, casting="unsafe")


def knn_from_full_distances(dist_set, k, seed=0):
    """Per-vertex k nearest others from a full distance set (C1).

    Ties at the k-th distance are broken by numpy's SeedSequence(seed,
    spawn_key=(v,)) -> PCG64 permutation, restated on device, so the result
    is identical to neighbors.py:183-237.  A lazy set from ``all_pairs_bfs``
    runs the fused bitset BFS-kNN kernel (no n x n matrix); a set carrying
    an explicit matrix is uploaded in row chunks.
    """
    if not dist_set.full:
        raise ValueError("knn_from_full_distances requires a full distance set")
    if k < 1:
        raise ValueError("k must be >= 1")
    dev = require_cuda()
    n = int(dist_set.n)
    g = getattr(dist_set, "_graph", None)
    recs = dist_set._take_records(k, seed) if isinstance(dist_set, SparseDistanceSet) else None
    if recs is not None:  # the BFS already ran (SparseDistanceSet.run_bfs)
        nbr, dist, cnt = recs
    elif g is not None:
        csr = device_csr(g, dev)
        nbr, dist, cnt = full_knn_records(csr, k, seed, 0, n)
    else:
        nbr, dist, cnt = _knn_from_matrix(np.asarray(dist_set.matrix), k, seed, dev)
    short = int((cnt < k).sum().item()) if n else 0
    _warn_short(short)
    indptr, dst, dd = _pack(n, k, nbr, dist, cnt, dev, full=(short == 0))
    return DirectedKnn(n=n, k=k, _dev=dict(indptr=indptr, dst=dst, dist=dd))


def _knn_from_matrix(matrix, k, seed, dev, chunk_bytes=256 << 20):
    n = matrix.shape[0]
    kk = max(k, 1)
    nbr = torch.empty((n, kk), dtype=torch.int32, device=dev)
    dist = torch.empty((n, kk), dtype=torch.int32, device=dev)
    cnt = torch.empty(n, dtype=torch.int32, device=dev)
    if n == 0:
        return nbr, dist, cnt
    rows_per = max(1, chunk_bytes // max(4 * n, 1))
    slots = int(min(148 * 8, rows_per))
    lib = _lib.load()
    ws = workspace(lib.gu_knn_from_rows_workspace_size(n, slots), dev)
    for start in range(0, n, rows_per):
        stop = min(start + rows_per, n)
        rows = to_device(matrix[start:stop], np.int32, dev)
        _lib.call("gu_knn_from_rows", n, _lib.ptr(rows), start, stop - start, k,
                  int(seed) & (2**64 - 1), _lib.ptr(nbr[start:]), _lib.ptr(dist[start:]),
                  _lib.ptr(cnt[start:]), _lib.ptr(ws), ws.numel(), slots, stream_ptr(dev))
        torch.cuda.current_stream(dev).synchronize()
    return nbr, dist, cnt


# ------------------------------------------------------------------- C1
def smooth_knn_weights(knn, k=None):
    """Fuzzy membership weights from raw kNN distances, then symmetrisation.

    rho_i = distance to the nearest neighbour; sigma_i by the reference's
    64-step bisection on (SIGMA_MIN, SIGMA_MAX) so that
    sum_j exp(-(d_ij - rho_i) / sigma_i) = log2(k) (tolerance 1e-5); the
    directed weights are combined with the fuzzy union (both orientations
    materialised, lexicographically sorted) -- neighbors.py:245-350.
    """
    if k is None:
        k = knn.k
    dev = require_cuda()
    n = int(knn.n)
    indptr = knn.device("indptr", dev) if isinstance(knn, DirectedKnn) else \
        to_device(knn.indptr, np.int64, dev)
    dst = knn.device("dst", dev) if isinstance(knn, DirectedKnn) else \
        to_device(knn.dst, np.int32, dev)
    dist = knn.device("dist", dev) if isinstance(knn, DirectedKnn) else \
        to_device(knn.dist, np.int32, dev)
    counts = indptr[1:] - indptr[:-1]
    if n == 0 or bool((counts < 1).any()):
        raise ValueError("every vertex needs at least one outgoing kNN edge")
    kmax = int(counts.max().item())
    nnz = int(dst.shape[0])
    target = float(np.log2(k))
    rho = torch.empty(n, dtype=torch.float64, device=dev)
    sigma = torch.empty(n, dtype=torch.float64, device=dev)
    w = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    st = stream_ptr(dev)
    lib = _lib.load()
    sws = workspace(lib.gu_smooth_knn_workspace_size(n), dev)
    _lib.call("gu_smooth_knn", n, _lib.ptr(indptr), _lib.ptr(dist), kmax, target,
              _lib.ptr(rho), _lib.ptr(sigma), _lib.ptr(w), _lib.ptr(sws), sws.numel(), st)
    ws = workspace(lib.gu_symmetrize_workspace_size(n, nnz), dev)
    cap = max(2 * nnz, 1)
    sym_src = torch.empty(cap, dtype=torch.int32, device=dev)
    sym_dst = torch.empty(cap, dtype=torch.int32, device=dev)
    sym_w = torch.empty(cap, dtype=torch.float64, device=dev)
    nbr_indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    import ctypes
    E = ctypes.c_int64(0)
    # the smooth workspace rides along: the union reads backward weights from
    # its per-profile table instead of gathering w in destination order
    _lib.call("gu_symmetrize_memo", n, nnz, _lib.ptr(indptr), _lib.ptr(dst), _lib.ptr(w),
              _lib.ptr(sym_src), _lib.ptr(sym_dst), _lib.ptr(sym_w), _lib.ptr(nbr_indptr),
              ctypes.byref(E), _lib.ptr(ws), ws.numel(),
              _lib.ptr(sws), sws.numel(), st)
    E = int(E.value)
    sym_dst = sym_dst[:E]
    return KnnGraph(n=n, k=k, directed=knn,
                    _dev=dict(rho=rho, sigma=sigma, w=w[:nnz], sym_src=sym_src[:E],
                              sym_dst=sym_dst, sym_w=sym_w[:E], nbr_indptr=nbr_indptr,
                              nbr_indices=sym_dst))
