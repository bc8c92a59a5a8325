"""Host-side value types mirroring graph_umap's ``Graph`` and ``Layout``.

Reference: /root/reference/pkg/src/graph_umap/graph.py:16-96 (types) and
:114-129 (``_from_canonical``).  The hot-path functions of this package accept
either these types or the reference's own objects (duck typing on ``n``,
``adj_indptr``, ``adj_indices``), so a reference user can pass their existing
graphs unchanged.
"""

from dataclasses import dataclass

import numpy as np

ALGORITHMS = ("GUMAP", "SS", "SL", "SSSL", "SPECTRAL_INIT", "RANDOM")


class GraphError(ValueError):
    pass


@dataclass(frozen=True)
class Graph:
    """Immutable undirected simple graph, CSR with rows sorted ascending
    (graph.py:16-71).  ``edges`` is (m, 2) int64 with u < v."""

    n: int
    m: int
    adj_indptr: np.ndarray
    adj_indices: np.ndarray
    edges: np.ndarray
    labels: tuple = ()
    dropped_self_loops: int = 0
    dropped_duplicates: int = 0

    def __post_init__(self):
        self.adj_indptr.setflags(write=False)
        self.adj_indices.setflags(write=False)
        self.edges.setflags(write=False)

    def neighbors(self, v):
        return self.adj_indices[self.adj_indptr[v]:self.adj_indptr[v + 1]]

    def degree(self, v):
        return int(self.adj_indptr[v + 1] - self.adj_indptr[v])

    @property
    def degrees(self):
        return np.diff(self.adj_indptr)

    def __repr__(self):
        return f"Graph(n={self.n}, m={self.m})"


@dataclass(frozen=True)
class Layout:
    """float64 (n, 2) read-only coordinates plus provenance (graph.py:74-96)."""

    coords: np.ndarray
    algorithm_tag: str = "RANDOM"
    seed: int = 0
    iterations: int = 0

    def __post_init__(self):
        coords = np.ascontiguousarray(np.asarray(self.coords, dtype=np.float64))
        if coords.ndim != 2 or coords.shape[1] != 2:
            raise ValueError("layout coordinates must have shape (n, 2)")
        if not np.all(np.isfinite(coords)):
            raise ValueError("layout coordinates must be finite")
        if self.algorithm_tag not in ALGORITHMS:
            raise ValueError(f"unknown algorithm tag {self.algorithm_tag!r}")
        object.__setattr__(self, "coords", coords)
        coords.setflags(write=False)

    @property
    def n(self):
        return self.coords.shape[0]


def csr_from_canonical(n, edges):
    """(indptr int64[n+1], indices int32[2m]) from unique u<v edges.

    Same arrays as graph.py:114-129 but built with one int64 key sort instead
    of a lexsort, so multi-million-edge fixtures build in seconds.
    """
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    indptr = np.zeros(n + 1, dtype=np.int64)
    if edges.shape[0] == 0:
        return indptr, np.empty(0, dtype=np.int32)
    keys = np.concatenate([edges[:, 0] * n + edges[:, 1], edges[:, 1] * n + edges[:, 0]])
    keys.sort()
    src = keys // n
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    return indptr, (keys - src * n).astype(np.int32)


def graph_from_edges(n, edges, labels=()):
    """Graph from canonical (deduplicated, u < v) edges on vertices 0..n-1."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if edges.shape[0]:
        keys = edges[:, 0] * n + edges[:, 1]
        if np.any(keys[1:] < keys[:-1]):
            edges = edges[np.argsort(keys, kind="stable")]
    indptr, indices = csr_from_canonical(n, edges)
    return Graph(n=int(n), m=int(edges.shape[0]), adj_indptr=indptr,
                 adj_indices=indices, edges=edges, labels=tuple(labels))


def canonical_edges(n, pairs):
    """Drop self loops / duplicates, orient u < v (graph.py:159-175, vectorised
    for integer ids already dense in 0..n-1)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    u = np.minimum(pairs[:, 0], pairs[:, 1])
    v = np.maximum(pairs[:, 0], pairs[:, 1])
    keep = u != v
    keys = np.sort(u[keep] * n + v[keep])
    if keys.shape[0]:
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
    return np.stack([keys // n, keys % n], axis=1)


# integer inputs at least this large are built on the GPU when one is present
GPU_BUILD_MIN_PAIRS = 1 << 16


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001 -- no torch / no driver: host path
        return False


def _build_graph_labels(pairs_list):
    """graph.py:132-186 for arbitrary comparable labels (strings, ...)."""
    seen = set()
    for u, v in pairs_list:
        seen.add(u)
        seen.add(v)
    try:
        ordered = sorted(seen)
    except TypeError as exc:
        raise GraphError("vertex ids must be mutually comparable") from exc
    index = {label: i for i, label in enumerate(ordered)}
    dense = np.array([(index[u], index[v]) for u, v in pairs_list], dtype=np.int64)
    return _build_graph_dense(len(ordered), dense, tuple(ordered))


def _build_graph_dense(n, dense, labels):
    loops = int(np.count_nonzero(dense[:, 0] == dense[:, 1]))
    canon = canonical_edges(n, dense)
    if canon.shape[0] == 0:
        raise GraphError("empty graph")
    dups = dense.shape[0] - loops - canon.shape[0]
    g = graph_from_edges(n, canon, labels=labels)
    object.__setattr__(g, "dropped_self_loops", loops)
    object.__setattr__(g, "dropped_duplicates", int(dups))
    return g


def build_graph(edge_pairs, labels=None):
    """Graph from raw (id, id) pairs (graph.py:132-186): dense relabel in
    sorted label order, self loops and duplicates dropped (counted), edges
    canonical u < v in (u, v) order.  Non-negative integer inputs of
    GPU_BUILD_MIN_PAIRS pairs or more are built on the GPU
    (csrc/ingest.cu), which also leaves the CSR resident for the BFS."""
    if isinstance(edge_pairs, np.ndarray) and edge_pairs.dtype.kind in "iu":
        pairs = edge_pairs.astype(np.int64, copy=False).reshape(-1, 2)
    else:
        pairs_list = list(edge_pairs)
        if not pairs_list:
            raise GraphError("empty graph")
        # the integer fast path only for genuinely integral input: floats,
        # bools, numeric strings and mixed labels keep their own values and
        # sort order (the reference sorts the original labels)
        try:
            arr = np.asarray(pairs_list)
        except (TypeError, ValueError, OverflowError):
            arr = None
        if (arr is None or arr.dtype.kind not in "iu" or arr.ndim != 2 or arr.shape[1] != 2):
            return _build_graph_labels(pairs_list)
        if arr.dtype == np.uint64 and arr.size and int(arr.max()) > np.iinfo(np.int64).max:
            return _build_graph_labels(pairs_list)
        pairs = arr.astype(np.int64, copy=False)
    if pairs.shape[0] == 0:
        raise GraphError("empty graph")
    if pairs.shape[0] >= GPU_BUILD_MIN_PAIRS and _gpu_available() and int(pairs.min()) >= 0:
        return _build_graph_gpu(pairs)
    ids, inv = np.unique(pairs.reshape(-1), return_inverse=True)
    return _build_graph_dense(int(ids.shape[0]), inv.reshape(-1, 2),
                              tuple(ids.tolist()))


def _build_graph_gpu(pairs):
    import ctypes

    import torch

    from . import _lib
    from .device import DeviceCsr, register_device_csr, require_cuda, stream_ptr, to_device, to_host, workspace

    dev = require_cuda()
    npairs = int(pairs.shape[0])
    raw = to_device(np.ascontiguousarray(pairs), np.int64, dev)
    lib = _lib.load()
    ws = workspace(lib.gu_build_graph_workspace_size(npairs), dev)
    out = (ctypes.c_int64 * 3)()
    _lib.call("gu_build_graph_ids", npairs, _lib.ptr(raw), out, _lib.ptr(ws), ws.numel(),
              stream_ptr(dev))
    n, m, loops = int(out[0]), int(out[1]), int(out[2])
    if m == 0:
        raise GraphError("empty graph")
    ids = torch.empty(n, dtype=torch.int64, device=dev)
    edges = torch.empty((m, 2), dtype=torch.int64, device=dev)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(2 * m, dtype=torch.int32, device=dev)
    _lib.call("gu_build_graph_csr", npairs, n, m, _lib.ptr(ids), _lib.ptr(edges), _lib.ptr(indptr),
              _lib.ptr(indices), _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    g = Graph(n=n, m=m, adj_indptr=to_host(indptr), adj_indices=to_host(indices),
              edges=to_host(edges), labels=tuple(to_host(ids).tolist()),
              dropped_self_loops=loops, dropped_duplicates=npairs - loops - m)
    register_device_csr(g, DeviceCsr(n, indptr.to(torch.int32), indices, dev))
    return g


def _labels_monotone(g):
    """True when label order is vertex order (no labels, or strictly
    increasing ones -- build_graph's dense relabel guarantees it), so the
    smallest label of a component is the label of its smallest vertex id."""
    labels = getattr(g, "labels", ()) or ()
    if len(labels) < 2:
        return True
    try:
        a = np.asarray(labels)
        if a.dtype.kind in "iuf":
            return bool(np.all(a[1:] > a[:-1]))
        return all(labels[i] < labels[i + 1] for i in range(len(labels) - 1))
    except TypeError:
        return False


def largest_connected_component(g):
    """Induced subgraph on the largest component, relabelled densely in id
    order, labels carried (graph.py:201-232); ties go to the component
    holding the smallest original label (graph.py:211-214).  On the GPU when
    one is present (csrc/ingest.cu union-find + compaction); graphs whose
    labels are not in vertex order take the host path, whose tie rule
    compares labels."""
    monotone = _labels_monotone(g)
    if g.n >= 2 and _gpu_available() and monotone:
        return _lcc_gpu(g)
    import scipy.sparse as sp
    from scipy.sparse import csgraph

    a = sp.csr_matrix((np.ones(g.adj_indices.shape[0], np.int8), g.adj_indices,
                       g.adj_indptr), shape=(g.n, g.n))
    ncomp, member = csgraph.connected_components(a, directed=False)
    if ncomp <= 1:
        return g
    sizes = np.bincount(member, minlength=ncomp)
    best = np.flatnonzero(sizes == sizes.max())
    if len(best) > 1 and not monotone:
        labels = g.labels
        champion = min(best, key=lambda c: min(labels[v] for v in np.flatnonzero(member == c)))
    elif len(best) > 1:
        first_vertex = np.full(ncomp, g.n, dtype=np.int64)
        np.minimum.at(first_vertex, member, np.arange(g.n))
        champion = best[np.argmin(first_vertex[best])]
    else:
        champion = best[0]
    keep = np.flatnonzero(member == champion)
    remap = -np.ones(g.n, dtype=np.int64)
    remap[keep] = np.arange(len(keep))
    mask = member[g.edges[:, 0]] == champion
    edges = remap[g.edges[mask]]
    edges.sort(axis=1)
    return _with_labels(graph_from_edges(len(keep), edges), g, keep)


def _with_labels(h, g, keep):
    old = getattr(g, "labels", ()) or None
    labels = tuple(np.asarray(old, dtype=object)[keep].tolist()) if old else tuple(keep.tolist())
    object.__setattr__(h, "labels", labels)
    object.__setattr__(h, "dropped_self_loops", getattr(g, "dropped_self_loops", 0))
    object.__setattr__(h, "dropped_duplicates", getattr(g, "dropped_duplicates", 0))
    return h


def _lcc_gpu(g):
    import ctypes

    import torch

    from . import _lib
    from .device import DeviceCsr, device_csr, register_device_csr, stream_ptr, to_device, to_host, workspace

    dev = torch.device("cuda", torch.cuda.current_device())
    n, m = int(g.n), int(g.m)
    csr = device_csr(g, dev)
    edges_dev = to_device(np.ascontiguousarray(g.edges), np.int64, dev)
    lib = _lib.load()
    ws = workspace(lib.gu_lcc_workspace_size(n, m), dev)
    out = (ctypes.c_int64 * 3)()
    _lib.call("gu_lcc_plan", n, m, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), _lib.ptr(edges_dev),
              out, _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    ncomp, n2, m2 = int(out[0]), int(out[1]), int(out[2])
    if ncomp <= 1:
        return g
    old = torch.empty(n2, dtype=torch.int32, device=dev)
    edges = torch.empty((max(m2, 1), 2), dtype=torch.int64, device=dev)
    indptr = torch.empty(n2 + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(max(2 * m2, 1), dtype=torch.int32, device=dev)
    _lib.call("gu_lcc_build", n, m, n2, m2, _lib.ptr(old), _lib.ptr(edges), _lib.ptr(indptr),
              _lib.ptr(indices), _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    keep = to_host(old).astype(np.int64)
    h = Graph(n=n2, m=m2, adj_indptr=to_host(indptr), adj_indices=to_host(indices[: 2 * m2]),
              edges=to_host(edges[:m2]))
    h = _with_labels(h, g, keep)
    register_device_csr(h, DeviceCsr(n2, indptr.to(torch.int32), indices[: 2 * m2], dev))
    return h
