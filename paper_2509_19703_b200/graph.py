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


def build_graph(edge_pairs, labels=None):
    """Graph from raw integer pairs: dense relabel by sorted id, dedupe,
    drop self loops (graph.py:132-186 for integer ids)."""
    pairs = np.asarray(list(edge_pairs) if not isinstance(edge_pairs, np.ndarray)
                       else edge_pairs, dtype=np.int64).reshape(-1, 2)
    if pairs.shape[0] == 0:
        raise GraphError("empty graph")
    ids, inv = np.unique(pairs.reshape(-1), return_inverse=True)
    dense = inv.reshape(-1, 2)
    n = int(ids.shape[0])
    loops = int(np.count_nonzero(dense[:, 0] == dense[:, 1]))
    canon = canonical_edges(n, dense)
    if canon.shape[0] == 0:
        raise GraphError("empty graph")
    dups = pairs.shape[0] - loops - canon.shape[0]
    g = graph_from_edges(n, canon, labels=tuple(int(x) for x in ids))
    object.__setattr__(g, "dropped_self_loops", loops)
    object.__setattr__(g, "dropped_duplicates", int(dups))
    return g


def largest_connected_component(g):
    """Induced subgraph on the largest component, relabelled densely in id
    order; ties go to the component holding the smallest vertex id
    (graph.py:201-232)."""
    import scipy.sparse as sp
    from scipy.sparse import csgraph

    a = sp.csr_matrix((np.ones(g.adj_indices.shape[0], np.int8), g.adj_indices,
                       g.adj_indptr), shape=(g.n, g.n))
    ncomp, member = csgraph.connected_components(a, directed=False)
    if ncomp <= 1:
        return g
    sizes = np.bincount(member, minlength=ncomp)
    best = np.flatnonzero(sizes == sizes.max())
    if len(best) > 1:
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
    return graph_from_edges(len(keep), edges)
