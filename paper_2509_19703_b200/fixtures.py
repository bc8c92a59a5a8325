"""Deterministic synthetic graphs for the BASELINE.json configurations.

* ``grid`` and ``scale_free`` restate the reference generators
  (/root/reference/pkg/src/graph_umap/generators.py:11-22 and :27-48) draw for
  draw, so c1 and c3 are the exact graphs the reference builds with
  ``synth_graph("grid", 2500)`` and ``synth_graph("scale_free", 100000,
  seed=2, m0=3)``.
* ``random_connected_graph`` restates the test generator of
  /root/reference/pkg/tests/oracles.py:204-224 (used by the reference's own
  acceptance criterion 1, test_acceptance.py:45-63).
* ``erdos_renyi``, ``sparsify_er``, ``sbm`` and ``rgg`` are builder-owned
  (the reference has no such generators): pinned,
  numpy-vectorised, seeded.  They stand in for the paper's public datasets,
  which are not shipped.

Fixture generation is input preparation: it is never inside a timed region.
"""

import math

import numpy as np

from .graph import (GraphError, canonical_edges, graph_from_edges,
                    largest_connected_component)


# ------------------------------------------------------ reference restatements
def grid(n):
    """generators.py:11-22: sqrt(n) x ceil(n/sqrt(n)) mesh with exactly n vertices."""
    rows = int(math.isqrt(n))
    cols = (n + rows - 1) // rows
    v = np.arange(n, dtype=np.int64)
    r, c = v // cols, v % cols
    right = (c + 1 < cols) & (v + 1 < n) & ((v + 1) // cols == r)
    down = (r + 1) * cols + c
    e1 = np.stack([v[right], v[right] + 1], axis=1)
    e2 = np.stack([v[down < n], down[down < n]], axis=1)
    return graph_from_edges(n, canonical_edges(n, np.concatenate([e1, e2])))


def scale_free(n, seed=0, m0=2):
    """generators.py:27-48: preferential attachment from a complete core on
    m0+1 vertices; every draw is ``rng.integers(0, len(repeated))``."""
    if n < m0 + 2:
        raise GraphError("scale_free needs n >= m0 + 2")
    rng = np.random.default_rng(seed)
    core = m0 + 1
    # the repeated-endpoint pool as a preallocated array (same draw sequence)
    total = core * (core - 1) + 2 * m0 * (n - core)
    rep = np.empty(total, dtype=np.int64)
    edges = []
    L = 0
    for u in range(core):
        for v in range(u + 1, core):
            edges.append((u, v))
            rep[L] = u
            rep[L + 1] = v
            L += 2
    integers = rng.integers
    for v in range(core, n):
        targets = set()
        while len(targets) < m0:
            targets.add(int(rep[integers(0, L)]))
        for t in sorted(targets):
            edges.append((t, v))
            rep[L] = t
            rep[L + 1] = v
            L += 2
    return graph_from_edges(n, canonical_edges(n, np.array(edges, dtype=np.int64)))


def random_connected_graph(rng, n_max=200, extra_edges=1.6):
    """tests/oracles.py:204-224: random spanning tree plus extra edges.
    Returns (n, sorted edge list)."""
    n = int(rng.integers(5, n_max + 1))
    edges = set()
    order = rng.permutation(n)
    for i in range(1, n):
        u = int(order[i])
        v = int(order[rng.integers(0, i)])
        edges.add((min(u, v), max(u, v)))
    target_extra = int(extra_edges * n)
    for _ in range(target_extra * 3):
        if len(edges) >= n - 1 + target_extra:
            break
        u = int(rng.integers(0, n))
        v = int(rng.integers(0, n))
        if u != v:
            edges.add((min(u, v), max(u, v)))
    return n, sorted(edges)


def path_graph(n):
    e = np.stack([np.arange(n - 1), np.arange(1, n)], axis=1)
    return graph_from_edges(n, e)


# ------------------------------------------------------ builder-owned fixtures
def _unique_pairs(n, m, draw, rng):
    """First m distinct canonical pairs in draw order from ``draw(rng, size)``."""
    keys = np.empty(0, dtype=np.int64)
    order = np.empty(0, dtype=np.int64)
    drawn = 0
    while keys.shape[0] < m:
        need = int((m - keys.shape[0]) * 1.1) + 1024
        u, v = draw(rng, need)
        lo, hi = np.minimum(u, v), np.maximum(u, v)
        ok = lo != hi
        k = lo[ok] * n + hi[ok]
        allk = np.concatenate([keys, k])
        allo = np.concatenate([order, drawn + np.flatnonzero(ok)])
        drawn += need
        uk, first = np.unique(allk, return_index=True)
        keep = np.sort(first)
        keys, order = allk[keep], allo[keep]
    keys = keys[:m]
    return np.stack([keys // n, keys % n], axis=1)


def erdos_renyi(n=20000, avg_degree=200, seed=1):
    """G(n, M) with M = n*avg_degree/2 distinct uniform pairs (c2 base graph)."""
    m = int(round(n * avg_degree / 2))
    rng = np.random.default_rng(seed)

    def draw(r, size):
        return r.integers(0, n, size), r.integers(0, n, size)

    return graph_from_edges(n, canonical_edges(n, _unique_pairs(n, m, draw, rng)))


def sparsify_er(g, samples=None, seed=1):
    """Spectral-sparsifier stand-in G' for c2.

    Spielman-Srivastava sampling: q = 8 n ln n edge draws with replacement,
    probability proportional to the effective resistance, approximated by
    1/d_u + 1/d_v (tight on dense expanders such as G(n, 200/n)); the distinct
    sampled edges form G' (unweighted, as the BFS sees it), restricted to its
    largest component.  The same G' goes to both implementations.
    """
    n = g.n
    q = int(round(8 * n * math.log(n))) if samples is None else int(samples)
    deg = np.diff(g.adj_indptr).astype(np.float64)
    e = g.edges
    p = 1.0 / deg[e[:, 0]] + 1.0 / deg[e[:, 1]]
    p /= p.sum()
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(7,)))
    pick = np.unique(rng.choice(e.shape[0], size=q, replace=True, p=p))
    return largest_connected_component(graph_from_edges(n, e[pick]))


def sbm(n=1_000_000, blocks=20, intra_degree=8.0, inter_degree=2.0, seed=3):
    """Stochastic block model with equal blocks; expected intra / inter degree
    as given (c4); largest connected component (isolated vertices exist)."""
    rng = np.random.default_rng(seed)
    bs = n // blocks
    m_in = int(round(n * intra_degree / 2))
    m_out = int(round(n * inter_degree / 2))

    def draw_in(r, size):
        b = r.integers(0, blocks, size)
        return b * bs + r.integers(0, bs, size), b * bs + r.integers(0, bs, size)

    def draw_out(r, size):
        b1 = r.integers(0, blocks, size)
        b2 = (b1 + r.integers(1, blocks, size)) % blocks
        return b1 * bs + r.integers(0, bs, size), b2 * bs + r.integers(0, bs, size)

    e_in = _unique_pairs(n, m_in, draw_in, rng)
    e_out = _unique_pairs(n, m_out, draw_out, rng)
    g = graph_from_edges(n, canonical_edges(n, np.concatenate([e_in, e_out])))
    return largest_connected_component(g)


def rgg(n=4_000_000, avg_degree=12.0, seed=4, lcc=True):
    """Random geometric graph in the unit square, radius sqrt(deg/(pi n))
    (c5).  Vertex ids follow point generation order (no spatial relabelling),
    pairs with squared distance < r^2 are joined; largest component."""
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = math.sqrt(avg_degree / (math.pi * n))
    r2 = r * r
    ncell = max(1, int(1.0 / r))
    cx = np.minimum((pts[:, 0] * ncell).astype(np.int64), ncell - 1)
    cy = np.minimum((pts[:, 1] * ncell).astype(np.int64), ncell - 1)
    cell = cy * ncell + cx
    order = np.argsort(cell, kind="stable")
    cs = cell[order]
    start = np.searchsorted(cs, np.arange(ncell * ncell), side="left")
    end = np.searchsorted(cs, np.arange(ncell * ncell), side="right")
    px, py = pts[order, 0], pts[order, 1]
    ocx, ocy = cx[order], cy[order]
    out = []
    for dx, dy in ((0, 0), (1, 0), (-1, 1), (0, 1), (1, 1)):
        nx, ny = ocx + dx, ocy + dy
        valid = (nx >= 0) & (nx < ncell) & (ny < ncell)
        idx = np.flatnonzero(valid)
        ncel = ny[idx] * ncell + nx[idx]
        s, e = start[ncel], end[ncel]
        if dx == 0 and dy == 0:
            s = np.maximum(s, idx + 1)   # same cell: only later points
        cnt = np.maximum(e - s, 0)
        tot = int(cnt.sum())
        if tot == 0:
            continue
        i = np.repeat(idx, cnt)
        off = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        j = np.repeat(s, cnt) + off
        ddx = px[i] - px[j]
        ddy = py[i] - py[j]
        close = ddx * ddx + ddy * ddy < r2
        out.append(np.stack([order[i[close]], order[j[close]]], axis=1))
    pairs = np.concatenate(out)
    g = graph_from_edges(n, canonical_edges(n, pairs))
    return largest_connected_component(g) if lcc else g


CONFIGS = {
    "c1": lambda: grid(2500),
    "c2": lambda: sparsify_er(erdos_renyi(20000, 200, seed=1), seed=1),
    "c3": lambda: scale_free(100_000, seed=2, m0=3),
    "c4": lambda: sbm(1_000_000, 20, 8.0, 2.0, seed=3),
    "c5": lambda: rgg(4_000_000, 12.0, seed=4),
}


def config_graph(name):
    return CONFIGS[name]()
