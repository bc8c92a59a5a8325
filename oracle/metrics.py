"""Layout-quality metrics for parity check (c) -- TEST INFRASTRUCTURE ONLY.

numpy/scipy restatements of /root/reference/pkg/src/graph_umap/metrics.py:
  neighborhood_preservation  metrics.py:41-79  (r=2, mean Jaccard, stable ties)
  stress                     metrics.py:90-132 (optimal scale, chunked sums)
  count_crossings            metrics.py:135-190 (float filter + exact Fractions)
Pinned against the reference's own values on its own layouts
(tests/golden/quality_c1.npz, test_gpu_parity.test_quality_c1_vs_reference).
"""

from fractions import Fraction

import numpy as np
from scipy.spatial.distance import cdist

_ORIENT_EPS = 4e-16


def neighborhood_preservation(g, coords, hop=None, r=2):
    n = g.n
    coords = np.asarray(coords, np.float64)
    if hop is None:
        from . import oracle as O
        hop = O.all_pairs_bfs(g, nthreads=8)
    total = 0.0
    chunk = max(1, min(512, n))
    for start in range(0, n, chunk):
        stop = min(start + chunk, n)
        dists = cdist(coords[start:stop], coords)
        for v in range(start, stop):
            hv = hop[v]
            hood = np.flatnonzero((hv >= 1) & (hv <= r))
            q = hood.shape[0]
            if q == 0:
                total += 1.0
                continue
            row = dists[v - start].copy()
            row[v] = np.inf
            nearest = np.argsort(row, kind="stable")[:q]
            inter = np.intersect1d(hood, nearest, assume_unique=True).shape[0]
            total += inter / (2 * q - inter)
    return total / n


def stress(g, coords, hop, rescale=True):
    n = g.n
    coords = np.asarray(coords, np.float64)
    hop = np.asarray(hop, np.float64)
    chunk = max(1, min(1024, n))
    s_num = 0.0
    s_den = 0.0
    for start in range(0, n, chunk):
        if not rescale:
            break
        stop = min(start + chunk, n)
        delta = cdist(coords[start:stop], coords)
        d = hop[start:stop].copy()
        np.fill_diagonal(d[:, start:stop], np.inf)
        s_num += float((delta / d).sum())
        s_den += float((delta * delta / (d * d)).sum())
    scale = s_num / s_den if (rescale and s_den > 0) else 1.0
    total = 0.0
    for start in range(0, n, chunk):
        stop = min(start + chunk, n)
        delta = cdist(coords[start:stop], coords) * scale
        d = hop[start:stop].copy()
        np.fill_diagonal(d[:, start:stop], np.inf)
        term = (1.0 - delta / d) ** 2
        np.fill_diagonal(term[:, start:stop], 0.0)
        total += float(term.sum())
    return total / (n * n - n)


def _orient(ax, ay, bx, by, cx, cy):
    t1 = (bx - ax) * (cy - ay)
    t2 = (by - ay) * (cx - ax)
    det = t1 - t2
    bound = _ORIENT_EPS * (np.abs(t1) + np.abs(t2))
    return np.where(det > bound, 1, np.where(det < -bound, -1, 0))


def _orient_exact(pa, pb, pc):
    ax, ay = Fraction(pa[0]), Fraction(pa[1])
    bx, by = Fraction(pb[0]), Fraction(pb[1])
    cx, cy = Fraction(pc[0]), Fraction(pc[1])
    det = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    return (det > 0) - (det < 0)


def _cross_exact(p1, p2, p3, p4):
    o1 = _orient_exact(p1, p2, p3)
    o2 = _orient_exact(p1, p2, p4)
    o3 = _orient_exact(p3, p4, p1)
    o4 = _orient_exact(p3, p4, p2)
    if o1 != 0 and o2 != 0 and o3 != 0 and o4 != 0:
        return o1 != o2 and o3 != o4
    if o1 == 0 and o2 == 0 and o3 == 0 and o4 == 0:
        axis = 0 if abs(Fraction(p2[0]) - Fraction(p1[0])) >= abs(
            Fraction(p2[1]) - Fraction(p1[1])) else 1
        a_lo, a_hi = sorted((Fraction(p1[axis]), Fraction(p2[axis])))
        b_lo, b_hi = sorted((Fraction(p3[axis]), Fraction(p4[axis])))
        return max(a_lo, b_lo) < min(a_hi, b_hi)
    return False


def count_crossings(g, coords, block=256, rows=None):
    """Exact number of unordered edge pairs whose open segments cross
    (``rows`` = (i0, i1): only pairs whose first edge lies in [i0, i1))."""
    coords = np.asarray(coords, np.float64)
    e = np.asarray(g.edges, np.int64)
    m = e.shape[0]
    if m < 2:
        return 0
    r0, r1 = (0, m) if rows is None else rows
    P = coords[e[:, 0]]
    Q = coords[e[:, 1]]
    lox, hix = np.minimum(P[:, 0], Q[:, 0]), np.maximum(P[:, 0], Q[:, 0])
    loy, hiy = np.minimum(P[:, 1], Q[:, 1]), np.maximum(P[:, 1], Q[:, 1])
    certain = 0
    amb = []
    for i0 in range(r0, r1, block):
        i1 = min(i0 + block, r1)
        I = np.arange(i0, i1)[:, None]
        J = np.arange(m)[None, :]
        mask = J > I
        ei, ej = e[i0:i1], e
        share = ((ei[:, 0:1] == ej[None, :, 0]) | (ei[:, 0:1] == ej[None, :, 1]) |
                 (ei[:, 1:2] == ej[None, :, 0]) | (ei[:, 1:2] == ej[None, :, 1]))
        box = ((hix[None, :] >= lox[i0:i1, None]) & (lox[None, :] <= hix[i0:i1, None]) &
               (hiy[None, :] >= loy[i0:i1, None]) & (loy[None, :] <= hiy[i0:i1, None]))
        cand = mask & ~share & box
        ii, jj = np.nonzero(cand)
        if ii.shape[0] == 0:
            continue
        ii = ii + i0
        ax, ay, bx, by = P[ii, 0], P[ii, 1], Q[ii, 0], Q[ii, 1]
        cx, cy, dx, dy = P[jj, 0], P[jj, 1], Q[jj, 0], Q[jj, 1]
        o1 = _orient(ax, ay, bx, by, cx, cy)
        o2 = _orient(ax, ay, bx, by, dx, dy)
        o3 = _orient(cx, cy, dx, dy, ax, ay)
        o4 = _orient(cx, cy, dx, dy, bx, by)
        sep = ((o1 != 0) & (o1 == o2)) | ((o3 != 0) & (o3 == o4))
        allnz = (o1 != 0) & (o2 != 0) & (o3 != 0) & (o4 != 0)
        certain += int(np.count_nonzero(~sep & allnz & (o1 != o2) & (o3 != o4)))
        unsure = ~sep & ~allnz
        for a_, b_ in zip(ii[unsure], jj[unsure]):
            amb.append((a_, b_))
    extra = 0
    for i, j in amb:
        if _cross_exact(P[i], Q[i], P[j], Q[j]):
            extra += 1
    return certain + extra


# ----------------------------------------------------------- sampled metrics
# Exact per-vertex / per-pair terms of the two metrics above, averaged over a
# fixed sample of source vertices: unbiased estimators used for check (c) on
# graphs where the all-pairs versions do not fit a CPU (c3 and larger).

def sample_sources(n, size=2000, seed=12345):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(size, n), replace=False))


def sampled_neighborhood_preservation(coords, hop_rows, sources, r=2):
    """Mean over ``sources`` of the metrics.py:41-79 Jaccard term.  hop_rows:
    int32 BFS rows of the sources (INF32 unreachable)."""
    coords = np.asarray(coords, np.float64)
    total = 0.0
    for i, v in enumerate(sources):
        hv = hop_rows[i]
        hood = np.flatnonzero((hv >= 1) & (hv <= r))
        q = hood.shape[0]
        if q == 0:
            total += 1.0
            continue
        row = cdist(coords[v:v + 1], coords)[0]
        row[v] = np.inf
        nearest = np.argsort(row, kind="stable")[:q]
        inter = np.intersect1d(hood, nearest, assume_unique=True).shape[0]
        total += inter / (2 * q - inter)
    return total / len(sources)


def sampled_stress(coords, hop_rows, sources, chunk=64):
    """metrics.py:90-132 restricted to the rows of ``sources`` (optimal scale
    fitted on the same pairs); chunked over sources so the distance block
    stays small on million-vertex layouts."""
    coords = np.asarray(coords, np.float64)
    sources = np.asarray(sources)
    s_num = s_den = 0.0
    for a in range(0, len(sources), chunk):
        b = min(a + chunk, len(sources))
        delta = cdist(coords[sources[a:b]], coords)
        d = np.asarray(hop_rows[a:b]).astype(np.float64)
        d[np.arange(b - a), sources[a:b]] = np.inf
        d[d >= 2**31 - 1] = np.inf
        s_num += float((delta / d).sum())
        s_den += float((delta * delta / (d * d)).sum())
    scale = s_num / s_den if s_den > 0 else 1.0
    tot = 0.0
    cnt = 0
    for a in range(0, len(sources), chunk):
        b = min(a + chunk, len(sources))
        delta = cdist(coords[sources[a:b]], coords)
        d = np.asarray(hop_rows[a:b]).astype(np.float64)
        d[np.arange(b - a), sources[a:b]] = np.inf
        d[d >= 2**31 - 1] = np.inf
        term = (1.0 - scale * delta / d) ** 2
        term[np.arange(b - a), sources[a:b]] = 0.0
        finite = np.isfinite(d)
        tot += float(term[finite].sum())
        cnt += int(finite.sum())
    return tot / cnt
