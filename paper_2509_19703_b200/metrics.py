"""Layout-quality metrics on the GPU.

Drop-in for /root/reference/pkg/src/graph_umap/metrics.py's hot metrics:

  neighborhood_preservation(g, layout, r=2)   metrics.py:41-79
  stress(g, layout, rescale=True)             metrics.py:90-132
  count_crossings(g, layout)                  metrics.py:135-190

Same arguments, results and errors (MetricError on a layout / graph mismatch
and on a disconnected graph for stress).  Every metric runs in libgumap.so
(csrc/metrics.cu): the r-hop balls by GPU BFS, stress fused into the bitset
BFS (no hop rows in memory), layout-space
ranks with scipy cdist's float64 distances and stable id tie-break, exact
crossing predicates.  The proximity-graph shape score is out of scope
(DESIGN.md).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import device_csr, require_cuda, stream_ptr, workspace

# scratch budget (bytes) for the NP per-warp balls
NP_SCRATCH_BUDGET = 2 << 30
NP_MAX_SLOTS = 148 * 64


class MetricError(ValueError):
    pass


@dataclass(frozen=True)
class MetricReport:
    neighborhood_preservation: float = None
    stress: float = None
    crossings: int = None
    shape_jaccard: float = None

    def as_dict(self):
        return {
            "np": self.neighborhood_preservation,
            "stress": self.stress,
            "crossings": self.crossings,
            "shape": self.shape_jaccard,
        }


def _check(g, layout):
    if layout.n != g.n:
        raise MetricError("layout does not match graph")


def _coords(layout, dev):
    xy = np.ascontiguousarray(np.asarray(layout.coords, dtype=np.float64).reshape(-1, 2))
    return torch.from_numpy(xy).to(dev)


def _sources(sources, dev, n):
    if sources is None:
        return None
    s = np.asarray(sources)
    if s.size and (s.dtype.kind not in "iu" or int(s.min()) < 0 or int(s.max()) >= n):
        raise ValueError(f"sources must be vertex ids in [0, {n})")
    src = torch.from_numpy(np.ascontiguousarray(s, dtype=np.int32)).to(dev)
    if src.numel() == 0 or int(torch.unique(src).numel()) != src.numel():
        raise ValueError("sources must be distinct vertex ids")
    return src


def neighborhood_preservation(g, layout, r=2, sources=None):
    """Mean Jaccard overlap between r-hop and geometric neighborhoods
    (metrics.py:41-79): per vertex, the r-ball (excluding v) against the
    |ball| Euclidean-nearest other vertices, ties by vertex id.  ``sources``
    (distinct vertex ids, an extension): the mean over those vertices only --
    the sampled estimator for graphs too large for a CPU-side comparison."""
    _check(g, layout)
    n = int(g.n)
    if n <= 1:
        return 1.0
    dev = require_cuda()
    csr = device_csr(g, dev)
    xy = _coords(layout, dev)
    lib = _lib.load()
    slots = int(max(1, min(NP_MAX_SLOTS, NP_SCRATCH_BUDGET // (8 * n))))
    ws = workspace(lib.gu_np_workspace_size(n, slots), dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    src = _sources(sources, dev, g.n)
    _lib.call("gu_neighborhood_preservation", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices),
              _lib.ptr(xy), int(r), slots, _lib.ptr(src), 0 if src is None else src.numel(),
              _lib.ptr(out), _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    return float(out.item()) / (n if src is None else src.numel())


def stress(g, layout, rescale=True, sources=None):
    """Mean squared relative deviation of layout distances from hop
    distances over all ordered pairs i != j (metrics.py:90-132), after the
    closed-form optimal scale unless ``rescale=False``.  ``sources``
    (distinct vertex ids, an extension): only the pairs (s, j), s in sources
    -- the sampled estimator, scale fitted on the same pairs."""
    _check(g, layout)
    n = int(g.n)
    if n < 2:
        return 0.0
    dev = require_cuda()
    csr = device_csr(g, dev)
    xy = _coords(layout, dev)
    lib = _lib.load()
    ws = workspace(lib.gu_stress_workspace_size(n), dev)
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    src = _sources(sources, dev, g.n)
    _lib.call("gu_stress", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), _lib.ptr(xy),
              1 if rescale else 0, _lib.ptr(src), 0 if src is None else src.numel(),
              _lib.ptr(out), _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    total, _scale, unreachable = out.tolist()
    if unreachable:
        raise MetricError("stress requires a connected graph")
    return total / ((n * n - n) if src is None else src.numel() * (n - 1))


def _grid_side(m):
    return int(max(1, np.ceil(np.sqrt(max(m, 1) / 2.0))))


def count_crossings(g, layout):
    """Number of unordered edge pairs whose open segments properly intersect
    (metrics.py:135-190): pairs sharing an endpoint never count, collinear
    overlaps count once, predicates are exact."""
    _check(g, layout)
    m = int(g.m)
    if m < 2:
        return 0
    dev = require_cuda()
    lib = _lib.load()
    edges = torch.from_numpy(np.ascontiguousarray(np.asarray(g.edges), dtype=np.int32)).to(dev)
    xy = _coords(layout, dev)
    st = stream_ptr(dev)
    grid = workspace(lib.gu_grid_bytes(), dev)
    counts = torch.empty(m, dtype=torch.int64, device=dev)
    # a finer grid means fewer candidate pairs but more (edge, cell)
    # incidences; coarsen until the incidences stay within a few per edge
    side = _grid_side(m)
    while True:
        _lib.call("gu_crossings_grid", int(g.n), _lib.ptr(xy), side, _lib.ptr(grid), st)
        _lib.call("gu_crossings_incidences", m, _lib.ptr(edges), _lib.ptr(xy), _lib.ptr(grid),
                  _lib.ptr(counts), st)
        n_inc = int(counts.sum().item())
        if side == 1 or n_inc <= 8 * m + (1 << 20):
            break
        side = max(1, side // 2)
    ws = workspace(lib.gu_crossings_workspace_size(m, n_inc, side), dev)
    out = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.call("gu_crossings", m, _lib.ptr(edges), _lib.ptr(xy), _lib.ptr(grid), side, n_inc,
              _lib.ptr(out), _lib.ptr(ws), ws.numel(), st)
    return int(out.item())


def report(g, layout, hop_metrics=True, crossings=True):
    """MetricReport with the GPU metrics (shape score not computed)."""
    return MetricReport(
        neighborhood_preservation=neighborhood_preservation(g, layout) if hop_metrics else None,
        stress=stress(g, layout) if hop_metrics else None,
        crossings=count_crossings(g, layout) if crossings else None,
    )
