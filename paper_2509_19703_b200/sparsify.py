"""Effective resistance and the n*log2(n)-edge spectral sparsifier on the GPU
(SURVEY 8(f) row 3).

Drop-in for /root/reference/pkg/src/graph_umap/sparsify.py and the
resistance plumbing of layout.py:384-406: same names, arguments, results and
errors.
  effective_resistance_exact   sparsify.py:49-84   grounded Laplacian inverse
      (cuSOLVER Cholesky, n <= cap) + csrc/sparsify.cu gather
  effective_resistance_approx  sparsify.py:87-143  q Rademacher projections,
      block Jacobi-PCG (csrc/sparsify.cu); counter-based signs instead of
      numpy's stream (statistically equivalent: per-edge error ~epsilon)
  sparsify                     sparsify.py:176-205 sort by (-r, u, v),
      maximum spanning tree, budget (csrc/sparsify.cu)
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import device_csr, require_cuda, stream_ptr, workspace
from .graph import GraphError, graph_from_edges


class SolverError(RuntimeError):
    """Iterative solver failed to converge; carries the final residual."""

    def __init__(self, message, residual):
        super().__init__(message)
        self.residual = residual


@dataclass(frozen=True)
class ResistanceTable:
    """Per-edge effective resistance, aligned with ``Graph.edges``."""

    values: np.ndarray
    method: str = "exact"

    def __post_init__(self):
        vals = np.ascontiguousarray(np.asarray(self.values, dtype=np.float64))
        object.__setattr__(self, "values", vals)
        vals.setflags(write=False)

    def __len__(self):
        return self.values.shape[0]


def _require_connected(g):
    from .layout import _is_connected
    if not _is_connected(g):
        raise GraphError("sparsifier requires connected graph")


def _edges_dev(g, dev):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(g.edges), dtype=np.int32)).to(dev)


def effective_resistance_exact(g, cap=20000):
    """Exact r_e = (e_u - e_v)^T L^+ (e_u - e_v) per edge from the Laplacian
    grounded at vertex 0 (sparsify.py:49-84); dense float64 inverse on the
    GPU, n <= cap."""
    _require_connected(g)
    if g.n > cap:
        raise GraphError(f"exact resistance capped at n={cap}; use effective_resistance_approx")
    n, m = int(g.n), int(g.m)
    if n == 1 or m == 0:
        return ResistanceTable(values=np.zeros(m), method="exact")
    dev = require_cuda()
    csr = device_csr(g, dev)
    ip = csr.indptr.long()
    ix = csr.indices.long()
    deg = (ip[1:] - ip[:-1]).double()
    lap = torch.zeros((n, n), dtype=torch.float64, device=dev)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), ip[1:] - ip[:-1])
    lap[rows, ix] = -1.0
    lap[torch.arange(n, device=dev), torch.arange(n, device=dev)] = deg
    grounded = lap[1:, 1:]
    X = torch.cholesky_inverse(torch.linalg.cholesky(grounded)).contiguous()
    out = torch.empty(m, dtype=torch.float64, device=dev)
    _lib.call("gu_resistance_exact_gather", m, _lib.ptr(_edges_dev(g, dev)), _lib.ptr(X), n,
              _lib.ptr(out), stream_ptr(dev))
    return ResistanceTable(values=out.cpu().numpy(), method="exact")


def effective_resistance_approx(g, epsilon, seed=0, sketch_factor=4.0, maxiter=2000):
    """Sketch-based effective resistances with ~epsilon relative error
    (sparsify.py:87-143): q = ceil(sketch_factor log2 n / epsilon^2)
    Rademacher projections, q Jacobi-PCG solves (rtol 1e-8) in one block
    solve on the GPU.  Raises SolverError if CG does not converge."""
    if not (0.0 < epsilon < 1.0):
        raise ValueError("epsilon must lie in (0, 1)")
    _require_connected(g)
    n, m = int(g.n), int(g.m)
    if m == 0:
        return ResistanceTable(values=np.zeros(0), method="approx")
    q = max(1, math.ceil(sketch_factor * math.log2(max(n, 2)) / epsilon ** 2))
    dev = require_cuda()
    csr = device_csr(g, dev)
    lib = _lib.load()
    ws = workspace(lib.gu_resistance_sketch_workspace_size(n, q), dev)
    out = torch.empty(m, dtype=torch.float64, device=dev)
    iters = ctypes.c_int32(0)
    resid = ctypes.c_double(0.0)
    r = lib.gu_resistance_sketch(n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), m,
                                 _lib.ptr(_edges_dev(g, dev)), q, int(seed) & (2**64 - 1), 1e-8,
                                 int(maxiter), _lib.ptr(out), ctypes.byref(iters), ctypes.byref(resid),
                                 _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    if r == _lib.GU_ERR_UNSUPPORTED:  # CG not converged within maxiter
        raise SolverError(f"CG did not converge within {maxiter} iterations "
                          f"(residual {resid.value:.3e})", resid.value)
    _lib.check("gu_resistance_sketch", r)
    return ResistanceTable(values=out.cpu().numpy(), method="approx")


def sparsifier_target(n, m):
    """Edge budget min(m, ceil(n * log2 n)) of the sparsifier."""
    if n < 2:
        return m
    return min(m, math.ceil(n * math.log2(n)))


def sparsify(g, resistances):
    """Spectral sparsifier (sparsify.py:176-205): the maximum-resistance
    spanning tree, then non-tree edges in decreasing resistance (ties by
    canonical edge order) up to min(m, ceil(n log2 n)) edges."""
    if len(resistances) != g.m:
        raise ValueError("resistance table does not align with graph edges")
    target = sparsifier_target(g.n, g.m)
    if g.m <= target:
        return g
    _require_connected(g)
    n, m = int(g.n), int(g.m)
    dev = require_cuda()
    lib = _lib.load()
    r = torch.from_numpy(np.ascontiguousarray(resistances.values, dtype=np.float64)).to(dev)
    keep = torch.empty(m, dtype=torch.uint8, device=dev)
    ws = workspace(lib.gu_sparsify_workspace_size(n, m), dev)
    tree = ctypes.c_int32(0)
    _lib.call("gu_sparsify_select", n, m, _lib.ptr(_edges_dev(g, dev)), _lib.ptr(r), int(target),
              _lib.ptr(keep), ctypes.byref(tree), _lib.ptr(ws), ws.numel(), stream_ptr(dev))
    kept = np.asarray(g.edges)[keep.cpu().numpy().astype(bool)]
    return graph_from_edges(n, kept, labels=getattr(g, "labels", ()))


def compute_resistances(g, method="auto", epsilon=0.5, seed=0, exact_cap=20000, auto_cutoff=4000):
    """Effective resistances by the requested method (layout.py:384-397)."""
    if method == "auto":
        method = "exact" if g.n <= auto_cutoff else "approx"
    if method == "exact":
        return effective_resistance_exact(g, cap=exact_cap)
    if method == "approx":
        return effective_resistance_approx(g, epsilon=epsilon, seed=seed)
    raise ValueError(f"unknown resistance method {method!r}")


def make_sparsifier(g, method="auto", epsilon=0.5, seed=0):
    """Sparsify ``g`` to min(m, ceil(n log2 n)) edges (identity if already
    that sparse, layout.py:400-406)."""
    if g.m <= sparsifier_target(g.n, g.m):
        return g
    res = compute_resistances(g, method=method, epsilon=epsilon, seed=seed)
    return sparsify(g, res)
