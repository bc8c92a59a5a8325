"""Device CSR store and CUDA plumbing (subsystem 1 of the north star).

A graph's CSR (graph.py:16-71: int64 ``adj_indptr``, int32 ``adj_indices``
sorted per row) is uploaded once per (graph object, device) and kept resident
in HBM with int32 row offsets (every BASELINE config has 2m < 2^31).  The
cache is keyed by object identity with a weak reference, so repeated hot-path
calls on the same Graph (driver stages, benchmark steps) never re-upload.

PyTorch is plumbing only here: device memory, streams, events.
"""

import weakref

import numpy as np
import torch

from . import _lib


def require_cuda(device=None):
    """The hot path has no CPU fallback: fail loudly without a GPU."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_19703_b200 needs a CUDA device (B200, sm_100a); "
                           "no CPU fallback exists")
    _lib.load()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def stream_ptr(device=None):
    return torch.cuda.current_stream(device).cuda_stream


def workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


class DeviceCsr:
    """Resident CSR: ``indptr`` int32[n+1], ``indices`` int32[2m] on device."""

    def __init__(self, n, indptr, indices, device):
        self.n = int(n)
        self.device = device
        self.indptr = indptr
        self.indices = indices
        self.nnz = int(indices.shape[0])

    @classmethod
    def from_arrays(cls, n, adj_indptr, adj_indices, device, non_blocking=False):
        ip = np.asarray(adj_indptr)
        if ip.shape[0] != n + 1:
            raise ValueError("adj_indptr must have n + 1 entries")
        if int(ip[-1]) >= 2**31:
            raise ValueError("device CSR store uses int32 offsets: 2m must be < 2^31")
        ip32 = torch.from_numpy(np.ascontiguousarray(ip, dtype=np.int32))
        ix32 = torch.from_numpy(np.ascontiguousarray(adj_indices, dtype=np.int32))
        if non_blocking:
            ip32, ix32 = ip32.pin_memory(), ix32.pin_memory()
        return cls(n, ip32.to(device, non_blocking=non_blocking),
                   ix32.to(device, non_blocking=non_blocking), device)


_CSR_CACHE = {}


def device_csr(g, device=None):
    """Resident DeviceCsr for graph ``g`` (ours or graph_umap's; duck-typed)."""
    device = require_cuda(device)
    key = (id(g), str(device))
    hit = _CSR_CACHE.get(key)
    if hit is not None:
        ref, csr = hit
        if ref() is g:
            return csr
    csr = DeviceCsr.from_arrays(int(g.n), g.adj_indptr, g.adj_indices, device)
    try:
        ref = weakref.ref(g, lambda _r, k=key: _CSR_CACHE.pop(k, None))
    except TypeError:  # not weak-referenceable: do not cache
        return csr
    _CSR_CACHE[key] = (ref, csr)
    return csr


def to_host(t):
    """Device tensor -> numpy (synchronous)."""
    return t.detach().cpu().numpy()


def to_device(a, dtype, device):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device)
