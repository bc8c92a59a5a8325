"""Source-sharded BFS-kNN over several GPUs.

Every BFS source is independent and its RNG stream is per source
(_kernels.py:77 ``seed + gamma*(s+1)``; neighbors.py:213-215
``spawn_key=(v,)``), so splitting the source range across ranks reproduces
the single-GPU records bit for bit.  One process per GPU, the graph CSR
replicated in each GPU's HBM; each rank computes the fixed-size records
(k neighbour ids, k distances, count) of its contiguous source range straight
into padded per-rank buffers, and ``all_gather`` of those buffers (NCCL over
NVLink/NVSwitch on B200s, gloo in the CPU tests) hands every rank the full kNN
lists for C1 -- no packing copies on the data path.  C2 (SGD) stays on one
GPU.

The buffer / gather code below is backend-agnostic torch, so the exchange is
testable with gloo on CPU tensors; the records themselves only ever come
from the GPU kernels (or, in tests, from the oracle).
"""

import torch
import torch.distributed as dist

from .device import device_csr, require_cuda
from .neighbors import DirectedKnn, _pack, _warn_short, full_knn_records, partial_bfs_records


def shard_range(n, rank, world, align=1):
    """Contiguous source range [begin, end) of ``rank`` and the padded
    per-rank record count (a multiple of ``align``; 64 = one bitset word)."""
    blocks = -(-n // align)
    per = -(-blocks // world) * align
    begin = min(rank * per, n)
    end = min(begin + per, n)
    return begin, end, per


def shard_buffers(per, k, device, dtype=torch.int32):
    """Padded per-rank record buffers (nbr [per, k], dist [per, k], cnt [per])
    that the kernels write in place (first ns rows) and all_gather sends as
    they are; padding rows only ever sit past n, in the last rank's block."""
    return (torch.empty((per, k), dtype=dtype, device=device),
            torch.empty((per, k), dtype=dtype, device=device),
            torch.zeros(per, dtype=dtype, device=device))


def gather_shards(bufs, n, group=None, k=None):
    """all_gather each padded buffer -> the first n rows of the
    concatenation: (nbr [n, k], dist [n, k], cnt [n]).  Hop distances of a
    kNN record never exceed k (every BFS level up to the k-th neighbour holds
    at least one vertex), so for k <= 255 the distance block travels as uint8
    and is widened after the gather: a third less traffic on the link."""
    world = dist.get_world_size(group)
    narrow = k is not None and k <= 255
    out = []
    for j, b in enumerate(bufs):
        send = b
        if j == 1 and narrow:
            send = b.to(torch.uint8)
        send = send.contiguous()
        full = torch.empty((world * send.shape[0],) + tuple(send.shape[1:]), dtype=send.dtype,
                           device=send.device)
        dist.all_gather_into_tensor(full, send, group=group)
        full = full[:n]
        out.append(full.to(b.dtype) if full.dtype != b.dtype else full)
    return tuple(out)


def sharded_knn(g, k, seed=0, mode="partial", group=None):
    """kNN lists of every vertex, sources sharded over the process group.

    mode="partial": partial_bfs records (SL / SSSL); mode="full": fused
    full-BFS kNN records (GUMAP / SS).  Returns a DirectedKnn (device
    resident) identical on every rank and identical to the single-GPU
    result.
    """
    dev = require_cuda()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = int(g.n)
    csr = device_csr(g, dev)
    if mode == "partial":
        k_eff = min(k, n - 1) if n > 1 else 0
        begin, end, per = shard_range(n, rank, world, align=1)
    elif mode == "full":
        k_eff = k
        begin, end, per = shard_range(n, rank, world, align=64)
    else:
        raise ValueError(f"unknown mode {mode!r}")
    bufs = shard_buffers(per, max(k_eff, 1), dev)
    ns = end - begin
    out = (bufs[0][:ns], bufs[1][:ns], bufs[2][:ns])
    if mode == "partial":
        partial_bfs_records(csr, k_eff, seed, begin, end, out=out)
    else:
        full_knn_records(csr, k_eff, seed, begin, end, out=out)
    nbr, dd, cnt = gather_shards(bufs, n, group, k=max(k_eff, 1))
    short = int((cnt < k_eff).sum().item()) if n else 0
    if rank == 0:
        _warn_short(short)
    indptr, dst, dist_ = _pack(n, k_eff, nbr, dd, cnt, dev)
    return DirectedKnn(n=n, k=k, _dev=dict(indptr=indptr, dst=dst, dist=dist_))
