"""Source-sharded BFS-kNN over several GPUs.

Every BFS source is independent and its RNG stream is per source
(_kernels.py:77 ``seed + gamma*(s+1)``; neighbors.py:213-215
``spawn_key=(v,)``), so splitting the source range across ranks reproduces
the single-GPU records bit for bit.  One process per GPU, the graph CSR
replicated in each GPU's HBM; each rank computes the fixed-size records
(k neighbour ids, k distances, count) of its contiguous source range, and a
single ``all_gather`` (NCCL over NVLink/NVSwitch on B200s, gloo in the CPU
tests) hands every rank the full kNN lists for C1.  C2 (SGD) stays on one GPU.

The record packing / gather / unpacking below is backend-agnostic torch code,
so the exchange is testable with gloo on CPU tensors; the records
themselves only ever come from the GPU kernels (or, in tests, from the
oracle).
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


def pack_records(nbr, dist_, cnt, per):
    """(nbr[ns,k], dist[ns,k], cnt[ns]) -> int32 [per, 2k+1], zero padded."""
    ns, k = nbr.shape
    rec = torch.zeros((per, 2 * k + 1), dtype=torch.int32, device=nbr.device)
    rec[:ns, :k] = nbr
    rec[:ns, k:2 * k] = dist_
    rec[:ns, 2 * k] = cnt
    return rec


def gather_records(rec, group=None):
    """all_gather of equal-size record blocks -> [world * per, 2k+1]."""
    world = dist.get_world_size(group)
    out = torch.empty((world * rec.shape[0], rec.shape[1]), dtype=rec.dtype, device=rec.device)
    dist.all_gather_into_tensor(out, rec.contiguous(), group=group)
    return out


def unpack_records(allrec, n, k):
    """Inverse of pack_records over the concatenation, first n rows."""
    rows = allrec[:n]
    return rows[:, :k].contiguous(), rows[:, k:2 * k].contiguous(), rows[:, 2 * k].contiguous()


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
        nbr, dd, cnt = partial_bfs_records(csr, k_eff, seed, begin, end)
    elif mode == "full":
        k_eff = k
        begin, end, per = shard_range(n, rank, world, align=64)
        nbr, dd, cnt = full_knn_records(csr, k_eff, seed, begin, end)
    else:
        raise ValueError(f"unknown mode {mode!r}")
    rec = pack_records(nbr, dd, cnt, per)
    allrec = gather_records(rec, group)
    nbr, dd, cnt = unpack_records(allrec, n, max(k_eff, 1))
    short = int((cnt < k_eff).sum().item()) if n else 0
    if rank == 0:
        _warn_short(short)
    indptr, dst, dist_ = _pack(n, k_eff, nbr, dd, cnt, dev)
    return DirectedKnn(n=n, k=k, _dev=dict(indptr=indptr, dst=dst, dist=dist_))
