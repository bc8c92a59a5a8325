"""Source-sharded BFS-kNN over several GPUs.

Every BFS source is independent and its RNG stream is per source
(_kernels.py:77 ``seed + gamma*(s+1)``; neighbors.py:213-215
``spawn_key=(v,)``), so splitting the source range across ranks reproduces
the single-GPU records bit for bit.  One process per GPU, the graph CSR
replicated in each GPU's HBM; each rank computes the fixed-size records
(k neighbour ids, k distances, count) of its sources straight into record
buffers, and ``all_gather`` of those buffers (NCCL over NVLink/NVSwitch on
B200s, gloo in the CPU tests) hands every rank the full kNN lists for C1 --
no packing copies on the data path.  ``exchange_records`` interleaves the
source blocks over a few rounds so each round's gather overlaps the next
round's compute and still lands in source order.  C2 (SGD) stays on one
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


def chunk_rows(n, world, chunks, align=1):
    """Rows per (rank, chunk) of the interleaved source layout: chunk c of
    rank r covers sources [(c*world + r)*ch, (c*world + r + 1)*ch) clipped to
    n, ch a multiple of ``align`` (64 = one bitset word)."""
    per = -(-n // (world * chunks))
    return max(align, -(-per // align) * align)


def exchange_records(compute, n, k, device, group=None, chunks=4, align=1):
    """Source-sharded records of all n sources on every rank, the exchange
    overlapped with the compute.

    The sources are split into ``chunks`` rounds of ``world`` blocks; round c
    gives rank r the block (c*world + r).  ``compute(b, e, out)`` writes the
    records of sources [b, e) into ``out`` = (nbr [e-b, k], dist [e-b, k],
    cnt [e-b]) on the current stream; each round's blocks are then
    all-gathered asynchronously (``async_op``: the collective waits for the
    round's records on its own stream) while the next round computes.  A
    round's gather lands as one contiguous row block of the result, because
    the round's blocks are consecutive in source order: no permutation copy.
    Distances travel as uint8 when k <= 255 (hop distances never exceed k).
    Returns (nbr [n, k], dist [n, k], cnt [n])."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ch = chunk_rows(n, world, chunks, align)
    total = world * chunks * ch
    narrow = k <= 255
    nbr_full = torch.empty((total, k), dtype=torch.int32, device=device)
    dist_full = torch.empty((total, k), dtype=torch.uint8 if narrow else torch.int32, device=device)
    cnt_full = torch.empty(total, dtype=torch.int32, device=device)
    works, keep = [], []
    for c in range(chunks):
        b = (c * world + rank) * ch
        e = min(b + ch, n)
        ns = max(0, e - b)
        nbr_c = torch.empty((ch, k), dtype=torch.int32, device=device)
        dist_c = torch.empty((ch, k), dtype=torch.int32, device=device)
        cnt_c = torch.zeros(ch, dtype=torch.int32, device=device)
        if ns:
            compute(b, e, (nbr_c[:ns], dist_c[:ns], cnt_c[:ns]))
        send_d = dist_c.to(torch.uint8) if narrow else dist_c
        lo, hi = c * world * ch, (c + 1) * world * ch
        for full, send in ((nbr_full, nbr_c), (dist_full, send_d), (cnt_full, cnt_c)):
            works.append(dist.all_gather_into_tensor(full[lo:hi], send, group=group, async_op=True))
        keep.append((nbr_c, send_d, cnt_c))  # alive until the gathers finish
    for w in works:
        w.wait()
    d = dist_full[:n]
    return nbr_full[:n], (d.to(torch.int32) if narrow else d), cnt_full[:n]


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
    elif mode == "full":
        k_eff = k
    else:
        raise ValueError(f"unknown mode {mode!r}")
    kk = max(k_eff, 1)
    if mode == "partial":
        from .device import workspace
        from .neighbors import _tier2_warps
        from . import _lib
        tw = _tier2_warps(n)
        ch = chunk_rows(n, world, 4, 1)
        ws = workspace(_lib.load().gu_partial_bfs_workspace_size(n, ch, tw), dev)

        def compute(b, e, out):
            partial_bfs_records(csr, k_eff, seed, b, e, out=out, tier2_warps=tw, ws=ws)
    else:
        def compute(b, e, out):
            full_knn_records(csr, k_eff, seed, b, e, out=out)
    nbr, dd, cnt = exchange_records(compute, n, kk, dev, group, chunks=4,
                                    align=1 if mode == "partial" else 64)
    short = int((cnt < k_eff).sum().item()) if n else 0
    if rank == 0:
        _warn_short(short)
    indptr, dst, dist_ = _pack(n, k_eff, nbr, dd, cnt, dev)
    return DirectedKnn(n=n, k=k, _dev=dict(indptr=indptr, dst=dst, dist=dist_))
