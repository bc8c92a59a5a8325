"""world_size-2 gloo test of the source-sharded record exchange (CPU).

Each rank produces the fixed-size kNN records of its source shard (here with
the oracle, the checker; on B200s the GPU kernels write them in place) into
the padded shard buffers and all-gathers them through
paper_2509_19703_b200.distributed.  The gathered records must equal the single-process result
bit for bit (per-source RNG streams make sharding exact).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2509_19703_b200 import fixtures as F
    from paper_2509_19703_b200.distributed import gather_shards, shard_buffers, shard_range

    g = F.scale_free(3000, seed=7, m0=2) if mode == "partial" else F.grid(900)
    k = 15
    align = 1 if mode == "partial" else 64
    b, e, per = shard_range(g.n, rank, world, align)
    if mode == "partial":
        nbr, dd, cnt = O.partial_bfs_raw(g, k, seed=3, src_begin=b, src_end=e, nthreads=2)
    else:
        nbr, dd, cnt = O.full_knn(g, k, seed=3, src_begin=b, src_end=e, nthreads=2, packed=False)
    bufs = shard_buffers(per, k, torch.device("cpu"))
    ns = e - b
    bufs[0][:ns] = torch.from_numpy(nbr.reshape(-1, k))   # the kernels write these rows in place
    bufs[1][:ns] = torch.from_numpy(dd.reshape(-1, k))
    bufs[2][:ns] = torch.from_numpy(cnt)
    n2, d2, c2 = gather_shards(bufs, g.n, k=k)  # distances travel as uint8
    np.savez(os.path.join(out_dir, f"{mode}_{rank}.npz"), nbr=n2.numpy(), dist=d2.numpy(),
             cnt=c2.numpy())
    dist.destroy_process_group()


def _worker_exchange(rank, world, port, mode, out_dir):
    """exchange_records (interleaved rounds, async gathers) with the oracle
    as the record producer."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2509_19703_b200 import fixtures as F
    from paper_2509_19703_b200.distributed import exchange_records

    g = F.scale_free(3000, seed=7, m0=2) if mode == "partial" else F.grid(900)
    k = 15
    calls = []

    def compute(b, e, out):
        calls.append((b, e))
        if mode == "partial":
            nbr, dd, cnt = O.partial_bfs_raw(g, k, seed=3, src_begin=b, src_end=e, nthreads=2)
        else:
            nbr, dd, cnt = O.full_knn(g, k, seed=3, src_begin=b, src_end=e, nthreads=2, packed=False)
        out[0][...] = torch.from_numpy(nbr.reshape(-1, k))
        out[1][...] = torch.from_numpy(dd.reshape(-1, k))
        out[2][...] = torch.from_numpy(cnt)

    n2, d2, c2 = exchange_records(compute, g.n, k, torch.device("cpu"), chunks=3,
                                  align=1 if mode == "partial" else 64)
    np.savez(os.path.join(out_dir, f"x{mode}_{rank}.npz"), nbr=n2.numpy(), dist=d2.numpy(),
             cnt=c2.numpy(), calls=np.array(calls, dtype=np.int64).reshape(-1, 2))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["partial", "full"])
def test_exchange_records_match_single_process(tmp_path, mode):
    """Interleaved rounds with overlapped gathers reproduce the single-process
    records, every source computed exactly once across ranks."""
    from oracle import oracle as O
    from paper_2509_19703_b200 import fixtures as F

    O.build()
    world = 2
    mp.spawn(_worker_exchange, args=(world, _free_port(), mode, str(tmp_path)), nprocs=world,
             join=True)
    g = F.scale_free(3000, seed=7, m0=2) if mode == "partial" else F.grid(900)
    if mode == "partial":
        nbr, dd, cnt = O.partial_bfs_raw(g, 15, seed=3, nthreads=2)
    else:
        nbr, dd, cnt = O.full_knn(g, 15, seed=3, nthreads=2, packed=False)
    covered = np.zeros(g.n, dtype=np.int64)
    for r in range(world):
        z = np.load(tmp_path / f"x{mode}_{r}.npz")
        assert np.array_equal(z["nbr"].reshape(-1), nbr)
        assert np.array_equal(z["dist"].reshape(-1), dd)
        assert np.array_equal(z["cnt"], cnt)
        for b, e in z["calls"]:
            covered[b:e] += 1
    assert np.all(covered == 1)


@pytest.mark.parametrize("mode", ["partial", "full"])
def test_sharded_records_match_single_process(tmp_path, mode):
    from oracle import oracle as O
    from paper_2509_19703_b200 import fixtures as F

    O.build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), mode, str(tmp_path)), nprocs=world, join=True)
    g = F.scale_free(3000, seed=7, m0=2) if mode == "partial" else F.grid(900)
    if mode == "partial":
        nbr, dd, cnt = O.partial_bfs_raw(g, 15, seed=3, nthreads=2)
    else:
        nbr, dd, cnt = O.full_knn(g, 15, seed=3, nthreads=2, packed=False)
    for r in range(world):
        z = np.load(tmp_path / f"{mode}_{r}.npz")
        assert np.array_equal(z["nbr"].reshape(-1), nbr)
        assert np.array_equal(z["dist"].reshape(-1), dd)
        assert np.array_equal(z["cnt"], cnt)
