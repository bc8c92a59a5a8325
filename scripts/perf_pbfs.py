"""Quick timing of the partial BFS-kNN kernel on BASELINE configs (GPU)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19703_b200 import _lib, fixtures  # noqa: E402
from paper_2509_19703_b200.device import device_csr  # noqa: E402
from paper_2509_19703_b200.neighbors import partial_bfs_records  # noqa: E402
from oracle import oracle as O  # noqa: E402

names = sys.argv[1:] or ["c5", "c4", "c3"]
for name in names:
    t = time.time()
    g = fixtures.config_graph(name)
    gen = time.time() - t
    csr = device_csr(g)
    work = torch.zeros(2, dtype=torch.int64, device="cuda")
    nbr, dist, cnt = partial_bfs_records(csr, 15, 4, 0, g.n, work=work)
    torch.cuda.synchronize()
    sc, ex = work.tolist()
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(6):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        partial_bfs_records(csr, 15, 4, 0, g.n)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    # overflow counts of one call (tier 0 -> 1a -> 1b -> 2)
    from paper_2509_19703_b200.device import workspace, stream_ptr
    lib = _lib.load()
    tw = 64
    ws = workspace(lib.gu_partial_bfs_workspace_size(g.n, g.n, tw), "cuda")
    nb = torch.empty((g.n, 15), dtype=torch.int32, device="cuda"); dd = torch.empty_like(nb)
    cc = torch.empty(g.n, dtype=torch.int32, device="cuda")
    _lib.call("gu_partial_bfs_knn", g.n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), 15, 4, 0,
              g.n, _lib.ptr(nb), _lib.ptr(dd), _lib.ptr(cc), None, _lib.ptr(ws), ws.numel(), tw,
              stream_ptr())
    torch.cuda.synchronize()
    oc = (ctypes.c_int32 * 4)()
    lib.gu_partial_bfs_tier_counts(ctypes.c_void_p(ws.data_ptr()), g.n, oc)
    ovf = list(oc)
    alg = 8 * ex + 4 * sc + 8 * 15 * g.n
    # sample check vs oracle
    s0 = g.n // 3
    on, od, oc = O.partial_bfs_raw(g, 15, 4, s0, s0 + 5000, nthreads=8)
    ok = np.array_equal(nbr[s0:s0 + 5000].cpu().numpy().reshape(-1), on)
    print(f"{name}: n={g.n} m={g.m} gen={gen:.1f}s  {ms:.3f} ms  GTEPS={sc/ms/1e6:.1f}  "
          f"alg={alg/1e9:.3f} GB -> {alg/ms/1e6:.0f} GB/s  sample_ok={ok}  scanned/src={sc/g.n:.1f} "
          f"expanded/src={ex/g.n:.2f} left tier (F,1a,H,C)={ovf}", flush=True)
