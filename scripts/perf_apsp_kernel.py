"""A2 rows kernel alone (gu_apsp_rows over all sources into a device n x n
buffer) on c2's G' (GPU), CUDA events; checksum of the first 64 rows."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19703_b200 import _lib, fixtures
from paper_2509_19703_b200.device import device_csr, stream_ptr, workspace

for name in sys.argv[1:] or ["c2"]:
    g = fixtures.config_graph(name)
    csr = device_csr(g)
    n = g.n
    bif = 148 * 2
    ws = workspace(_lib.load().gu_full_bfs_workspace_size(n, 0, bif), csr.device)
    rows = torch.empty((n, n), dtype=torch.int32, device=csr.device)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("gu_apsp_rows", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), 0, n,
                  _lib.ptr(rows), _lib.ptr(ws), ws.numel(), bif, stream_ptr(csr.device))
        e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    alg = ((n + 63) // 64) * 2 * g.m * 12 + 4 * n * n
    print(f"{name}: apsp rows kernel {ms:.3f} ms  {alg / ms / 1e6:.0f} GB/s algorithmic  "
          f"checksum {int(rows[:64].to(torch.int64).sum())}", flush=True)
