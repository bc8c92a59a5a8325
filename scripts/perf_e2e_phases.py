"""Phase timing inside partial_bfs (c5) to locate host/launch overheads."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures, _lib
from paper_2509_19703_b200.device import device_csr, stream_ptr, workspace
from paper_2509_19703_b200.neighbors import partial_bfs_records, _pack

g = fixtures.config_graph("c5")
csr = device_csr(g)
def T():
    torch.cuda.synchronize(); return time.perf_counter()
for rep in range(4):
    t0 = T()
    n = g.n
    nbr = torch.empty((n, 15), dtype=torch.int32, device="cuda"); dist = torch.empty_like(nbr)
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    t1 = T()
    tw = int(max(1, min(148 * 8, (256 << 20) // max(8 * n, 1))))
    ws = workspace(_lib.load().gu_partial_bfs_workspace_size(n, n, tw), "cuda")
    t2 = T()
    _lib.call("gu_partial_bfs_knn", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), 15, 4, 0, n,
              _lib.ptr(nbr), _lib.ptr(dist), _lib.ptr(cnt), None, _lib.ptr(ws), ws.numel(), tw, stream_ptr())
    t3 = T()
    short = int((cnt < 15).sum().item())
    t4 = T()
    ip, d, dd = _pack(n, 15, nbr, dist, cnt, torch.device("cuda"), {})
    t5 = T()
    print(f"rep {rep}: alloc {1e3*(t1-t0):.2f} ws {1e3*(t2-t1):.2f} ws_bytes={ws.numel()/1e6:.0f}MB kernel {1e3*(t3-t2):.2f} short {1e3*(t4-t3):.2f} pack {1e3*(t5-t4):.2f} ms", flush=True)
    del nbr, dist, cnt, ws
