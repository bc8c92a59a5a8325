"""partial_bfs end to end on c5 from pinned vs pageable host arrays (GPU):
total per call and the CSR-upload share (device_csr alone)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures
from paper_2509_19703_b200.device import device_csr
from paper_2509_19703_b200.graph import Graph

g = fixtures.config_graph("c5")


def pinned(a):
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    out = t.numpy()
    out[...] = a
    return out


def make(kind):
    f = pinned if kind == "pinned" else np.array
    return Graph(n=g.n, m=g.m, adj_indptr=f(np.asarray(g.adj_indptr)),
                 adj_indices=f(np.asarray(g.adj_indices)), edges=g.edges)


for kind in ("pinned", "pageable", "pinned", "pageable"):
    tot, up = [], []
    for i in range(5):
        gg = make(kind)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        device_csr(gg)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        up.append(t1 - t0)
        gg = make(kind)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _, knn = gu.partial_bfs(gg, 15, seed=4)
        knn.indptr, knn.dst, knn.dist
        torch.cuda.synchronize(); tot.append(time.perf_counter() - t0)
    print(f"{kind:9s} upload {1e3*np.median(up):7.2f} ms  partial_bfs e2e {1e3*np.median(tot):7.2f} ms "
          f"(min {1e3*min(tot):.2f})", flush=True)
