"""Phase breakdown of the e2e partial_bfs call on c5 (pinned host Graph in,
numpy DirectedKnn out): upload, kernel + overlapped row copies, host reads."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures
from paper_2509_19703_b200.device import device_csr
from paper_2509_19703_b200.graph import Graph

g = fixtures.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c5")


def pinned(a):
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    out = t.numpy()
    out[...] = a
    return out


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(12):
    gg = Graph(n=g.n, m=g.m, adj_indptr=pinned(np.asarray(g.adj_indptr)),
               adj_indices=pinned(np.asarray(g.adj_indices)), edges=g.edges)
    t0 = T()
    device_csr(gg)
    t1 = T()
    _, knn = gu.partial_bfs(gg, 15, seed=4)
    t2 = time.perf_counter()
    ip = knn.indptr
    t3 = time.perf_counter()
    dst = knn.dst
    t4 = time.perf_counter()
    dd = knn.dist
    t5 = T()
    print(f"rep {rep}: upload {1e3*(t1-t0):.2f} ms ({(gg.adj_indptr.nbytes+gg.adj_indices.nbytes)/(t1-t0)/1e9:.1f} GB/s)"
          f"  partial_bfs call {1e3*(t2-t1):.2f}  indptr {1e3*(t3-t2):.2f}  dst {1e3*(t4-t3):.2f}"
          f"  dist {1e3*(t5-t4):.2f}  total {1e3*(t5-t0):.2f} ms", flush=True)
