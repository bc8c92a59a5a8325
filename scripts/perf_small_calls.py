"""Host-side cost of the public calls on a small graph (c3): partial_bfs and
smooth_knn_weights, with the kernel-only time beside them (GPU)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200.device import device_csr
from paper_2509_19703_b200.neighbors import partial_bfs_records
from paper_2509_19703_b200.graph import Graph


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


g0 = gu.config_graph("c3")
for rep in range(5):
    g = Graph(n=g0.n, m=g0.m, adj_indptr=np.array(g0.adj_indptr), adj_indices=np.array(g0.adj_indices),
              edges=g0.edges)
    t0 = T()
    csr = device_csr(g)
    t1 = T()
    partial_bfs_records(csr, 15, 2, 0, g.n)
    t2 = T()
    _, knn = gu.partial_bfs(g, 15, seed=2)
    t3 = T()
    gk = gu.smooth_knn_weights(knn)
    t4 = T()
    print(f"rep {rep}: csr upload {1e3*(t1-t0):.2f}  records {1e3*(t2-t1):.2f}  partial_bfs (cached csr) "
          f"{1e3*(t3-t2):.2f}  smooth {1e3*(t4-t3):.2f} ms", flush=True)
