"""e2e breakdown of partial_bfs through the public API on c5 (GPU)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures
from paper_2509_19703_b200.device import device_csr
from paper_2509_19703_b200.graph import Graph

g = fixtures.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c5")
for rep in range(4):
    gg = Graph(n=g.n, m=g.m, adj_indptr=np.array(g.adj_indptr), adj_indices=np.array(g.adj_indices), edges=g.edges)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    csr = device_csr(gg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, knn = gu.partial_bfs(gg, 15, seed=4)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ip = knn.indptr; t3 = time.perf_counter()
    dst = knn.dst; t4 = time.perf_counter()
    dd = knn.dist; t5 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):.1f} ms, kernel+pack {1e3*(t2-t1):.1f} ms, indptr {1e3*(t3-t2):.1f}, dst {1e3*(t4-t3):.1f}, dist {1e3*(t5-t4):.1f} ms; total {1e3*(t5-t0):.1f} ms", flush=True)
