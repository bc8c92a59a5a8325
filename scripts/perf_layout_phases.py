"""Phase timing of the c3 SL layout (public API, host arrays in and out):
partial BFS, smooth/union, SGD (200 epochs of 10% windows), result copy.

    python scripts/perf_layout_phases.py [c3]
"""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu  # noqa: E402


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


name = sys.argv[1] if len(sys.argv) > 1 else "c3"
g0 = gu.config_graph(name)
for rep in range(4):
    g = gu.Graph(n=g0.n, m=g0.m, adj_indptr=np.array(g0.adj_indptr), adj_indices=np.array(g0.adj_indices),
                 edges=g0.edges)
    t0 = T()
    _, knn = gu.partial_bfs(g, 15, seed=2)
    t1 = T()
    gk = gu.smooth_knn_weights(knn)
    t2 = T()
    E = gk.edge_count
    cfg = gu.OptimizerConfig(iterations=200, k=15, seed=2, samp=math.log(0.1 * E) / math.log(E))
    lay = gu.optimize_sampled(gk, gu.random_init(g, 2, 10.0), cfg, tag="SL")
    t3 = T()
    c = lay.coords
    t4 = T()
    print(f"{name} rep {rep}: bfs {1e3*(t1-t0):.2f}  smooth {1e3*(t2-t1):.2f}  sgd {1e3*(t3-t2):.2f} "
          f"({1e3*(t3-t2)/200:.1f} us/epoch, window {int(E ** cfg.samp)})  coords {1e3*(t4-t3):.2f}  "
          f"total {1e3*(t4-t0):.2f} ms", flush=True)
