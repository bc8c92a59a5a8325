"""C1 (smooth_knn_weights) phase timing on a BASELINE config (GPU)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures
g = fixtures.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c5")
_, knn = gu.partial_bfs(g, 15, seed=4)
for rep in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    gk = gu.smooth_knn_weights(knn)
    torch.cuda.synchronize(); print(f"rep {rep}: smooth_knn_weights {1e3*(time.perf_counter()-t):.2f} ms E={gk.edge_count}", flush=True)
