"""Phase timing of the c1 GUMAP layout (public API): full BFS kNN, smooth /
union, SGD (200 full epochs), result copy."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import fixtures  # noqa: E402


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


g = fixtures.grid(2500)
for rep in range(4):
    t0 = T()
    knn = gu.knn_from_full_distances(gu.all_pairs_bfs(g), 15, seed=0)
    t1 = T()
    gk = gu.smooth_knn_weights(knn)
    t2 = T()
    lay = gu.optimize_full(gk, gu.random_init(g, 0, 10.0), gu.OptimizerConfig(iterations=200, k=15, seed=0),
                           tag="GUMAP")
    t3 = T()
    c = lay.coords
    t4 = T()
    print(f"c1 rep {rep}: knn {1e3*(t1-t0):.2f}  smooth {1e3*(t2-t1):.2f}  sgd {1e3*(t3-t2):.2f} "
          f"({1e3*(t3-t2)/200:.1f} us/epoch, E={gk.edge_count})  coords {1e3*(t4-t3):.2f}  total {1e3*(t4-t0):.2f} ms",
          flush=True)
