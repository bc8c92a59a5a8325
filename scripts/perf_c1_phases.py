"""C1 (smooth kNN weights + fuzzy union) timing on a BASELINE config (GPU):
the kNN records stay on the device; the call is timed with CUDA events.

    python scripts/perf_c1_phases.py [c5]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import fixtures  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
g = fixtures.config_graph(name)
_, knn = gu.partial_bfs(g, 15, seed=4)
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gk = gu.smooth_knn_weights(knn)
    e1.record()
    e1.synchronize()
    print(f"{name} rep {rep}: C1 {e0.elapsed_time(e1):.3f} ms  nnz={knn.edge_count} E={gk.edge_count}",
          flush=True)
