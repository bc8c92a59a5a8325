"""C1 (smooth_knn_weights) device time with CUDA events on a BASELINE
config's kNN graph (GPU): mean of 6 calls after 2 warm-ups."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
g = fixtures.config_graph(name)
_, knn = gu.partial_bfs(g, 15, seed=4)
knn.device("indptr")
for _ in range(2):
    gu.smooth_knn_weights(knn)
ts = []
for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gk = gu.smooth_knn_weights(knn)
    e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{name} packed={os.environ.get('GU_SYM_PACKED', '1')}: C1 {sum(ts)/len(ts):.3f} ms "
      f"(min {min(ts):.3f}) E={gk.edge_count}", flush=True)
