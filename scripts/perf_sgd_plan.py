"""SgdPlan construction vs epochs for the c3 SL layout (GPU)."""
import math, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200.layout import SgdPlan


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


g = gu.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c3")
_, knn = gu.partial_bfs(g, 15, seed=2)
for rep in range(4):
    gk = gu.smooth_knn_weights(knn)
    E = gk.edge_count
    t0 = T()
    for name in ("sym_src", "sym_dst", "sym_w", "nbr_indptr", "nbr_indices"):
        gk.device(name, torch.device("cuda"))
    t1 = T()
    SgdPlan(gk, 2, torch.device("cuda"))
    t2 = T()
    cfg = gu.OptimizerConfig(iterations=200, k=15, seed=2, samp=math.log(0.1 * E) / math.log(E))
    init = gu.random_init(g, 2, 10.0)
    t3 = T()
    gu.optimize_sampled(gk, init, cfg, tag="SL")
    t4 = T()
    gu.optimize_sampled(gk, init, cfg, tag="SL")
    t5 = T()
    print(f"rep {rep}: device arrays {1e3*(t1-t0):.2f}  plan {1e3*(t2-t1):.2f}  random_init {1e3*(t3-t2):.2f}  "
          f"optimize (new plan) {1e3*(t4-t3):.2f}  optimize (cached plan) {1e3*(t5-t4):.2f} ms", flush=True)
