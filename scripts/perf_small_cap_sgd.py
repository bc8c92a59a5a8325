"""Small-cap SGD (c1 GUMAP full epochs, c3 SL windowed epochs; cap n/4):
200 epochs through the public optimize_* calls, device-resident graph (GPU)."""
import math, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu

cases = []
g1 = gu.synth_graph("grid", 2500)
gk1 = gu.smooth_knn_weights(gu.knn_from_full_distances(gu.all_pairs_bfs(g1), 15, seed=0))
cases.append(("c1 GUMAP full", g1, gk1, False, 0.9))
g3 = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
_, knn3 = gu.partial_bfs(g3, 15, seed=2)
gk3 = gu.smooth_knn_weights(knn3)
E = gk3.edge_count
cases.append(("c3 SL window", g3, gk3, True, math.log(0.1 * E) / math.log(E)))
for name, g, gk, win, samp in cases:
    cfg = gu.OptimizerConfig(iterations=200, k=15, seed=2, samp=samp)
    init = gu.random_init(g, 2, 10.0)
    f = gu.optimize_sampled if win else gu.optimize_full
    f(gk, init, cfg)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        f(gk, init, cfg)
        torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{name}: 200 epochs {min(ts):.2f} ms",
          flush=True)
