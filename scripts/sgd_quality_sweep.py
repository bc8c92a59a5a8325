import os, sys, time, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import layout as L
from oracle.metrics import count_crossings, neighborhood_preservation, stress
z = np.load('tests/golden/quality_c1.npz')
g = gu.synth_graph("grid", 2500)
dset = gu.all_pairs_bfs(g)
hop = np.array(dset.matrix, dtype=np.float64)
print("ref means", z["np_"].mean(), z["stress"].mean(), z["crossings"].mean())
for div in (0, 2, 8, 32, 128):
    os.environ["GU_SGD_CONCURRENCY_DIV"] = str(div)
    vals = []
    t = time.time()
    for seed in range(4):
        knn = gu.knn_from_full_distances(dset, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0), gu.OptimizerConfig(iterations=200, k=15, seed=seed)).coords
        vals.append((neighborhood_preservation(g, lay, hop), stress(g, lay, hop), count_crossings(g, lay)))
    print("div", div, np.array(vals).mean(axis=0), f"{time.time()-t:.1f}s", flush=True)
