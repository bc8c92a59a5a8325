"""Layout quality of the SGD stored-edge orders on a geometric graph (GPU):
plain (one global shuffle, 128-bit Bloom records) vs the BFS locality order
with the window records and block-local shuffles of several sizes.  NP over
2000 fixed sources (exact per-source terms), mean over seeds."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures, metrics as M

g = fixtures.rgg(int(sys.argv[1]) if len(sys.argv) > 1 else 700_000, 12.0, seed=5)
_, knn = gu.partial_bfs(g, 15, seed=1)
src = np.random.default_rng(1).choice(g.n, size=2000, replace=False)
variants = [("plain", {"GU_SGD_RELABEL": "0"}), ("range-global", {"GU_SGD_LOCAL_BLOCK": "0"}),
            ("range-block-65536", {"GU_SGD_LOCAL_BLOCK": "65536"}),
            ("range-block-32768", {"GU_SGD_LOCAL_BLOCK": "32768"}),
            ("range-block-16384", {"GU_SGD_LOCAL_BLOCK": "16384"})]
res = {}
for name, env in variants:
    vals = []
    for seed in range(4):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            gk = gu.smooth_knn_weights(knn)
            lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0),
                                   gu.OptimizerConfig(iterations=200, k=15, seed=seed))
            vals.append(M.neighborhood_preservation(g, lay, sources=src))
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    res[name] = vals
    print(f"{name:20s} NP mean {np.mean(vals):.5f} sd {np.std(vals, ddof=1):.5f} "
          f"ratio-to-plain {np.mean(vals) / np.mean(res['plain']):.4f}", flush=True)
