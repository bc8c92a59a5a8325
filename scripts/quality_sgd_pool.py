"""Layout quality of the GPU-filling SGD kernel on a geometric graph (GPU):
run once per library build (GU_LIB_PATH), e.g. the default build (warp-pooled
first tries consumed in place) and one built with -DSGD_POOL=0 (independent
first tries).  NP and stress over 2000 fixed sources, mean over seeds."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures, metrics as M

g = fixtures.rgg(int(sys.argv[1]) if len(sys.argv) > 1 else 700_000, 12.0, seed=5)
_, knn = gu.partial_bfs(g, 15, seed=1)
src = np.random.default_rng(1).choice(g.n, size=2000, replace=False)
nps, sts = [], []
for seed in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    gk = gu.smooth_knn_weights(knn)
    lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0),
                           gu.OptimizerConfig(iterations=200, k=15, seed=seed))
    nps.append(M.neighborhood_preservation(g, lay, sources=src))
    sts.append(M.stress(g, lay, sources=src))
print(f"{os.environ.get('GU_LIB_PATH', 'default build')}: n={g.n} seeds={len(nps)} "
      f"NP mean {np.mean(nps):.5f} sd {np.std(nps, ddof=1):.5f}  "
      f"stress mean {np.mean(sts):.5f} sd {np.std(sts, ddof=1):.5f}", flush=True)
