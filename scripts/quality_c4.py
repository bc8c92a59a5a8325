"""Check (c) at 1M scale (BASELINE c4: SBM 1M fixture, random init, partial
BFS kNN k=15, 200 epochs at the default samp=0.9): sampled NP and stress
(GPU metrics over the fixed sources, the oracle's estimators) of the GPU
layouts vs the reference's own c4 layouts
(tests/golden/quality_c4.npz).  Mean ratios with bootstrap 95% CIs ->
profiles/r01_quality_c4.json.

    python scripts/quality_c4.py [S]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import metrics as M  # noqa: E402


def main(nseeds):
    z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c4.npz"))
    ref = np.stack([z["np_"], z["stress"]], axis=1)
    src = z["sources"]
    g = gu.config_graph("c4")
    vals = []
    for seed in range(nseeds):
        _, knn = gu.partial_bfs(g, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0),
                                  gu.OptimizerConfig(iterations=200, k=15, seed=seed))
        vals.append((M.neighborhood_preservation(g, lay, sources=src),
                     M.stress(g, lay, sources=src)))
        print("gpu c4 seed", seed, vals[-1], flush=True)
    v = np.array(vals)
    rng = np.random.default_rng(0)
    boot = np.array([v[rng.integers(0, len(v), len(v))].mean(axis=0) /
                     ref[rng.integers(0, len(ref), len(ref))].mean(axis=0) for _ in range(2000)])
    res = {"config": "c4 SBM(1M, 20 blocks, 8 / 2), partial BFS k=15, 200 epochs at samp 0.9, "
                     "random init; sampled NP / stress over 2000 fixed sources",
           "gpu_seeds": nseeds, "reference_seeds": int(ref.shape[0]), "metrics": {}}
    for i, nm in enumerate(["neighborhood_preservation", "stress"]):
        res["metrics"][nm] = {"gpu_mean": float(v[:, i].mean()), "ref_mean": float(ref[:, i].mean()),
                              "ratio": float(v[:, i].mean() / ref[:, i].mean()),
                              "ratio_ci95": [float(np.percentile(boot[:, i], 2.5)),
                                             float(np.percentile(boot[:, i], 97.5))]}
    with open(os.path.join(ROOT, "profiles", "r01_quality_c4.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
