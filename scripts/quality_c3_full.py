"""Check (c) at c3 with exact metrics on both sides: GPU metrics of this
package's c3 SL layouts (seeds 0..S-1) vs the oracle metrics of the
reference's own c3 SL layouts (tests/golden/quality_c3_full.npz).
Mean ratios with bootstrap 95% CIs -> profiles/r01_quality_c3_full.json.

    python scripts/quality_c3_full.py [S]
"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import metrics as M  # noqa: E402


def main(nseeds):
    z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c3_full.npz"))
    ref = np.stack([z["np_"], z["stress"], z["crossings"].astype(np.float64)], axis=1)
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    vals = []
    for seed in range(nseeds):
        _, knn = gu.partial_bfs(g, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        E = gk.edge_count
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed,
                                 samp=math.log(0.1 * E) / math.log(E))
        lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0), cfg)
        vals.append((M.neighborhood_preservation(g, lay), M.stress(g, lay), M.count_crossings(g, lay)))
    v = np.array(vals, dtype=np.float64)
    rng = np.random.default_rng(0)
    boot = np.array([v[rng.integers(0, len(v), len(v))].mean(axis=0) /
                     ref[rng.integers(0, len(ref), len(ref))].mean(axis=0) for _ in range(2000)])
    res = {"config": "c3 SL-GUMAP BA(100k, m0=3), 200 epochs, 10% window, random init; exact metrics",
           "gpu_seeds": nseeds, "reference_seeds": int(ref.shape[0]), "metrics": {}}
    for i, nm in enumerate(["neighborhood_preservation", "stress", "crossings"]):
        res["metrics"][nm] = {"gpu_mean": float(v[:, i].mean()), "ref_mean": float(ref[:, i].mean()),
                              "gpu_cv": float(v[:, i].std(ddof=1) / v[:, i].mean()),
                              "ref_cv": float(ref[:, i].std(ddof=1) / ref[:, i].mean()),
                              "ratio": float(v[:, i].mean() / ref[:, i].mean()),
                              "ratio_ci95": [float(np.percentile(boot[:, i], 2.5)),
                                             float(np.percentile(boot[:, i], 97.5))]}
    with open(os.path.join(ROOT, "profiles", "r01_quality_c3_full.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
