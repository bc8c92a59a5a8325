"""Exact check (c) at c3 for several Hogwild concurrency caps
(GU_SGD_CONCURRENCY_DIV = n / cap): GPU metrics of 5 GPU seeds vs the
reference's seeds in tests/golden/quality_c3_full.npz.
    python scripts/quality_c3_sweep.py [div ...] -> profiles/r01_quality_c3_sweep.json
"""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import metrics as M  # noqa: E402


def main(divs, nseeds=5):
    z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c3_full.npz"))
    ref = np.stack([z["np_"], z["stress"], z["crossings"].astype(np.float64)], axis=1)
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    out = {"reference_seeds": int(ref.shape[0]), "ref_mean": ref.mean(axis=0).tolist(),
           "ref_sd": ref.std(axis=0, ddof=1).tolist(), "gpu": {}}
    for div in divs:
        os.environ["GU_SGD_CONCURRENCY_DIV"] = str(div)
        vals, secs = [], []
        for seed in range(nseeds):
            _, knn = gu.partial_bfs(g, 15, seed=seed)
            gk = gu.smooth_knn_weights(knn)
            E = gk.edge_count
            cfg = gu.OptimizerConfig(iterations=200, k=15, seed=seed,
                                     samp=math.log(0.1 * E) / math.log(E))
            t = time.perf_counter()
            lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0), cfg)
            secs.append(time.perf_counter() - t)
            vals.append((M.neighborhood_preservation(g, lay), M.stress(g, lay), M.count_crossings(g, lay)))
        v = np.array(vals, dtype=np.float64)
        rng = np.random.default_rng(0)
        boot = np.array([v[rng.integers(0, len(v), len(v))].mean(axis=0) /
                         ref[rng.integers(0, len(ref), len(ref))].mean(axis=0) for _ in range(2000)])
        out["gpu"][str(div)] = {"mean": v.mean(axis=0).tolist(), "sd": v.std(axis=0, ddof=1).tolist(),
                                "ratio": (v.mean(axis=0) / ref.mean(axis=0)).tolist(),
                                "ratio_ci95_lo": np.percentile(boot, 2.5, axis=0).tolist(),
                                "ratio_ci95_hi": np.percentile(boot, 97.5, axis=0).tolist(),
                                "sgd_seconds": float(np.mean(secs))}
        print(div, json.dumps(out["gpu"][str(div)]), flush=True)
    with open(os.path.join(ROOT, "profiles", "r01_quality_c3_sweep.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main([float(x) for x in sys.argv[1:]] or [16, 4, 2, 1])
