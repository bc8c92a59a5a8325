"""Check (c) report: final-layout quality of the GPU pipeline on BASELINE c1
(GUMAP: 50x50 grid, full BFS kNN k=15, random init [-10, 10], 200 full
epochs, 5 negatives, lr 1, min_dist 0.1) over seeds 0..S-1, against the
reference's own 20-seed distribution frozen in tests/golden/quality_c1.npz.

Metrics are the oracle restatements of graph_umap.metrics (pinned to the
reference's values on its own layouts).  Writes a JSON summary (default
profiles/r01_quality_c1.json) with per-metric means, the GPU/reference mean
ratio and a bootstrap 95% CI of that ratio.
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402
from oracle.metrics import count_crossings, neighborhood_preservation, stress  # noqa: E402


def main(nseeds=20, out=os.path.join(ROOT, "profiles", os.environ.get("QOUT", "r01_quality_c1.json"))):
    z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c1.npz"))
    ref = np.stack([z["np_"], z["stress"], z["crossings"]], axis=1)
    g = gu.synth_graph("grid", 2500)
    dset = gu.all_pairs_bfs(g)
    hop = np.array(dset.matrix, dtype=np.float64)
    vals, secs = [], []
    for seed in range(nseeds):
        t0 = time.perf_counter()
        knn = gu.knn_from_full_distances(dset, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0),
                               gu.OptimizerConfig(iterations=200, k=15, seed=seed), tag="GUMAP")
        secs.append(time.perf_counter() - t0)
        c = lay.coords
        vals.append((neighborhood_preservation(g, c, hop), stress(g, c, hop), count_crossings(g, c)))
    v = np.array(vals)
    rng = np.random.default_rng(0)
    boot = []
    for _ in range(2000):
        a = v[rng.integers(0, len(v), len(v))].mean(axis=0)
        b = ref[rng.integers(0, len(ref), len(ref))].mean(axis=0)
        boot.append(a / b)
    boot = np.array(boot)
    names = ["neighborhood_preservation", "stress", "crossings"]
    res = {"config": "c1 GUMAP grid 50x50, k=15, 200 full epochs, random init, seeds 0..%d" % (nseeds - 1),
           "gpu_seeds": nseeds, "reference_seeds": int(ref.shape[0]),
           "gpu_pipeline_seconds_mean": float(np.mean(secs)), "metrics": {}}
    for i, nm in enumerate(names):
        res["metrics"][nm] = {
            "gpu_mean": float(v[:, i].mean()), "gpu_cv": float(v[:, i].std(ddof=1) / v[:, i].mean()),
            "ref_mean": float(ref[:, i].mean()), "ref_cv": float(ref[:, i].std(ddof=1) / ref[:, i].mean()),
            "ratio": float(v[:, i].mean() / ref[:, i].mean()),
            "ratio_ci95": [float(np.percentile(boot[:, i], 2.5)), float(np.percentile(boot[:, i], 97.5))],
            "higher_is_better": nm == "neighborhood_preservation"}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
