"""Check (c) at c2 (SS-GUMAP on the G' fixture of ER(20000, 200)) with exact
metrics on both sides: the reference's own final c2 layouts are frozen in
tests/golden/quality_c2.npz (tests/golden/make_golden.py gen_quality_c2), and
the GPU metrics evaluate NP, stress and crossings for them and for this
package's c2 layouts (seeds 0..S-1).  Mean ratios with bootstrap 95% CIs ->
profiles/r01_quality_c2.json.

    python scripts/quality_c2.py [S] [--no-crossings]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import metrics as M  # noqa: E402


def _metrics(g, lay, crossings):
    t = time.perf_counter()
    a = M.neighborhood_preservation(g, lay)
    t1 = time.perf_counter()
    b = M.stress(g, lay)
    t2 = time.perf_counter()
    c = M.count_crossings(g, lay) if crossings else 0
    t3 = time.perf_counter()
    print(f"  np {a:.6f} ({t1 - t:.2f}s) stress {b:.6e} ({t2 - t1:.2f}s) "
          f"crossings {c} ({t3 - t2:.2f}s)", flush=True)
    return a, b, c


def main(nseeds, crossings):
    z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c2.npz"))
    g = gu.config_graph("c2")
    assert g.n == int(z["n"]) and g.m == int(z["m"])
    ref = []
    for i, coords in enumerate(z["layouts"]):
        print("reference seed", i, flush=True)
        ref.append(_metrics(g, gu.Layout(coords=coords, algorithm_tag="SS"), crossings))
    ref = np.array(ref, dtype=np.float64)
    dset = gu.all_pairs_bfs(g)
    vals = []
    for seed in range(nseeds):
        print("gpu seed", seed, flush=True)
        knn = gu.knn_from_full_distances(dset, 15, seed=seed)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_full(gk, gu.random_init(g, seed, 10.0),
                               gu.OptimizerConfig(iterations=200, k=15, seed=seed), tag="SS")
        vals.append(_metrics(g, lay, crossings))
    v = np.array(vals, dtype=np.float64)
    rng = np.random.default_rng(0)
    names = ["neighborhood_preservation", "stress"] + (["crossings"] if crossings else [])
    res = {"config": "c2 SS-GUMAP on G' (ER(20000, 200) sparsifier stand-in), full BFS kNN k=15, "
                     "200 full epochs, random init; exact metrics on G'",
           "gpu_seeds": nseeds, "reference_seeds": int(ref.shape[0]), "metrics": {}}
    for j, name in enumerate(names):
        boot = [v[rng.integers(0, len(v), len(v)), j].mean() /
                ref[rng.integers(0, len(ref), len(ref)), j].mean() for _ in range(2000)]
        res["metrics"][name] = {
            "gpu_mean": float(v[:, j].mean()), "gpu_std": float(v[:, j].std(ddof=1)),
            "ref_mean": float(ref[:, j].mean()), "ref_std": float(ref[:, j].std(ddof=1)),
            "ratio": float(v[:, j].mean() / ref[:, j].mean()),
            "ratio_ci95": [float(np.percentile(boot, 2.5)), float(np.percentile(boot, 97.5))]}
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "r01_quality_c2.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(int(args[0]) if args else 5, "--no-crossings" not in sys.argv)
