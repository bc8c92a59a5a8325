"""Timing of the GPU layout-quality metrics.

    python scripts/perf_metrics.py [c1 c3 c4]

c1: the reference's own layout (tests/golden/quality_c1.npz, its values
checked); c3 / c4: layouts from this package's SL / SSSL pipeline (seed 0).
Prints one JSON line per config with seconds per metric.
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import metrics as M  # noqa: E402


def timed(fn, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    v = fn(*a, **k)
    torch.cuda.synchronize()
    return v, time.perf_counter() - t


def layout_for(name):
    if name == "c1":
        z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c1.npz"))
        return gu.synth_graph("grid", 2500), gu.Layout(coords=z["layout0"]), z
    g = gu.config_graph(name)
    _, knn = gu.partial_bfs(g, 15, seed=0)
    gk = gu.smooth_knn_weights(knn)
    E = gk.edge_count
    samp = math.log(0.1 * E) / math.log(E) if name == "c3" else 0.9
    lay = gu.optimize_sampled(gk, gu.random_init(g, 0, 10.0),
                              gu.OptimizerConfig(iterations=200, k=15, seed=0, samp=samp))
    return g, lay, None


def main(names):
    for name in names:
        g, lay, z = layout_for(name)
        M.neighborhood_preservation(g, gu.Layout(coords=np.zeros((g.n, 2)) + np.arange(g.n)[:, None]))
        res = {"config": name, "n": g.n, "m": g.m}
        v, t = timed(M.neighborhood_preservation, g, lay)
        res.update(np=v, np_s=round(t, 4))
        if g.n <= 1_000_000:
            v, t = timed(M.stress, g, lay)
            res.update(stress=v, stress_s=round(t, 4))
        v, t = timed(M.count_crossings, g, lay)
        res.update(crossings=v, crossings_s=round(t, 4))
        if z is not None:
            res["matches_reference"] = bool(abs(res["np"] - z["np_"][0]) < 1e-12 and
                                            abs(res["stress"] - z["stress"][0]) < 1e-12 and
                                            res["crossings"] == int(z["crossings"][0]))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c3", "c4"])
