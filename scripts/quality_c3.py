"""Check (c) at SL scale (BASELINE c3: BA 100k, SL-GUMAP, random init, 200
epochs, 10% window): sampled NP / stress of the GPU layouts vs the
reference's 5-seed values in tests/golden/quality_c3.npz, for several Hogwild
concurrency caps (GU_SGD_CONCURRENCY_DIV = n / cap; 0 = fill the GPU).

    python scripts/quality_c3.py [div ...]     -> profiles/r01_quality_c3.json
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
from oracle import oracle as O  # noqa: E402
from oracle.metrics import sampled_neighborhood_preservation, sampled_stress  # noqa: E402


def main(divs):
    z = np.load(os.path.join(ROOT, "tests", "golden", "quality_c3.npz"))
    src = z["sources"]
    g = gu.synth_graph("scale_free", 100000, seed=2, m0=3)
    O.build()
    rows = O.all_pairs_bfs_rows(g, src)
    res = {"config": "c3 SL-GUMAP BA(100k, m0=3), random init, 200 epochs, 10% window; "
                     "sampled NP / stress over 2000 fixed sources",
           "reference": {"np_mean": float(z["np_"].mean()), "np_sd": float(z["np_"].std(ddof=1)),
                         "stress_mean": float(z["stress"].mean()),
                         "stress_sd": float(z["stress"].std(ddof=1)), "seeds": int(len(z["np_"]))},
           "gpu": {}}
    for div in divs:
        os.environ["GU_SGD_CONCURRENCY_DIV"] = str(div)
        vals, secs = [], []
        for seed in range(len(z["np_"])):
            _, knn = gu.partial_bfs(g, 15, seed=seed)
            gk = gu.smooth_knn_weights(knn)
            E = gk.edge_count
            samp = math.log(0.1 * E) / math.log(E)
            t0 = time.perf_counter()
            lay = gu.optimize_sampled(gk, gu.random_init(g, seed, 10.0),
                                      gu.OptimizerConfig(iterations=200, k=15, seed=seed, samp=samp))
            secs.append(time.perf_counter() - t0)
            vals.append((sampled_neighborhood_preservation(lay.coords, rows, src),
                         sampled_stress(lay.coords, rows, src)))
        v = np.array(vals)
        res["gpu"][str(div)] = {"np_mean": float(v[:, 0].mean()), "np_sd": float(v[:, 0].std(ddof=1)),
                                "stress_mean": float(v[:, 1].mean()),
                                "stress_sd": float(v[:, 1].std(ddof=1)),
                                "np_ratio": float(v[:, 0].mean() / z["np_"].mean()),
                                "stress_ratio": float(v[:, 1].mean() / z["stress"].mean()),
                                "sgd_seconds": float(np.mean(secs))}
        print(div, res["gpu"][str(div)], flush=True)
    out = os.path.join(ROOT, "profiles", "r01_quality_c3.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [16, 4, 1, 0])
