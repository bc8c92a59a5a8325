"""Per-call timing of SgdPlan construction (GPU): every C-ABI call of the plan
builder bracketed by synchronisations."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import _lib
from paper_2509_19703_b200.layout import SgdPlan

g = gu.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c5")
_, knn = gu.partial_bfs(g, 15, seed=2)
gk = gu.smooth_knn_weights(knn)
for name in ("sym_src", "sym_dst", "sym_w", "nbr_indptr", "nbr_indices"):
    gk.device(name, torch.device("cuda"))
orig = _lib.call
times = {}


def timed(name, *a):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = orig(name, *a)
    torch.cuda.synchronize()
    times[name] = times.get(name, 0.0) + time.perf_counter() - t
    return r


import paper_2509_19703_b200.layout as L
for rep in range(3):
    times.clear()
    L._lib.call = timed
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    SgdPlan(gk, 2, torch.device("cuda"))
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    L._lib.call = orig
    print(f"rep {rep}: plan {1e3 * tot:.2f} ms: " +
          ", ".join(f"{k} {1e3 * v:.2f}" for k, v in times.items()) +
          f", python/torch rest {1e3 * (tot - sum(times.values())):.2f}", flush=True)
