"""Timing of graph construction and LCC extraction at
c5 scale: build_graph on the c5 edge list (24M pairs, shuffled and with
duplicates / loops) and largest_connected_component, GPU vs the vectorised
numpy host path (the reference's own build_graph is pure-Python sets).

    python scripts/perf_ingest.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_19703_b200 import fixtures as F  # noqa: E402
from paper_2509_19703_b200 import graph as G  # noqa: E402


def timed(fn, *a):
    torch.cuda.synchronize()
    t = time.perf_counter()
    v = fn(*a)
    torch.cuda.synchronize()
    return v, time.perf_counter() - t


def main():
    g5 = F.config_graph("c5")
    rng = np.random.default_rng(0)
    pairs = np.asarray(g5.edges)[rng.permutation(g5.m)]
    pairs = np.concatenate([pairs, pairs[: 1 << 20][:, ::-1], np.repeat(pairs[:1000, :1], 2, axis=1)])
    G.build_graph(pairs[:100000])  # warm
    gd, t_gpu = timed(G.build_graph, pairs)
    orig = G.GPU_BUILD_MIN_PAIRS
    G.GPU_BUILD_MIN_PAIRS = 1 << 62
    gh, t_host = timed(G.build_graph, pairs)
    G.GPU_BUILD_MIN_PAIRS = orig
    same = (np.array_equal(gd.adj_indices, gh.adj_indices) and np.array_equal(gd.edges, gh.edges))
    res = {"pairs": int(pairs.shape[0]), "n": gd.n, "m": gd.m, "build_gpu_s": round(t_gpu, 3),
           "build_host_numpy_s": round(t_host, 3), "identical": bool(same)}
    raw = F.rgg(lcc=False)
    lc, t_lcc = timed(G.largest_connected_component, raw)
    G._gpu_available = lambda: False
    lh, t_lcch = timed(G.largest_connected_component, raw)
    res.update(lcc_in_n=raw.n, lcc_n=lc.n, lcc_gpu_s=round(t_lcc, 3), lcc_host_scipy_s=round(t_lcch, 3),
               lcc_identical=bool(np.array_equal(lc.edges, lh.edges)))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
