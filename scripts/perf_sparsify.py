"""Timing of make_sparsifier on the c2 base graph
(ER n=20000, avg degree 200): GPU vs the reference algorithm on the host
(numpy Rademacher signs + scipy Jacobi-PCG per projection, sparsify.py:87-143,
restated here as the CPU baseline; run with --cpu).

    python scripts/perf_sparsify.py [--cpu]
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

from paper_2509_19703_b200 import fixtures as F  # noqa: E402
from paper_2509_19703_b200 import sparsify as S  # noqa: E402


def cpu_sketch(g, epsilon=0.5, seed=0):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    n, m = g.n, g.m
    q = max(1, math.ceil(4.0 * math.log2(max(n, 2)) / epsilon ** 2))
    rng = np.random.default_rng(seed)
    a = sp.csr_matrix((np.ones(len(g.adj_indices)), g.adj_indices, g.adj_indptr), shape=(n, n))
    lap = (sp.diags(np.asarray(a.sum(axis=1)).ravel()) - a).tocsr()
    pre = sp.diags(1.0 / lap.diagonal())
    e = g.edges
    inc = sp.coo_matrix((np.concatenate([np.ones(m), -np.ones(m)]),
                         (np.concatenate([np.arange(m), np.arange(m)]),
                          np.concatenate([e[:, 0], e[:, 1]]))), shape=(m, n)).tocsr()
    signs = rng.choice(np.array([-1.0, 1.0]), size=(q, m)) / math.sqrt(q)
    proj = signs @ inc
    acc = np.zeros(m)
    for i in range(q):
        y, _ = spla.cg(lap, proj[i], rtol=1e-8, atol=0.0, maxiter=2000, M=pre)
        d = y[e[:, 0]] - y[e[:, 1]]
        acc += d * d
    return acc


def main(cpu):
    g = F.erdos_renyi(20000, avg_degree=200, seed=1)
    S.make_sparsifier(F.erdos_renyi(300, avg_degree=30, seed=11))  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = S.effective_resistance_approx(g, epsilon=0.5, seed=0)
    torch.cuda.synchronize()
    t_r = time.perf_counter() - t
    t = time.perf_counter()
    sg = S.sparsify(g, r)
    torch.cuda.synchronize()
    res = {"graph": "c2 base ER(20000, avg deg 200)", "n": g.n, "m": g.m, "kept": sg.m,
           "gpu_resistance_s": round(t_r, 3), "gpu_select_s": round(time.perf_counter() - t, 3)}
    if cpu:
        t = time.perf_counter()
        cpu_sketch(g)
        res["cpu_resistance_s"] = round(time.perf_counter() - t, 2)
        res["cpu_threads"] = os.cpu_count()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main("--cpu" in sys.argv)
