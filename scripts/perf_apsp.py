"""all_pairs_bfs(g).matrix timing (A2: the n x n hop matrix, host copy included).

    python scripts/perf_apsp.py [c1 c2]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2"]:
    g = gu.config_graph(name)
    gu.all_pairs_bfs(gu.synth_graph("grid", 400)).matrix  # warm
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        m = gu.all_pairs_bfs(g).matrix
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    te = g.n * 2 * g.m
    print(f"{name}: n={g.n} m={g.m} matrix {m.nbytes / 1e9:.2f} GB  {dt * 1e3:.1f} ms  "
          f"{te / dt / 1e9:.1f} GTEPS (n*2m)  checksum {int(m[: min(g.n, 64)].astype(np.int64).sum())}",
          flush=True)
