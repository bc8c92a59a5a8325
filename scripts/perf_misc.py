"""Timing of the full-BFS kNN (c1, c2), smooth/symmetrize, SGD epochs and the
e2e copy breakdown (GPU)."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu  # noqa: E402
from paper_2509_19703_b200 import fixtures  # noqa: E402
from paper_2509_19703_b200.device import device_csr  # noqa: E402
from paper_2509_19703_b200.neighbors import full_knn_records, partial_bfs_records  # noqa: E402


def cuda_ms(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:]) if len(ts) > 1 else ts[0]


for name in ("c1", "c2"):
    g = fixtures.config_graph(name)
    csr = device_csr(g)
    work = torch.zeros(2, dtype=torch.int64, device="cuda")
    full_knn_records(csr, 15, 0, 0, g.n, work=work)
    torch.cuda.synchronize()
    te = int(work[0])
    ms = cuda_ms(lambda: full_knn_records(csr, 15, 0, 0, g.n))
    ms_apsp = cuda_ms(lambda: gu.all_pairs_bfs(g).matrix, reps=3)
    print(f"{name} full kNN: n={g.n} m={g.m} {ms:.3f} ms  TE={te}  GTEPS={te/ms/1e6:.2f}  "
          f"all_pairs_bfs(+D2H matrix) {ms_apsp:.1f} ms", flush=True)

for name in ("c3", "c4", "c5"):
    g = fixtures.config_graph(name)
    _, knn = gu.partial_bfs(g, 15, seed=4)
    torch.cuda.synchronize()
    ms_c1 = cuda_ms(lambda: gu.smooth_knn_weights(knn), reps=4)
    gk = gu.smooth_knn_weights(knn)
    E = gk.edge_count
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import stream_ptr
    from paper_2509_19703_b200.layout import INT32_MAX, _plan_for, sgd_concurrency
    dev = torch.device("cuda")
    a, b = gu.fit_ab(0.1, 1.0)
    plan = _plan_for(gk, 4, dev)
    xy = torch.from_numpy(np.random.default_rng(0).uniform(-10, 10, (g.n, 2)).astype(np.float32)).to(dev)
    div = torch.full((1,), INT32_MAX, dtype=torch.int32, device=dev)
    samp = math.log(0.1 * E) / math.log(E)
    window = int(math.floor(E ** samp))
    res = []
    for mode, items in (("full", E), ("window10%", window)):
        ep = [0]

        def run(mode=mode):
            e = ep[0] % 200
            ep[0] += 1
            _lib.call("gu_sgd_epochs", plan.n, plan.E, _lib.ptr(xy), _lib.ptr(plan.edges), plan.record_mode,
                      _lib.ptr(plan.nbr_indptr), _lib.ptr(plan.nbr_indices), _lib.ptr(plan.filter), float(a), float(b), 1.0,
                      200, e, e + 1, 5, window if mode != "full" else E, 0 if mode == "full" else 1,
                      plan.seed, sgd_concurrency(plan.n), _lib.ptr(div), stream_ptr(dev))
        ms = cuda_ms(run, reps=6)
        res.append(f"{mode}: {ms:.3f} ms/epoch {items/ms/1e6:.2f} G upd/s ({88*items/ms/1e6:.0f} GB/s alg)")
    print(f"{name}: smooth+sym {ms_c1:.2f} ms (E={E}); SGD " + "; ".join(res), flush=True)

# e2e breakdown on c5
g = fixtures.config_graph("c5")
from paper_2509_19703_b200.graph import Graph
gg = Graph(n=g.n, m=g.m, adj_indptr=np.array(g.adj_indptr), adj_indices=np.array(g.adj_indices), edges=g.edges)
torch.cuda.synchronize()
t0 = time.perf_counter()
csr = device_csr(gg)
torch.cuda.synchronize()
t1 = time.perf_counter()
_, knn = gu.partial_bfs(gg, 15, seed=4)
torch.cuda.synchronize()
t2 = time.perf_counter()
ip, dst, dd = knn.indptr, knn.dst, knn.dist
t3 = time.perf_counter()
print(f"e2e c5 breakdown: upload {1e3*(t1-t0):.1f} ms, kernel+pack {1e3*(t2-t1):.1f} ms, "
      f"D2H+numpy {1e3*(t3-t2):.1f} ms", flush=True)
