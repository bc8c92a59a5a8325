"""C1 timing before and after an SGD plan + epochs on c5 (GPU): locates the
slowdown of a C1 call that follows the SGD benchmark."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import fixtures, _lib
from paper_2509_19703_b200.device import stream_ptr
from paper_2509_19703_b200.layout import _plan_for, sgd_concurrency, INT32_MAX

g = fixtures.config_graph("c5")


def c1_time(tag):
    _, knn = gu.partial_bfs(g, 15, seed=4)
    knn.device("indptr")
    gu.smooth_knn_weights(knn)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        gu.smooth_knn_weights(knn)
        torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{tag}: C1 {np.round(ts, 2)} ms; mem alloc {torch.cuda.memory_allocated()/1e9:.1f} GB "
          f"reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)


c1_time("before")
_, knn = gu.partial_bfs(g, 15, seed=4)
gk = gu.smooth_knn_weights(knn)
plan = _plan_for(gk, 4, torch.device("cuda"))
c1_time("after plan")
xy = torch.from_numpy(np.random.default_rng(0).uniform(-10, 10, (g.n, 2)).astype(np.float32)).cuda()
div = torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda")
a, b = gu.fit_ab(0.1, 1.0)
_lib.call("gu_sgd_epochs", plan.n, plan.E, _lib.ptr(xy), _lib.ptr(plan.edges), plan.record_mode,
          _lib.ptr(plan.nbr_indptr), _lib.ptr(plan.nbr_indices), _lib.ptr(plan.filter), float(a),
          float(b), 1.0, 200, 0, 3, 5, plan.E, 0, plan.seed, sgd_concurrency(plan.n),
          _lib.ptr(div), stream_ptr())
torch.cuda.synchronize()
c1_time("after epochs")
del plan, gk, knn, xy
c1_time("after del")
torch.cuda.empty_cache()
c1_time("after empty_cache")
