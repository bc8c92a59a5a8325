"""SGD epoch timing on a BASELINE config's kNN graph (GPU)."""
import math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import _lib, fixtures
from paper_2509_19703_b200.device import stream_ptr
from paper_2509_19703_b200.layout import INT32_MAX, _plan_for, sgd_concurrency

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
g = fixtures.config_graph(name)
_, knn = gu.partial_bfs(g, 15, seed=4)
gk = gu.smooth_knn_weights(knn)
E = gk.edge_count
dev = torch.device("cuda")
a, b = gu.fit_ab(0.1, 1.0)
plan = _plan_for(gk, 4, dev)
xy = torch.from_numpy(np.random.default_rng(0).uniform(-10, 10, (g.n, 2)).astype(np.float32)).to(dev)
div = torch.full((1,), INT32_MAX, dtype=torch.int32, device=dev)
conc = int(os.environ.get("CONC", sgd_concurrency(plan.n)))
for ep in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("gu_sgd_epochs", plan.n, plan.E, _lib.ptr(xy), _lib.ptr(plan.edges), plan.record_mode,
              _lib.ptr(plan.nbr_indptr), _lib.ptr(plan.nbr_indices), _lib.ptr(plan.filter), float(a), float(b), 1.0,
              200, ep, ep + 1, 5, E, 0, plan.seed, conc, _lib.ptr(div), stream_ptr(dev))
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
print(f"{name}: E={E} conc={conc} mode={plan.record_mode} window={getattr(plan, 'mean_window', None)} full epoch {ms:.3f} ms  {E/ms/1e6:.2f} G upd/s", flush=True)
