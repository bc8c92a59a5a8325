"""Small hub-heavy graph through smooth_knn_weights (sanitizer target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_19703_b200 as gu
from oracle import oracle as O
g = gu.synth_graph("scale_free", int(sys.argv[1]) if len(sys.argv) > 1 else 3000, seed=5, m0=2)
_, knn = gu.partial_bfs(g, 15, seed=3)
gk = gu.smooth_knn_weights(knn)
ip, dst, dist = O.partial_bfs(g, 15, seed=3)
o = O.smooth_knn_weights(g.n, ip, dst, dist, 15)
print("E", gk.edge_count, len(o["sym_src"]), np.array_equal(gk.sym_src, o["sym_src"]),
      np.array_equal(gk.sym_dst, o["sym_dst"]), float(np.max(np.abs(gk.sym_w - o["sym_w"]))))
