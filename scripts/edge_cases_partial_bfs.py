"""Edge-case graphs through partial_bfs vs the oracle (GPU): n=1, no edges, K20 at k up to n, a star with k around 32, a path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, warnings
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200.fixtures import canonical_edges, graph_from_edges
from oracle import oracle as O
def check(g, k, seed=3):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, knn = gu.partial_bfs(g, k, seed=seed)
        ip, dst, dist = O.partial_bfs(g, k, seed=seed)
    ok = np.array_equal(knn.indptr, ip) and np.array_equal(knn.dst, dst) and np.array_equal(knn.dist, dist)
    return ok
cases = []
cases.append(("n1", graph_from_edges(1, canonical_edges(1, np.zeros((0,2),np.int64))), 5))
cases.append(("n2 no edges", graph_from_edges(2, canonical_edges(2, np.zeros((0,2),np.int64))), 1))
K = 20; pairs = np.array([(i,j) for i in range(K) for j in range(i+1,K)])
gK = graph_from_edges(K, canonical_edges(K, pairs))
for k in (1, 15, 19, 25): cases.append((f"K20 k={k}", gK, k))
n=1000; star = graph_from_edges(n, canonical_edges(n, np.stack([np.zeros(n-1,np.int64), np.arange(1,n)],1)))
for k in (15, 32, 33): cases.append((f"star1000 k={k}", star, k))
path = graph_from_edges(300, canonical_edges(300, np.stack([np.arange(299), np.arange(1,300)],1)))
cases.append(("path300 k=15", path, 15))
for name, g, k in cases:
    print(name, check(g, k))
