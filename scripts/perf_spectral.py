"""Timing of spectral_init: GPU path vs the reference's
CPU algorithm (scipy ARPACK eigsh on the same deflated operator,
layout.py:249-291, restated here as the CPU baseline).

    python scripts/perf_spectral.py [c3 c4 c5] [--cpu c3,c4]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2509_19703_b200 as gu  # noqa: E402


def cpu_spectral_vectors(g, seed=0):
    """layout.py:249-291 (the two deflated eigsh runs) on the host."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    n = g.n
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(17,)))
    deg = np.diff(g.adj_indptr).astype(np.float64)
    inv_sqrt = 1.0 / np.sqrt(deg)
    adj = sp.csr_matrix((np.ones(g.adj_indices.shape[0]), g.adj_indices, g.adj_indptr), shape=(n, n))
    u0 = np.sqrt(deg)
    u0 /= np.linalg.norm(u0)
    basis, found = [u0], []
    for _ in range(2):
        bmat = np.column_stack(basis)

        def matvec(x, bmat=bmat):
            y = x - bmat @ (bmat.T @ x)
            y = y + inv_sqrt * (adj @ (inv_sqrt * y))
            return y - bmat @ (bmat.T @ y)

        op = spla.LinearOperator((n, n), matvec=matvec, dtype=np.float64)
        v0 = rng.standard_normal(n)
        v0 -= bmat @ (bmat.T @ v0)
        _, vec = spla.eigsh(op, k=1, which="LM", v0=v0, maxiter=10 * n, tol=1e-6, ncv=32)
        v = vec[:, 0]
        v -= bmat @ (bmat.T @ v)
        v /= np.linalg.norm(v)
        basis.append(v)
        found.append(v)
    return np.column_stack(found)


def main(args):
    cpu = set()
    if "--cpu" in args:
        i = args.index("--cpu")
        cpu = set(args[i + 1].split(","))
        args = args[:i] + args[i + 2:]
    for name in args or ["c3", "c4", "c5"]:
        g = gu.config_graph(name)
        gu.spectral_init(gu.synth_graph("scale_free", 2000, seed=1, m0=2), seed=0)  # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        lay = gu.spectral_init(g, seed=0)
        torch.cuda.synchronize()
        res = {"config": name, "n": g.n, "m": g.m, "gpu_s": round(time.perf_counter() - t, 3),
               "extent": float(np.abs(lay.coords).max())}
        if name in cpu:
            t = time.perf_counter()
            cpu_spectral_vectors(g)
            res["cpu_eigsh_s"] = round(time.perf_counter() - t, 3)
            res["cpu_threads"] = os.cpu_count()
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
