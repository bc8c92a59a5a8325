import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgumap.so")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def split(arr, off, i):
    return arr[off[i]:off[i + 1]]


def golden_graphs(name):
    """Yield (graph, k, seed, expected dict) from a *_small.npz fixture."""
    from paper_2509_19703_b200.graph import graph_from_edges

    z = load_golden(name)
    for i in range(z["n"].shape[0]):
        e = split(z["edges"], z["edges_off"], i).reshape(-1, 2)
        g = graph_from_edges(int(z["n"][i]), e)
        exp = dict(indptr=split(z["indptr"], z["indptr_off"], i),
                   dst=split(z["dst"], z["dst_off"], i),
                   dist=split(z["dist"], z["dst_off"], i))
        if "apsp_sha" in z:
            exp["apsp_sha"] = str(z["apsp_sha"][i])
        yield g, int(z["k"][i]), int(z["seed"][i]), exp


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O
