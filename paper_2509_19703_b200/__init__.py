"""B200-native hot path of the graph_umap layouts (arXiv 2509.19703).

Drop-in for the reference package's hot-path API
(/root/reference/pkg/src/graph_umap/__init__.py): the same names,
signatures, return types and exceptions for C0/C1/C2 -- full and partial
BFS-kNN, smooth-kNN weights and fuzzy-union symmetrisation, and the UMAP SGD
epochs -- plus the four drivers.  Every array operation runs in
libgumap.so (hand-written sm_100a CUDA) through a ctypes C ABI
(include/gumap.h); there is no CPU fallback.
"""

from .graph import (
    ALGORITHMS,
    Graph,
    GraphError,
    Layout,
    build_graph,
    largest_connected_component,
)
from .neighbors import (
    UNREACHABLE,
    DirectedKnn,
    KnnGraph,
    SparseDistanceSet,
    all_pairs_bfs,
    fuzzy_union,
    knn_from_full_distances,
    partial_bfs,
    smooth_knn_weights,
)
from .layout import (
    DRIVERS,
    ConvergenceError,
    OptimizationDiverged,
    OptimizerConfig,
    RunReport,
    fit_ab,
    make_sparsifier,
    optimize_full,
    optimize_sampled,
    random_init,
    run_gumap,
    run_sl_gumap,
    run_ss_gumap,
    run_sssl_gumap,
    sgd_replay,
    spectral_init,
)
from .fixtures import config_graph


def synth_graph(kind, n, seed=0, **params):
    """grid / scale_free fixtures identical to graph_umap.synth_graph
    (generators.py:116-146); random_regular is not provided."""
    from . import fixtures

    if kind == "grid":
        return fixtures.grid(n)
    if kind == "scale_free":
        return fixtures.scale_free(n, seed=seed, m0=int(params.get("m0", 2)))
    raise GraphError(f"unsupported synthetic kind {kind!r}")


__version__ = "0.1.0"
