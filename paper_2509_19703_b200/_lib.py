"""ctypes binding of libgumap.so (include/gumap.h).

The library is built in-tree (``paper_2509_19703_b200/_build/libgumap.so``)
by ``__graft_entry__.build()`` / ``make -C paper_2509_19703_b200/csrc``.
There is no CPU fallback: if the library or a CUDA device is missing, every
hot-path call raises.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GU_LIB_PATH") or os.path.join(_HERE, "_build", "libgumap.so")

ABI_VERSION = 1

GU_OK, GU_ERR_ARG, GU_ERR_CUDA, GU_ERR_WORKSPACE, GU_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_c_u64 = ctypes.c_uint64
_c_f64 = ctypes.c_double
_c_f32 = ctypes.c_float
_c_sz = ctypes.c_size_t
_vp = ctypes.c_void_p

# name -> (restype, argtypes), mirrors include/gumap.h
SIGNATURES = {
    "gu_build_graph_workspace_size": (_c_sz, [_c_i64]),
    "gu_build_graph_ids": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _c_sz, _vp]),
    "gu_build_graph_csr": (ctypes.c_int, [_c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _c_sz,
                                          _vp]),
    "gu_lcc_workspace_size": (_c_sz, [_c_i64, _c_i64]),
    "gu_lcc_plan": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "gu_lcc_build": (ctypes.c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _c_sz,
                                    _vp]),
    "gu_resistance_exact_gather": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _vp]),
    "gu_resistance_sketch_workspace_size": (_c_sz, [_c_i64, _c_i32]),
    "gu_resistance_sketch": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _c_i32, _c_u64,
                                            ctypes.c_double, _c_i32, _vp, _vp, _vp, _vp, _c_sz,
                                            _vp]),
    "gu_sparsify_workspace_size": (_c_sz, [_c_i64, _c_i64]),
    "gu_sparsify_select": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp, _c_sz,
                                          _vp]),
    "gu_spectral_degree": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp]),
    "gu_spectral_op_workspace_size": (_c_sz, [_c_i64]),
    "gu_lanczos_workspace_size": (_c_sz, [_c_i64]),
    "gu_lanczos_prepare": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i32, _vp, _vp, _vp, _c_sz, _vp]),
    "gu_lanczos_step": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _c_i32, _vp, _vp, _vp, _c_i32,
                                       _c_i32, _vp, _c_sz, _vp]),
    "gu_spectral_op": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _c_i32, _vp, _vp, _vp, _c_sz,
                                      _vp]),
    "gu_components_workspace_size": (_c_sz, [_c_i64]),
    "gu_connected_components": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "gu_stress_workspace_size": (_c_sz, [_c_i64]),
    "gu_stress": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _c_i32, _vp, _c_i64, _vp, _vp, _c_sz,
                                 _vp]),
    "gu_grid_bytes": (_c_sz, []),
    "gu_crossings_grid": (ctypes.c_int, [_c_i64, _vp, _c_i32, _vp, _vp]),
    "gu_crossings_incidences": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp]),
    "gu_crossings_workspace_size": (_c_sz, [_c_i64, _c_i64, _c_i32]),
    "gu_crossings": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _c_i32, _c_i64, _vp, _vp, _c_sz,
                                    _vp]),
    "gu_np_workspace_size": (_c_sz, [_c_i64, _c_i32]),
    "gu_neighborhood_preservation": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _c_i32, _c_i32, _vp,
                                                    _c_i64, _vp, _vp, _c_sz, _vp]),
    "gu_version": (ctypes.c_int, []),
    "gu_last_error": (ctypes.c_char_p, []),
    "gu_device_sync": (ctypes.c_int, [_vp]),
    "gu_host_is_pinned": (ctypes.c_int, [_vp]),
    "gu_partial_bfs_workspace_size": (_c_sz, [_c_i64, _c_i64, _c_i32]),
    "gu_partial_bfs_knn": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i32, _c_u64, _c_i64, _c_i64,
                                          _vp, _vp, _vp, _vp, _vp, _c_sz, _c_i32, _vp]),
    "gu_partial_bfs_overflow_counts": (ctypes.c_int, [_vp, _c_i64, _vp]),
    "gu_partial_bfs_tier_counts": (ctypes.c_int, [_vp, _c_i64, _vp]),
    "gu_full_bfs_workspace_size": (_c_sz, [_c_i64, _c_i32, _c_i32]),
    "gu_apsp_rows": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _c_i64, _vp, _vp, _c_sz,
                                    _c_i32, _vp]),
    "gu_full_bfs_knn": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i32, _c_u64, _c_i64, _c_i64,
                                       _vp, _vp, _vp, _vp, _vp, _c_sz, _c_i32, _vp]),
    "gu_knn_from_rows_workspace_size": (_c_sz, [_c_i64, _c_i32]),
    "gu_knn_from_rows": (ctypes.c_int, [_c_i64, _vp, _c_i64, _c_i64, _c_i32, _c_u64, _vp,
                                        _vp, _vp, _vp, _c_sz, _c_i32, _vp]),
    "gu_pack_records": (ctypes.c_int, [_c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _c_sz, _vp]),
    "gu_pack_records_workspace_size": (_c_sz, [_c_i64]),
    "gu_smooth_knn_workspace_size": (_c_sz, [_c_i64]),
    "gu_smooth_knn": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i32, _c_f64, _vp, _vp, _vp, _vp, _c_sz,
                                     _vp]),
    "gu_symmetrize_workspace_size": (_c_sz, [_c_i64, _c_i64]),
    "gu_symmetrize": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     ctypes.POINTER(_c_i64), _vp, _c_sz, _vp]),
    "gu_symmetrize_memo": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                          ctypes.POINTER(_c_i64), _vp, _c_sz, _vp, _c_sz, _vp]),
    "gu_sgd_record_bytes_for": (_c_i32, [_c_i64]),
    "gu_sgd_prepare_edges": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _c_i32, _c_u64,
                                            _vp, _vp, _vp]),
    "gu_sgd_prepare_edges_local": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                                  _c_i64, _c_u64, _vp, _vp, _vp]),
    "gu_bfs_order_workspace_size": (_c_sz, [_c_i64, _c_i64]),
    "gu_bfs_order": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "gu_sgd_neighbor_filter": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp]),
    "gu_random_uniform": (ctypes.c_int, [_c_i64, _c_u64, _c_f64, _c_f64, _vp, _vp]),
    "gu_sgd_neighbor_hash_layout": (ctypes.c_int, [_c_i64, _vp, _vp, ctypes.POINTER(_c_i64), _vp]),
    "gu_sgd_neighbor_hash": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _c_i64, _vp]),
    "gu_sgd_prepare_edges_hash": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _c_u64, _vp, _vp,
                                                 _vp]),
    "gu_sgd_epochs": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _c_i32, _vp, _vp, _vp, _c_f32,
                                     _c_f32, _c_f32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i64,
                                     _c_i32, _c_u64, _c_i64, _vp, _vp]),
    "gu_sgd_epochs_deterministic": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _c_i32, _vp, _vp,
                                                   _vp, _c_f32, _c_f32, _c_f32, _c_i32, _c_i32,
                                                   _c_i32, _c_i32, _c_i64, _c_i32, _c_u64, _c_i64,
                                                   _vp, _vp, _vp]),
    "gu_sgd_visit_order": (ctypes.c_int, [_c_i64, _c_i32, _c_i64, _c_i32, _c_u64, _vp, _vp]),
    "gu_replay_schedule": (ctypes.c_int, [_c_i64, _c_i64, _vp, _vp, _vp, _vp, _c_i32, _vp,
                                          _vp, ctypes.POINTER(_c_i64)]),
    "gu_sgd_replay_f64": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i32,
                                         _c_f64, _c_f64, _c_f64, _vp, _vp, _c_i64, _vp]),
}

_lib = None


class GumapError(RuntimeError):
    """A libgumap call failed (CUDA error, workspace, unsupported input)."""


def load():
    """Load libgumap.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` or `make -C paper_2509_19703_b200/csrc` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.gu_version() != ABI_VERSION:
            raise ImportError(f"libgumap ABI {lib.gu_version()} != {ABI_VERSION}")
        _lib = lib
    return _lib


def check(name, r):
    """Map a libgumap status to the exception the wrappers raise."""
    if r != GU_OK:
        msg = load().gu_last_error().decode(errors="replace")
        if r == GU_ERR_ARG:
            raise ValueError(f"{name}: {msg}")
        raise GumapError(f"{name} failed ({r}): {msg}")
    return r


def call(name, *args):
    """Call a status-returning entry point; map failures to exceptions."""
    return check(name, getattr(load(), name)(*args))


def ptr(t):
    """Device (or host) address of a torch tensor / numpy array; None -> NULL."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()
