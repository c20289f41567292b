"""ctypes bindings for the C-ABI boundary, include/cagra/capi.h.

This is exactly the binding a Python user of the reference would add
(INTEGRATION.md shows the cgo and ctypes stubs).  The shared library is built
in-tree by `make` / `__graft_entry__.build()`; importing this module without it
fails loudly — there is no CPU fallback behind this API.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CAGRA_LIB") or os.path.join(_HERE, "lib", "libcagra_b200.so")

OK, ERR_USAGE, ERR_FORMAT, ERR_CUDA, ERR_NCCL, ERR_LOGIC = 0, 2, 3, 4, 5, 6
HASH_STANDARD, HASH_FORGETTABLE = 0, 1
MODE_PER_QUERY, MODE_SHARED = 0, 1
INVALID_ID = 0xFFFFFFFF


class CagraError(RuntimeError):
    code = -1


class UsageError(CagraError, ValueError):
    """fodg::UsageError (common.hpp:13-15)."""
    code = ERR_USAGE


class FormatError(CagraError):
    """fodg::FormatError (common.hpp:18-20)."""
    code = ERR_FORMAT


class CudaError(CagraError):
    code = ERR_CUDA


class LogicError(CagraError):
    """std::logic_error (search.cpp:180)."""
    code = ERR_LOGIC


_ERRORS = {ERR_USAGE: UsageError, ERR_FORMAT: FormatError, ERR_CUDA: CudaError,
           ERR_LOGIC: LogicError, ERR_NCCL: CagraError}


class SearchParamsC(C.Structure):
    _fields_ = [("k", C.c_uint32), ("topm", C.c_uint32), ("width", C.c_uint32),
                ("max_iterations", C.c_uint32), ("min_iterations", C.c_uint32),
                ("hash_policy", C.c_uint32), ("hash_bits", C.c_uint32),
                ("reset_interval", C.c_uint32), ("seed", C.c_uint64)]


class EngineOptsC(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("team_count", C.c_uint32), ("num_threads", C.c_uint32),
                ("seed_mode", C.c_uint32), ("query_offset", C.c_uint64),
                ("exact_distances", C.c_uint32), ("team_size", C.c_uint32),
                ("multi_cta", C.c_uint32), ("_pad", C.c_uint32)]


class SearchStatsC(C.Structure):
    _fields_ = [("iterations", C.c_uint32), ("hash_resets", C.c_uint32),
                ("distance_evals", C.c_uint64), ("converged", C.c_uint32), ("_pad", C.c_uint32)]


STATS_DTYPE = np.dtype([("iterations", np.uint32), ("hash_resets", np.uint32),
                        ("distance_evals", np.uint64), ("converged", np.uint32),
                        ("_pad", np.uint32)])


class OptStatsC(C.Structure):
    _fields_ = [("count_seconds", C.c_double), ("reorder_seconds", C.c_double),
                ("reverse_seconds", C.c_double), ("merge_seconds", C.c_double),
                ("total_seconds", C.c_double)]


# Every symbol include/cagra/capi.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "cagra_last_error", "cagra_version", "cagra_device_count", "cagra_search_params_default",
    "cagra_engine_opts_default", "cagra_uniform_dataset", "cagra_mix_seed",
    "cagra_exact_knn_graph", "cagra_exact_topk", "cagra_knn_last_stats",
    "cagra_count_detourable_routes", "cagra_count_detourable_routes_distance",
    "cagra_reorder_and_prune", "cagra_build_reverse_graph", "cagra_merge_graphs",
    "cagra_optimize", "cagra_build_graph", "cagra_index_create", "cagra_index_create_dev",
    "cagra_index_destroy", "cagra_index_info", "cagra_index_row_stride", "cagra_search",
    "cagra_search_dev", "cagra_last_launch_count", "cagra_merge_shard_topk_dev",
    "cagra_graph_metrics", "cagra_trim_scratch", "cagra_knn_last_filter",
    "cagra_exact_knn_rows", "cagra_build_graph_multi", "cagra_mindex_create",
    "cagra_mindex_destroy", "cagra_mindex_info", "cagra_msearch", "cagra_exact_knn_graph_multi",
    "cagra_nn_descent",
]

_lib = None


def lib() -> C.CDLL:
    """Load libcagra_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: build the CUDA engine first (make, or "
                "__graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        L.cagra_last_error.restype = C.c_char_p
        L.cagra_version.restype = C.c_char_p
        L.cagra_mix_seed.restype = u64
        L.cagra_mix_seed.argtypes = [u64]
        L.cagra_uniform_dataset.argtypes = [u64, u64, vp]
        L.cagra_exact_knn_graph.argtypes = [vp, u32, u32, u32, i32, vp, vp]
        L.cagra_exact_topk.argtypes = [vp, u32, u32, vp, u32, u32, i32, vp, vp]
        L.cagra_knn_last_stats.argtypes = [vp, vp, vp, vp]
        L.cagra_count_detourable_routes.argtypes = [vp, vp, u32, u32, i32, vp]
        L.cagra_graph_metrics.argtypes = [vp, u32, u32, i32, vp, vp]
        L.cagra_count_detourable_routes_distance.argtypes = [vp, vp, u32, u32, vp, u32, u32, i32,
                                                             vp]
        L.cagra_reorder_and_prune.argtypes = [vp, vp, u32, u32, u32, i32, vp]
        L.cagra_build_reverse_graph.argtypes = [vp, u32, u32, u32, i32, vp, vp]
        L.cagra_merge_graphs.argtypes = [vp, vp, vp, u32, u32, u32, i32, vp]
        L.cagra_optimize.argtypes = [vp, vp, u32, u32, u32, u32, u32, i32, vp, vp]
        L.cagra_build_graph.argtypes = [vp, u32, u32, u32, u32, i32, vp, vp, vp, vp]
        L.cagra_index_create.argtypes = [vp, u32, u32, vp, u32, i32, C.POINTER(vp)]
        L.cagra_index_create_dev.argtypes = [vp, u32, u32, vp, u32, i32, C.POINTER(vp)]
        L.cagra_index_destroy.argtypes = [vp]
        L.cagra_index_info.argtypes = [vp, vp, vp, vp, vp]
        L.cagra_index_row_stride.restype = u32
        L.cagra_index_row_stride.argtypes = [vp]
        L.cagra_search.argtypes = [vp, vp, u32, u32, vp, vp, vp, vp, vp, vp]
        L.cagra_search_dev.argtypes = [vp, vp, u32, vp, vp, vp, vp, vp, vp, vp]
        L.cagra_last_launch_count.restype = u32
        L.cagra_last_launch_count.argtypes = [vp]
        L.cagra_merge_shard_topk_dev.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, i32, vp]
        L.cagra_exact_knn_rows.argtypes = [vp, u32, u32, u32, u32, u32, i32, vp, vp]
        L.cagra_build_graph_multi.argtypes = [vp, u32, u32, u32, u32, vp, u32, vp, vp, vp, vp]
        L.cagra_mindex_create.argtypes = [vp, u32, u32, vp, u32, vp, u32, u32, C.POINTER(vp)]
        L.cagra_mindex_destroy.argtypes = [vp]
        L.cagra_mindex_info.argtypes = [vp, vp, vp, vp, vp, vp]
        L.cagra_msearch.argtypes = [vp, vp, u32, u32, vp, vp, vp, vp, vp, vp]
        L.cagra_exact_knn_graph_multi.argtypes = [vp, u32, u32, u32, vp, u32, vp, vp]
        L.cagra_nn_descent.argtypes = [vp, u32, u32, u32, C.c_double, C.c_double, u32, u64, i32,
                                       vp, vp, vp, vp]
        L.cagra_trim_scratch.argtypes = [i32]
        L.cagra_knn_last_filter.argtypes = [vp, vp]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().cagra_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, CagraError)(msg)


def ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    if isinstance(a, int):
        return C.c_void_p(a)
    return C.c_void_p(a.data_ptr())  # torch tensor (device pointers for *_dev)


def device_count() -> int:
    c = C.c_int(0)
    lib().cagra_device_count(C.byref(c))
    return c.value


def knn_last_stats() -> dict:
    """Counters of the last tensor-core kNN / top-k call (rows, fallback_rows,
    reranked); all zero when the SIMT path ran."""
    v = (C.c_uint64 * 4)()
    lib().cagra_knn_last_stats(C.byref(v, 0), C.byref(v, 8), C.byref(v, 16), C.byref(v, 24))
    f = (C.c_uint32 * 2)()
    lib().cagra_knn_last_filter(C.byref(f, 0), C.byref(f, 4))
    return {"rows": v[0], "fallback_rows": v[1], "reranked": v[2], "retried_rows": v[3],
            "split_terms": f[0], "gemm_k": f[1]}


def graph_metrics(graph: np.ndarray, device: int = 0):
    """(strong-CC count, distinct <=2-hop total) of an n x d uint32 graph,
    computed on the device (cagra_graph_metrics)."""
    g = np.ascontiguousarray(graph, np.uint32)
    n, d = g.shape
    scc = C.c_uint64(0)
    tot = C.c_uint64(0)
    check(lib().cagra_graph_metrics(ptr(g), n, d, device, C.byref(scc), C.byref(tot)))
    return int(scc.value), int(tot.value)


def mix_seed(x: int) -> int:
    return int(lib().cagra_mix_seed(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def uniform_dataset(n: int, dim: int, seed: int) -> np.ndarray:
    out = np.empty((n, dim), np.float32)
    check(lib().cagra_uniform_dataset(C.c_uint64(seed), C.c_uint64(n * dim), ptr(out)))
    return out
