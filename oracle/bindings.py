"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings for
  * oracle/liboracle.so        — the plain-C restatement (fodg_oracle.c), and
  * oracle/_ref/libfodg_ref.so — the unmodified reference compiled from
                                 /root/reference (ref_capi.cpp wrapper).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline.  The product package (paper_2308_15136_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfodg_ref.so")

INVALID = 0xFFFFFFFF


class Params(C.Structure):
    """SearchParams mirror (search.hpp:14-27)."""

    _fields_ = [("k", C.c_uint32), ("topm", C.c_uint32), ("width", C.c_uint32),
                ("max_iterations", C.c_uint32), ("min_iterations", C.c_uint32),
                ("hash_policy", C.c_uint32), ("hash_bits", C.c_uint32),
                ("reset_interval", C.c_uint32), ("seed", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_uint32), ("hash_resets", C.c_uint32),
                ("distance_evals", C.c_uint64), ("converged", C.c_uint32),
                ("_pad", C.c_uint32)]


def make_params(k=10, topm=64, width=1, max_iterations=0, min_iterations=1, hash_policy=0,
                hash_bits=11, reset_interval=1, seed=0) -> Params:
    return Params(k, topm, width, max_iterations, min_iterations, hash_policy, hash_bits,
                  reset_interval, seed)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle returned {code}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc)


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        self.lib[self.prefix + "mix_seed"].restype = C.c_uint64
        self.lib[self.prefix + "mix_seed"].argtypes = [C.c_uint64]

    def fn(self, name):
        return self.lib[self.prefix + name]

    def mix_seed(self, x):
        return int(self.fn("mix_seed")(C.c_uint64(x)))

    # ---- build -------------------------------------------------------------
    def exact_knn_graph(self, data, k, threads=0):
        n, dim = data.shape
        ids = np.empty((n, k), np.uint32)
        dists = np.empty((n, k), np.float32)
        _check(self.fn("exact_knn_graph")(_p(data), C.c_uint32(n), C.c_uint32(dim),
                                          C.c_uint32(k), _p(ids), _p(dists), C.c_int(threads)))
        return ids, dists

    def exact_topk_batch(self, data, queries, k, threads=0):
        n, dim = data.shape
        nq = queries.shape[0]
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        _check(self.fn("exact_topk_batch")(_p(data), C.c_uint32(n), C.c_uint32(dim),
                                           _p(queries), C.c_uint32(nq), C.c_uint32(k),
                                           _p(ids), _p(dists), C.c_int(threads)))
        return ids, dists

    def count_detourable_routes(self, ids, dists):
        n, deg = ids.shape
        counts = np.empty((n, deg), np.uint32)
        _check(self.fn("count_detourable_routes")(_p(ids), _p(dists), C.c_uint32(n),
                                                  C.c_uint32(deg), _p(counts)))
        return counts

    def build_reverse_graph(self, pruned, cap):
        n, d = pruned.shape
        rc = np.empty(n, np.uint32)
        ri = np.full((n, cap), INVALID, np.uint32)
        _check(self.fn("build_reverse_graph")(_p(pruned), C.c_uint32(n), C.c_uint32(d),
                                              C.c_uint32(cap), _p(rc), _p(ri)))
        return rc, ri


class Oracle(_Lib):
    """The C restatement (kind "port")."""

    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        self.lib.orc_uniform_dataset.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        self.lib.orc_squared_l2.restype = C.c_float
        self.lib.orc_squared_l2.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32]

    def uniform_dataset(self, n, dim, seed):
        out = np.empty((n, dim), np.float32)
        self.lib.orc_uniform_dataset(C.c_uint64(seed), C.c_uint64(n * dim), _p(out))
        return out

    def squared_l2(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return float(self.lib.orc_squared_l2(_p(a), _p(b), C.c_uint32(a.size)))

    def reorder_and_prune(self, ids, counts, d):
        n, deg = ids.shape
        out = np.empty((n, d), np.uint32)
        _check(self.lib.orc_reorder_and_prune(_p(ids), _p(counts), C.c_uint32(n),
                                              C.c_uint32(deg), C.c_uint32(d), _p(out)))
        return out

    def merge_graphs(self, pruned, rev_counts, rev_ids):
        n, d = pruned.shape
        out = np.empty((n, d), np.uint32)
        _check(self.lib.orc_merge_graphs(_p(pruned), _p(rev_counts), _p(rev_ids), C.c_uint32(n),
                                         C.c_uint32(d), C.c_uint32(rev_ids.shape[1]), _p(out)))
        return out

    def optimize(self, ids, dists, d):
        n, deg = ids.shape
        out = np.empty((n, d), np.uint32)
        _check(self.lib.orc_optimize(_p(ids), _p(dists), C.c_uint32(n), C.c_uint32(deg),
                                     C.c_uint32(d), _p(out)))
        return out

    def search_one(self, graph, data, query, params):
        n, deg = graph.shape
        dim = data.shape[1]
        ids = np.empty(params.k, np.uint32)
        dists = np.empty(params.k, np.float32)
        cnt = C.c_uint32()
        st = Stats()
        q = np.ascontiguousarray(query, np.float32)
        _check(self.lib.orc_search_one(_p(graph), C.c_uint32(n), C.c_uint32(deg), _p(data),
                                       C.c_uint32(dim), _p(q), C.byref(params), _p(ids),
                                       _p(dists), C.byref(cnt), C.byref(st)))
        return ids[:cnt.value].copy(), dists[:cnt.value].copy(), st

    def batch_search(self, graph, data, queries, params, mode=0, team_count=4,
                     query_offset=0, threads=0):
        n, deg = graph.shape
        dim = data.shape[1]
        nq = queries.shape[0]
        ids = np.empty((nq, params.k), np.uint32)
        dists = np.empty((nq, params.k), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = (Stats * max(nq, 1))()
        _check(self.lib.orc_batch_search(
            _p(graph), C.c_uint32(n), C.c_uint32(deg), _p(data), C.c_uint32(dim), _p(queries),
            C.c_uint32(nq), C.byref(params), C.c_uint32(mode), C.c_uint32(team_count),
            C.c_uint64(query_offset), _p(ids), _p(dists), _p(counts), stats, C.c_int(threads)))
        return ids, dists, counts, stats_to_numpy(stats, nq)


def stats_to_numpy(stats, nq):
    arr = np.ctypeslib.as_array(stats)[:nq] if nq else np.zeros(0)
    return {
        "iterations": np.array([s.iterations for s in stats[:nq]], np.uint32),
        "hash_resets": np.array([s.hash_resets for s in stats[:nq]], np.uint32),
        "distance_evals": np.array([s.distance_evals for s in stats[:nq]], np.uint64),
        "converged": np.array([s.converged for s in stats[:nq]], np.uint32),
    } if nq else arr


class Reference(_Lib):
    """The unmodified reference library (kind "reference")."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self.lib.ref_index_create.restype = C.c_void_p
        self.lib.ref_index_create.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                              C.c_uint32]
        self.lib.ref_index_destroy.argtypes = [C.c_void_p]
        self.lib.ref_hardware_threads.restype = C.c_uint

    def hardware_threads(self):
        return int(self.lib.ref_hardware_threads())

    def optimize(self, ids, dists, d, reorder=True, add_reverse=True):
        n, deg = ids.shape
        out = np.empty((n, d), np.uint32)
        secs = np.zeros(5, np.float64)
        _check(self.lib.ref_optimize(_p(ids), _p(dists), C.c_uint32(n), C.c_uint32(deg),
                                     C.c_uint32(d), C.c_uint32(int(reorder)),
                                     C.c_uint32(int(add_reverse)), _p(out), _p(secs)))
        return out, secs

    def graph_metrics(self, graph):
        """(strong_cc_count, avg_2hop_count) of an n x d uint32 graph."""
        n, d = graph.shape
        scc = C.c_uint64(0)
        avg = C.c_double(0)
        _check(self.lib.ref_graph_metrics(_p(graph), C.c_uint32(n), C.c_uint32(d),
                                          C.byref(scc), C.byref(avg)))
        return int(scc.value), float(avg.value)

    def index(self, data, graph):
        return RefIndex(self, data, graph)


class RefIndex:
    def __init__(self, ref, data, graph):
        self.ref = ref
        self.data = np.ascontiguousarray(data, np.float32)
        self.graph = np.ascontiguousarray(graph, np.uint32)
        n, dim = self.data.shape
        self.dim = dim
        self.h = ref.lib.ref_index_create(_p(self.data), n, dim, _p(self.graph),
                                          self.graph.shape[1])

    def close(self):
        if self.h:
            self.ref.lib.ref_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def batch_search(self, queries, params, mode=0, team_count=4, threads=0):
        queries = np.ascontiguousarray(queries, np.float32)
        nq = queries.shape[0]
        ids = np.empty((nq, params.k), np.uint32)
        dists = np.empty((nq, params.k), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = (Stats * max(nq, 1))()
        _check(self.ref.lib.ref_index_batch_search(
            C.c_void_p(self.h), _p(queries), C.c_uint32(nq), C.c_uint32(self.dim),
            C.byref(params), C.c_uint32(mode), C.c_uint32(team_count), C.c_uint32(threads),
            _p(ids), _p(dists), _p(counts), stats))
        return ids, dists, counts, stats_to_numpy(stats, nq)

    def search_one(self, query, params):
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(params.k, np.uint32)
        dists = np.empty(params.k, np.float32)
        cnt = C.c_uint32()
        st = Stats()
        _check(self.ref.lib.ref_index_search_one(C.c_void_p(self.h), _p(q), C.byref(params),
                                                 _p(ids), _p(dists), C.byref(cnt), C.byref(st)))
        return ids[:cnt.value].copy(), dists[:cnt.value].copy(), st

    def run_benchmark(self, queries, truth, params, mode=0, team_count=4, threads=0):
        queries = np.ascontiguousarray(queries, np.float32)
        truth = np.ascontiguousarray(truth, np.uint32)
        rec = C.c_double()
        qps = C.c_double()
        it = C.c_double()
        _check(self.ref.lib.ref_index_run_benchmark(
            C.c_void_p(self.h), _p(queries), C.c_uint32(queries.shape[0]), C.c_uint32(self.dim),
            _p(truth), C.c_uint32(truth.shape[1]), C.byref(params), C.c_uint32(mode),
            C.c_uint32(team_count), C.c_uint32(threads), C.byref(rec), C.byref(qps),
            C.byref(it)))
        return rec.value, qps.value, it.value


def load_oracle():
    return Oracle()


def load_reference():
    """The reference library, or None when oracle/_ref was not built."""
    if not os.path.exists(REF_SO):
        return None
    return Reference()
