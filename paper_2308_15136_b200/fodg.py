"""Python mirror of the reference's public `fodg::` API (proj/core/include/fodg).

Same names, argument meaning and error classes as the reference, so parity
tests read like the reference's own tests.  Compute goes through the C ABI to
the sm_100a kernels (capi.py); the only host code here is validation, container
types and the cheap bookkeeping the reference also does on the host
(recall, sorting a KnnGraph, CSV formatting).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import capi
from .capi import CudaError, FormatError, LogicError, UsageError, check, lib, ptr

kIdMask = 0x7FFFFFFF
kParentFlag = 0x80000000
kInvalidId = 0xFFFFFFFF
kMaxNodes = kIdMask

__all__ = [
    "UsageError", "FormatError", "LogicError", "CudaError", "HashPolicy", "ExecutionMode",
    "ReorderMode", "SearchParams", "EngineOptions", "ModeThresholds", "OptimizeOptions",
    "OptimizeStats", "Dataset", "Graph", "KnnGraph", "ReverseGraph", "NeighborList",
    "SearchStats", "SearchResult", "squared_l2", "mix_seed", "exact_topk", "recall",
    "exact_knn_graph", "sort_neighbor_lists", "knn_graph_recall", "count_detourable_routes",
    "reorder_and_prune", "truncate_graph", "build_reverse_graph", "merge_graphs", "optimize",
    "build_graph", "Index", "search_one", "batch_search", "choose_mode", "mode_name",
    "BenchRecord", "bench_csv_header", "bench_csv_row", "run_benchmark", "make_uniform_dataset",
]


class HashPolicy(IntEnum):
    kStandard = 0
    kForgettable = 1


class ExecutionMode(IntEnum):
    kPerQueryWorker = 0
    kSharedQueryWorkers = 1


class ReorderMode(IntEnum):
    kRank = 0
    kDistance = 1


mix_seed = capi.mix_seed


# ------------------------------------------------------------------ params --
@dataclass
class SearchParams:
    """search.hpp:14-27."""
    k: int = 10
    topm: int = 64
    width: int = 1
    max_iterations: int = 0
    min_iterations: int = 1
    hash_policy: HashPolicy = HashPolicy.kStandard
    hash_bits: int = 11
    reset_interval: int = 1
    seed: int = 0

    def resolved_max_iterations(self) -> int:  # search.cpp:33-37
        if self.max_iterations:
            return self.max_iterations
        it = (2 * self.topm + self.width - 1) // self.width
        return min(max(it, 16), 256)

    def validate(self) -> None:  # search.cpp:39-50
        if self.k == 0:
            raise UsageError("search: k must be >= 1")
        if self.k > self.topm:
            raise UsageError("search: require k <= M")
        if self.width == 0:
            raise UsageError("search: p must be >= 1")
        if self.min_iterations > self.resolved_max_iterations():
            raise UsageError("search: min_iterations exceeds max_iterations")
        if self.hash_policy == HashPolicy.kForgettable:
            if not 4 <= self.hash_bits <= 24:
                raise UsageError("search: forgettable hash_bits out of range")
            if self.reset_interval == 0:
                raise UsageError("search: reset_interval must be >= 1")

    def c(self) -> capi.SearchParamsC:
        return capi.SearchParamsC(self.k, self.topm, self.width, self.max_iterations,
                                  self.min_iterations, int(self.hash_policy), self.hash_bits,
                                  self.reset_interval, self.seed & 0xFFFFFFFFFFFFFFFF)


@dataclass
class ModeThresholds:
    """engine.hpp:18-21; batch_threshold 0 = the device's parallel workers (SMs)."""
    batch_threshold: int = 0
    topm_threshold: int = 512


@dataclass
class EngineOptions:
    """engine.hpp:27-31 plus device knobs."""
    mode: ExecutionMode = ExecutionMode.kPerQueryWorker
    team_count: int = 4
    num_threads: int = 0
    device: int = 0
    exact_distances: bool = False
    team_size: int = 0
    multi_cta: int = 0  # shared mode: 0 auto, 1 lockstep single CTA, 2 one CTA per team

    def c(self, seed_mode=0, query_offset=0) -> capi.EngineOptsC:
        return capi.EngineOptsC(int(self.mode), self.team_count, self.num_threads, seed_mode,
                                query_offset, int(bool(self.exact_distances)), self.team_size,
                                self.multi_cta, 0)


@dataclass
class OptimizeOptions:
    """graph_opt.hpp:25-30."""
    mode: ReorderMode = ReorderMode.kRank
    reorder: bool = True
    add_reverse: bool = True
    num_threads: int = 0
    device: int = 0


@dataclass
class OptimizeStats:
    """graph_opt.hpp:33-41 (device-event timed)."""
    count_seconds: float = 0.0
    reorder_seconds: float = 0.0
    reverse_seconds: float = 0.0
    merge_seconds: float = 0.0
    total_seconds: float = 0.0

    def report(self) -> str:  # graph_opt.cpp:35-43
        return (f"stage_detour_count_seconds={self.count_seconds}\n"
                f"stage_reorder_seconds={self.reorder_seconds}\n"
                f"stage_reverse_seconds={self.reverse_seconds}\n"
                f"stage_merge_seconds={self.merge_seconds}\n"
                f"optimize_total_seconds={self.total_seconds}\n")


# -------------------------------------------------------------- containers --
class Dataset:
    """dataset.hpp:12-29 / dataset.cpp:7-18: N x dim fp32, row-major."""

    def __init__(self, dim: int, data):
        if dim == 0:
            raise UsageError("dataset dimension must be >= 1")
        arr = np.ascontiguousarray(np.asarray(data, dtype=np.float32).reshape(-1))
        if arr.size == 0 or arr.size % dim != 0:
            raise UsageError("dataset size is not a multiple of the dimension")
        rows = arr.size // dim
        if rows > kMaxNodes:
            raise UsageError("dataset exceeds 2^31 - 1 vectors (index MSB is reserved)")
        if not np.isfinite(arr).all():
            raise UsageError("dataset contains non-finite components")
        self.data = arr.reshape(rows, dim)

    @classmethod
    def from_array(cls, a) -> "Dataset":
        a = np.asarray(a, np.float32)
        return cls(a.shape[1], a)

    def size(self) -> int:
        return self.data.shape[0]

    def dim(self) -> int:
        return self.data.shape[1]

    def row(self, i: int) -> np.ndarray:
        return self.data[i]

    def raw(self) -> np.ndarray:
        return self.data


def make_uniform_dataset(n_rows: int, dim: int, seed: int) -> Dataset:
    """tests/test_util.hpp:11-18 (the reference fixture generator)."""
    return Dataset(dim, capi.uniform_dataset(n_rows, dim, seed))


@dataclass
class Graph:
    """graph.hpp:14-25: N rows of exactly `degree` ids."""
    num_nodes: int = 0
    degree: int = 0
    ids: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint32))

    def row(self, i: int) -> np.ndarray:
        return self.ids[i]


@dataclass
class KnnGraph:
    """knn_build.hpp:14-28."""
    num_nodes: int = 0
    degree: int = 0
    ids: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint32))
    dists: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.float32))
    converged: bool = True
    graph_recall: float = -1.0

    def row_ids(self, i):
        return self.ids[i]

    def row_dists(self, i):
        return self.dists[i]


@dataclass
class ReverseGraph:
    """graph_opt.hpp:20-23."""
    num_nodes: int = 0
    rows: List[List[int]] = field(default_factory=list)


@dataclass
class NeighborList:
    ids: np.ndarray
    dists: np.ndarray


@dataclass
class SearchStats:
    iterations: int = 0
    distance_evals: int = 0
    hash_resets: int = 0
    converged: bool = False


@dataclass
class SearchResult:
    ids: np.ndarray
    dists: np.ndarray
    stats: SearchStats


# ----------------------------------------------------------------- helpers --
def squared_l2(a, b) -> np.float32:
    """dataset.hpp:33-43 on the host: sequential fp32 chain (add.accumulate is
    strictly sequential, each product rounded separately)."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    diff = (a - b).astype(np.float32)
    sq = (diff * diff).astype(np.float32)
    if sq.size == 0:
        return np.float32(0.0)
    return np.add.accumulate(sq, dtype=np.float32)[-1]


def _as_rows(x, dim=None) -> np.ndarray:
    if isinstance(x, Dataset):
        return x.data
    a = np.ascontiguousarray(np.asarray(x, np.float32))
    if a.ndim == 1:
        a = a.reshape(1, -1)
    return a


# ---------------------------------------------------------- kNN / ground truth
def exact_topk(ds: Dataset, q, k: int, device: int = 0) -> NeighborList:
    """topk.hpp:20 (single query; batch form: exact_topk_batch)."""
    q = np.asarray(q, np.float32).reshape(-1)
    if q.size != ds.dim():
        raise UsageError("exact_topk: query dimension mismatch")
    ids, dists = exact_topk_batch(ds, q.reshape(1, -1), k, device)
    return NeighborList(ids[0], dists[0])


def exact_topk_batch(ds: Dataset, queries, k: int, device: int = 0):
    data = ds.data
    qs = _as_rows(queries)
    if qs.shape[1] != ds.dim():
        raise UsageError("exact_topk: query dimension mismatch")
    nq = qs.shape[0]
    ids = np.empty((nq, k), np.uint32)
    dists = np.empty((nq, k), np.float32)
    check(lib().cagra_exact_topk(ptr(data), data.shape[0], data.shape[1], ptr(qs), nq, k,
                                 device, ptr(ids), ptr(dists)))
    return ids, dists


def recall(result_ids: Sequence[int], truth_ids: Sequence[int]) -> float:
    """topk.cpp:45-59."""
    truth = list(truth_ids)
    res = list(result_ids)
    if not truth:
        raise UsageError("recall: empty ground truth")
    if len(res) != len(truth):
        raise UsageError("recall: result and truth lengths differ")
    ts = set(truth)
    if len(ts) != len(truth):
        raise UsageError("recall: duplicate ids in truth")
    seen = set()
    hits = 0
    for i in res:
        if i in seen:
            raise UsageError("recall: duplicate ids in result")
        seen.add(i)
        hits += i in ts
    return hits / len(truth)


def exact_knn_graph(ds: Dataset, k: int, num_threads: int = 0, device: int = 0) -> KnnGraph:
    """knn_build.hpp:40 / knn_build.cpp:40-63."""
    n, dim = ds.data.shape
    if k == 0 or k >= n:
        raise UsageError("exact_knn_graph: require 1 <= k < N")
    ids = np.empty((n, k), np.uint32)
    dists = np.empty((n, k), np.float32)
    check(lib().cagra_exact_knn_graph(ptr(ds.data), n, dim, k, device, ptr(ids), ptr(dists)))
    return KnnGraph(n, k, ids, dists)


@dataclass
class NNDescentParams:
    """knn_build.hpp:33-39."""
    sample_rate: float = 0.5
    termination_delta: float = 0.001
    max_rounds: int = 20
    seed: int = 0
    num_threads: int = 0


def nn_descent(ds: Dataset, k: int, params: Optional[NNDescentParams] = None,
               device: int = 0) -> KnnGraph:
    """knn_build.hpp:42 / knn_build.cpp:96-231, on the device (cagra_nn_descent)."""
    params = params or NNDescentParams()
    n, dim = ds.data.shape
    ids = np.empty((n, k), np.uint32) if 0 < k < n else np.empty((0, 0), np.uint32)
    dists = np.empty(ids.shape, np.float32)
    conv = C.c_uint32(0)
    rounds = C.c_uint32(0)
    check(lib().cagra_nn_descent(ptr(ds.data), n, dim, k, float(params.sample_rate),
                                 float(params.termination_delta), int(params.max_rounds),
                                 int(params.seed) & 0xFFFFFFFFFFFFFFFF, device, ptr(ids),
                                 ptr(dists), C.byref(conv), C.byref(rounds)))
    g = KnnGraph(n, k, ids, dists)
    g.converged = bool(conv.value)
    g.rounds = int(rounds.value)
    return g


def sort_neighbor_lists(g: KnnGraph) -> None:
    """knn_build.cpp:65-79 (host bookkeeping)."""
    if g.dists.shape != g.ids.shape:
        raise UsageError("sort_neighbor_lists: rows have no distances")
    order = np.lexsort((g.ids, g.dists), axis=1) if g.ids.size else None
    if order is not None:
        g.ids = np.take_along_axis(g.ids, order, 1)
        g.dists = np.take_along_axis(g.dists, order, 1)


def knn_graph_recall(g: KnnGraph, exact: KnnGraph) -> float:
    """knn_build.cpp:81-94."""
    if g.num_nodes != exact.num_nodes or g.degree != exact.degree:
        raise UsageError("knn_graph_recall: shape mismatch")
    s = 0.0
    for v in range(g.num_nodes):
        s += len(set(g.ids[v].tolist()) & set(exact.ids[v].tolist())) / g.degree
    return s / g.num_nodes


# ------------------------------------------------------------- optimization --
def _rank_only(mode):
    if mode != ReorderMode.kRank:
        raise UsageError("graph_opt: only rank mode runs on device (distance mode is the "
                         "paper's comparison-only variant, out of scope)")


def count_detourable_routes(g: KnnGraph, mode: ReorderMode = ReorderMode.kRank,
                            ds: Optional[Dataset] = None, num_threads: int = 0,
                            device: int = 0) -> np.ndarray:
    """graph_opt.hpp:47-49, rank mode."""
    _rank_only(mode)
    if g.dists.shape != g.ids.shape:
        raise UsageError("graph_opt: input rows have no distances")
    ids = np.ascontiguousarray(g.ids, np.uint32)
    dists = np.ascontiguousarray(g.dists, np.float32)
    counts = np.empty(ids.shape, np.uint32)
    check(lib().cagra_count_detourable_routes(ptr(ids), ptr(dists), g.num_nodes, g.degree,
                                              device, ptr(counts)))
    return counts


def reorder_and_prune(g: KnnGraph, counts, d: int, num_threads: int = 0,
                      device: int = 0) -> Graph:
    """graph_opt.hpp:53-54."""
    if d == 0 or d > g.degree:
        raise UsageError("reorder_and_prune: require 1 <= d <= input degree")
    counts = np.ascontiguousarray(np.asarray(counts, np.uint32).reshape(g.ids.shape))
    ids = np.ascontiguousarray(g.ids, np.uint32)
    out = np.empty((g.num_nodes, d), np.uint32)
    check(lib().cagra_reorder_and_prune(ptr(ids), ptr(counts), g.num_nodes, g.degree, d,
                                        device, ptr(out)))
    return Graph(g.num_nodes, d, out)


def truncate_graph(g: KnnGraph, d: int) -> Graph:
    """graph_opt.cpp:126-139 (ablation only)."""
    if d == 0 or d > g.degree:
        raise UsageError("truncate_graph: require 1 <= d <= input degree")
    return Graph(g.num_nodes, d, np.ascontiguousarray(g.ids[:, :d]))


def _reverse_arrays(pruned: Graph, cap: int, device: int = 0):
    ids = np.ascontiguousarray(pruned.ids, np.uint32)
    rc = np.empty(pruned.num_nodes, np.uint32)
    ri = np.empty((pruned.num_nodes, max(min(cap, pruned.num_nodes), 1)), np.uint32)
    check(lib().cagra_build_reverse_graph(ptr(ids), pruned.num_nodes, pruned.degree, cap,
                                          device, ptr(rc), ptr(ri)))
    return rc, ri


def build_reverse_graph(pruned: Graph, cap: int, device: int = 0) -> ReverseGraph:
    """graph_opt.hpp:59."""
    rc, ri = _reverse_arrays(pruned, cap, device)
    return ReverseGraph(pruned.num_nodes, [ri[y, :rc[y]].tolist() for y in range(len(rc))])


def merge_graphs(pruned: Graph, rev: ReverseGraph, d: int, device: int = 0) -> Graph:
    """graph_opt.hpp:63."""
    if pruned.degree != d:
        raise UsageError("merge_graphs: pruned degree must equal d")
    if rev.num_nodes != pruned.num_nodes:
        raise UsageError("merge_graphs: size mismatch")
    cap = max([len(r) for r in rev.rows] + [1])
    rc = np.array([len(r) for r in rev.rows], np.uint32)
    ri = np.full((pruned.num_nodes, cap), kInvalidId, np.uint32)
    for y, r in enumerate(rev.rows):
        ri[y, :len(r)] = r
    out = np.empty((pruned.num_nodes, d), np.uint32)
    ids = np.ascontiguousarray(pruned.ids, np.uint32)
    check(lib().cagra_merge_graphs(ptr(ids), ptr(rc), ptr(ri), pruned.num_nodes, d, cap, device,
                                   ptr(out)))
    return Graph(pruned.num_nodes, d, out)


def optimize(g: KnnGraph, d: int, opts: Optional[OptimizeOptions] = None,
             ds: Optional[Dataset] = None, stats: Optional[OptimizeStats] = None) -> Graph:
    """graph_opt.hpp:67-68: count -> reorder+prune -> reverse -> merge, on device."""
    opts = opts or OptimizeOptions()
    if d == 0 or d > g.degree:
        raise UsageError("optimize: require 1 <= d <= input degree")
    if opts.reorder:
        _rank_only(opts.mode)
    if g.dists.shape != g.ids.shape:
        raise UsageError("graph_opt: input rows have no distances")
    ids = np.ascontiguousarray(g.ids, np.uint32)
    dists = np.ascontiguousarray(g.dists, np.float32)
    out = np.empty((g.num_nodes, d), np.uint32)
    st = capi.OptStatsC()
    check(lib().cagra_optimize(ptr(ids), ptr(dists), g.num_nodes, g.degree, d,
                               int(opts.reorder), int(opts.add_reverse), opts.device, ptr(out),
                               C.byref(st)))
    if stats is not None:
        stats.count_seconds = st.count_seconds
        stats.reorder_seconds = st.reorder_seconds
        stats.reverse_seconds = st.reverse_seconds
        stats.merge_seconds = st.merge_seconds
        stats.total_seconds = st.total_seconds
    return Graph(g.num_nodes, d, out)


def build_graph(ds: Dataset, d: int, d_init: Optional[int] = None, device: int = 0,
                return_knn: bool = False):
    """exact_knn_graph(ds, d_init) -> optimize(., d) fully on device
    (tools/main.cpp:72-123 with d_init defaulting to 2d, :74).
    Returns (Graph, seconds dict[, KnnGraph])."""
    d_init = d_init or 2 * d
    n, dim = ds.data.shape
    out = np.empty((n, d), np.uint32)
    kid = np.empty((n, d_init), np.uint32) if return_knn else None
    kd = np.empty((n, d_init), np.float32) if return_knn else None
    secs = np.zeros(2, np.float64)
    check(lib().cagra_build_graph(ptr(ds.data), n, dim, d_init, d, device, ptr(out), ptr(kid),
                                  ptr(kd), ptr(secs)))
    g = Graph(n, d, out)
    info = {"knn_seconds": float(secs[0]), "optimize_seconds": float(secs[1])}
    if return_knn:
        return g, info, KnnGraph(n, d_init, kid, kd)
    return g, info


def exact_knn_rows(ds: Dataset, k: int, row_begin: int, row_end: int,
                   device: int = 0) -> KnnGraph:
    """Rows [row_begin, row_end) of exact_knn_graph(ds, k) (knn_build.cpp:40-63,
    the parallel_for over rows at :49, one range): the unit of a row-sharded
    build.  Returns a KnnGraph of row_end - row_begin rows (global ids)."""
    n, dim = ds.data.shape
    cnt = row_end - row_begin
    ids = np.empty((cnt, k), np.uint32)
    dists = np.empty((cnt, k), np.float32)
    check(lib().cagra_exact_knn_rows(ptr(ds.data), n, dim, k, row_begin, row_end, device,
                                     ptr(ids), ptr(dists)))
    return KnnGraph(cnt, k, ids, dists)


def _devset(devices: Sequence[int]):
    arr = np.ascontiguousarray(np.asarray(list(devices), np.int32))
    if arr.size == 0:
        raise UsageError("device set: empty")
    return arr


def build_graph_multi(ds: Dataset, d: int, devices: Sequence[int], d_init: Optional[int] = None,
                      return_knn: bool = False):
    """build_graph with the exact kNN rows spread over `devices` (row-sharded
    K1, peer copies to devices[0], optimize there) — bit-identical graph."""
    d_init = d_init or 2 * d
    n, dim = ds.data.shape
    dv = _devset(devices)
    out = np.empty((n, d), np.uint32)
    kid = np.empty((n, d_init), np.uint32) if return_knn else None
    kd = np.empty((n, d_init), np.float32) if return_knn else None
    secs = np.zeros(2, np.float64)
    check(lib().cagra_build_graph_multi(ptr(ds.data), n, dim, d_init, d, ptr(dv), dv.size,
                                        ptr(out), ptr(kid), ptr(kd), ptr(secs)))
    g = Graph(n, d, out)
    info = {"knn_seconds": float(secs[0]), "optimize_seconds": float(secs[1])}
    if return_knn:
        return g, info, KnnGraph(n, d_init, kid, kd)
    return g, info


class MultiIndex:
    """A device set in one process (cagra_mindex): `replicate` = a replica
    per device with the batch split over them (same results as one device);
    `dataset` = contiguous id-range shards with their own graphs, every query
    searched on every shard, per-shard top-k merged by K8 on devices[0]."""

    MODES = {"replicate": 0, "dataset": 1}

    def __init__(self, ds, devices: Sequence[int], graph=None, degree: int = 64,
                 shard_mode: str = "replicate"):
        data = ds.data if isinstance(ds, Dataset) else np.ascontiguousarray(ds, np.float32)
        self._data = data
        gids = None
        if graph is not None:
            gids = graph.ids if isinstance(graph, Graph) else np.asarray(graph)
            gids = np.ascontiguousarray(gids.reshape(data.shape[0], -1), np.uint32)
            degree = gids.shape[1]
        self._graph = gids
        dv = _devset(devices)
        h = C.c_void_p()
        check(lib().cagra_mindex_create(ptr(data), data.shape[0], data.shape[1], ptr(gids),
                                        degree, ptr(dv), dv.size, self.MODES[shard_mode],
                                        C.byref(h)))
        self.h = h
        self.dim = data.shape[1]

    def close(self):
        if getattr(self, "h", None):
            lib().cagra_mindex_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, queries, params: SearchParams, options: Optional[EngineOptions] = None,
               query_offset: int = 0):
        """(ids [nq,k], dists [nq,k], counts [nq], stats recarray)."""
        options = options or EngineOptions()
        qs = _as_rows(queries)
        nq, k = qs.shape[0], params.k
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.empty(nq, capi.STATS_DTYPE)
        pc, oc = params.c(), options.c(0, query_offset)
        check(lib().cagra_msearch(self.h, ptr(qs), nq, qs.shape[1] if nq else self.dim,
                                  C.byref(pc), C.byref(oc), ptr(ids), ptr(dists), ptr(counts),
                                  ptr(stats)))
        return ids, dists, counts, stats


# ------------------------------------------------------------------- search --
@dataclass
class GraphQualityReport:
    """graph_metrics.hpp:10-19."""
    num_nodes: int = 0
    degree: int = 0
    strong_cc: int = 0
    avg_2hop: float = 0.0
    max_2hop: int = 0

    def report(self) -> str:
        return (f"num_nodes={self.num_nodes}\ndegree={self.degree}\nstrong_cc={self.strong_cc}\n"
                f"avg_2hop={self.avg_2hop:g}\nmax_2hop={self.max_2hop}\n")


def strong_cc_count(g: Graph, device: int = 0) -> int:
    """graph_metrics.hpp:22 (on the device: trimming + colouring)."""
    return capi.graph_metrics(g.ids.reshape(g.num_nodes, g.degree), device)[0] if g.num_nodes else 0


def avg_2hop_count(g: Graph, num_threads: int = 0, device: int = 0) -> float:
    """graph_metrics.hpp:26: mean distinct <=2-hop neighbours (exact integer total / n)."""
    if g.num_nodes == 0:
        return 0.0
    return capi.graph_metrics(g.ids.reshape(g.num_nodes, g.degree), device)[1] / g.num_nodes


def measure_graph(g: Graph, num_threads: int = 0, device: int = 0) -> GraphQualityReport:
    """graph_metrics.hpp:28."""
    scc, tot = (capi.graph_metrics(g.ids.reshape(g.num_nodes, g.degree), device)
                if g.num_nodes else (0, 0))
    return GraphQualityReport(g.num_nodes, g.degree, scc, tot / g.num_nodes if g.num_nodes else 0.0,
                              g.degree * (1 + g.degree))


class Index:
    """Device-resident (dataset, graph) — replaces the per-call `const Graph&,
    const Dataset&` of batch_search (engine.hpp:38-40)."""

    def __init__(self, ds, graph, device: int = 0):
        data = ds.data if isinstance(ds, Dataset) else np.ascontiguousarray(ds, np.float32)
        gids = graph.ids if isinstance(graph, Graph) else np.asarray(graph)
        gids = np.ascontiguousarray(gids, np.uint32)
        if gids.shape[0] != data.shape[0]:
            raise UsageError("search: graph/dataset size mismatch")
        self.n, self.dim = data.shape
        self.degree = gids.shape[1]
        h = C.c_void_p()
        check(lib().cagra_index_create(ptr(data), self.n, self.dim, ptr(gids), self.degree,
                                       device, C.byref(h)))
        self.h = h
        self.device = device
        self.ld = int(lib().cagra_index_row_stride(h))

    def close(self):
        if getattr(self, "h", None):
            lib().cagra_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, queries, params: SearchParams, options: Optional[EngineOptions] = None,
               seed_mode: int = 0, query_offset: int = 0):
        """Array form: (ids [nq,k], dists [nq,k], counts [nq], stats recarray)."""
        options = options or EngineOptions()
        qs = _as_rows(queries)
        nq = qs.shape[0]
        k = params.k
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.empty(nq, capi.STATS_DTYPE)
        pc = params.c()
        oc = options.c(seed_mode, query_offset)
        check(lib().cagra_search(self.h, ptr(qs), nq, qs.shape[1] if nq else self.dim,
                                 C.byref(pc), C.byref(oc), ptr(ids), ptr(dists), ptr(counts),
                                 ptr(stats)))
        return ids, dists, counts, stats

    def search_dev(self, d_queries, nq, params: SearchParams, options: EngineOptions,
                   d_ids, d_dists, d_counts=None, d_stats=None, stream: int = 0,
                   query_offset: int = 0):
        pc = params.c()
        oc = options.c(0, query_offset)
        check(lib().cagra_search_dev(self.h, ptr(d_queries), nq, C.byref(pc), C.byref(oc),
                                     ptr(d_ids), ptr(d_dists), ptr(d_counts), ptr(d_stats),
                                     C.c_void_p(stream)))

    def last_launch_count(self) -> int:
        return int(lib().cagra_last_launch_count(self.h))

    def batch_search(self, queries, params: SearchParams,
                     options: Optional[EngineOptions] = None) -> List[SearchResult]:
        ids, dists, counts, stats = self.search(queries, params, options)
        return _results(ids, dists, counts, stats)


def _results(ids, dists, counts, stats) -> List[SearchResult]:
    out = []
    for i in range(ids.shape[0]):
        c = int(counts[i])
        s = stats[i]
        out.append(SearchResult(ids[i, :c].copy(), dists[i, :c].copy(),
                                SearchStats(int(s["iterations"]), int(s["distance_evals"]),
                                            int(s["hash_resets"]), bool(s["converged"]))))
    return out


_INDEX_CACHE: dict = {}


def _index_for(graph: Graph, ds: Dataset, device: int) -> Index:
    # The reference re-reads host memory on every call; we keep the uploaded
    # index keyed on the host buffers' identity, shape and a content digest.
    key = (id(graph.ids), id(ds.data), graph.ids.shape, ds.data.shape, device)
    digest = (hash(graph.ids[:2].tobytes()), hash(ds.data[:2].tobytes()))
    hit = _INDEX_CACHE.get(key)
    if hit is not None and hit[1] == digest:
        return hit[0]
    if len(_INDEX_CACHE) > 8:
        _INDEX_CACHE.clear()
    ix = Index(ds, graph, device)
    _INDEX_CACHE[key] = (ix, digest, graph, ds)
    return ix


def batch_search(graph: Graph, ds: Dataset, queries: Dataset, params: SearchParams,
                 options: Optional[EngineOptions] = None) -> List[SearchResult]:
    """engine.hpp:38-40, validation order of engine.cpp:98-102."""
    options = options or EngineOptions()
    if queries.size() == 0:
        return []
    if queries.dim() != ds.dim():
        raise UsageError("batch_search: query dimension mismatch")
    params.validate()
    if options.mode == ExecutionMode.kSharedQueryWorkers and options.team_count < 2:
        raise UsageError("batch_search: shared mode requires team_count >= 2")
    if graph.num_nodes != ds.size():
        raise UsageError("search: graph/dataset size mismatch")
    return _index_for(graph, ds, options.device).batch_search(queries.data, params, options)


def search_one(graph: Graph, ds: Dataset, query, params: SearchParams,
               device: int = 0) -> SearchResult:
    """search.hpp:156-157: one traversal seeded with params.seed as given."""
    params.validate()
    q = np.asarray(query, np.float32).reshape(1, -1)
    if q.shape[1] != ds.dim():
        raise UsageError("search: query dimension mismatch")
    if graph.num_nodes != ds.size():
        raise UsageError("search: graph/dataset size mismatch")
    ix = _index_for(graph, ds, device)
    ids, dists, counts, stats = ix.search(q, params, EngineOptions(device=device), seed_mode=1)
    return _results(ids, dists, counts, stats)[0]


_SM_COUNT = None


def _parallel_workers() -> int:
    global _SM_COUNT
    if _SM_COUNT is None:
        try:
            import torch

            _SM_COUNT = torch.cuda.get_device_properties(0).multi_processor_count
        except Exception:
            _SM_COUNT = 148  # B200
    return _SM_COUNT


def choose_mode(batch_size: int, topm: int, thresholds: Optional[ModeThresholds] = None
                ) -> ExecutionMode:
    """engine.cpp:86-93; the default b_T is the device's SM count."""
    th = thresholds or ModeThresholds()
    b_t = th.batch_threshold if th.batch_threshold else _parallel_workers()
    if batch_size < b_t or topm > th.topm_threshold:
        return ExecutionMode.kSharedQueryWorkers
    return ExecutionMode.kPerQueryWorker


def mode_name(mode: ExecutionMode) -> str:
    return "per_query" if mode == ExecutionMode.kPerQueryWorker else "shared"


@dataclass
class BenchRecord:
    """engine.hpp:42-50."""
    dataset: str = ""
    mode: ExecutionMode = ExecutionMode.kPerQueryWorker
    params: SearchParams = field(default_factory=SearchParams)
    graph_degree: int = 0
    mean_iterations: float = 0.0
    recall: float = 0.0
    qps: float = 0.0


def bench_csv_header() -> str:
    return "dataset,mode,M,p,d,k,iterations,recall,qps"


def bench_csv_row(r: BenchRecord) -> str:
    """engine.cpp:124-131."""
    return (f"{r.dataset},{mode_name(r.mode)},{r.params.topm},{r.params.width},"
            f"{r.graph_degree},{r.params.k},{r.mean_iterations:.2f},{r.recall:.6f},{r.qps:.1f}")


def run_benchmark(graph: Graph, ds: Dataset, queries: Dataset, truth, param_grid,
                  options: Optional[EngineOptions] = None, dataset_name: str = "dataset"
                  ) -> List[BenchRecord]:
    """engine.cpp:133-180: per grid point an untimed warm-up then one timed
    batch_search (host wall clock, H2D/D2H included, index upload excluded)."""
    options = options or EngineOptions()
    if queries.size() == 0:
        raise UsageError("run_benchmark: no queries")
    if len(truth) < queries.size():
        raise UsageError("run_benchmark: missing ground truth rows")
    for p in param_grid:
        p.validate()
        for qi in range(queries.size()):
            if len(truth[qi]) < p.k:
                raise UsageError("run_benchmark: ground truth shorter than k")
    ix = _index_for(graph, ds, options.device)
    records = []
    for p in param_grid:
        ix.search(queries.data, p, options)
        t0 = time.perf_counter()
        ids, dists, counts, stats = ix.search(queries.data, p, options)
        el = time.perf_counter() - t0
        rsum = 0.0
        for qi in range(queries.size()):
            t = set(int(x) for x in truth[qi][:p.k])
            rsum += sum(1 for x in ids[qi, :counts[qi]] if int(x) in t) / p.k
        records.append(BenchRecord(dataset_name, options.mode, p, graph.degree,
                                   float(stats["iterations"].mean()), rsum / queries.size(),
                                   queries.size() / max(el, 1e-12)))
    return records
