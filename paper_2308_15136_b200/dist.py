"""Multi-GPU search on one box: one process per GPU (torch.distributed).

Two layouts; the reference itself has no distributed code:

* query-sharded (replicated index) — every rank holds the whole index and
  searches its own contiguous slice of the batch; no collective on the data
  path.  `query_slice` gives the slice and the `query_offset` that keeps every
  query's seed (mix_seed(seed ^ (0x0bad + global index)), engine.cpp:108)
  identical to a single-GPU run, so results do not depend on the GPU count.

* dataset-sharded — rank r indexes the contiguous id range `shard_bounds(n,
  G)[r]` with its own graph (ids local to the shard); every rank searches
  every query, the per-shard top-k lists are exchanged with ONE all-gather
  (NCCL over NVLink on the box, gloo in the CPU tests) and merged by the K8
  kernel (cagra_merge_shard_topk_dev): shard offsets turn local ids into
  global ids, order (dist, id) as merge_team_results (engine.cpp:24-34).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import capi, fodg


def shard_bounds(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced [start, end) id ranges (first n % world shards one longer)."""
    if world < 1 or n < world:
        raise fodg.UsageError("shard_bounds: need 1 <= world <= n")
    base, extra = divmod(n, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def query_slice(nq: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, end) of this rank's queries; start is the rank's query_offset."""
    return shard_bounds(nq, world)[rank] if nq >= world else ((0, nq) if rank == 0 else (nq, nq))


def exchange_topk(ids, dists, group=None):
    """All-gather of every rank's [nq, k] (ids, dists): returns [G, nq, k]
    tensors on every rank.  The one data-path collective of the
    dataset-sharded layout (NCCL on device tensors, gloo on CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gi = [torch.empty_like(ids) for _ in range(world)]
    gd = [torch.empty_like(dists) for _ in range(world)]
    dist.all_gather(gi, ids.contiguous(), group=group)
    dist.all_gather(gd, dists.contiguous(), group=group)
    return torch.stack(gi), torch.stack(gd)


def merge_shard_topk(stacked_ids, stacked_dists, offsets, device: int = 0, stream: int = 0):
    """K8 on the device: [G, nq, k] local (ids, dists) + shard offsets -> global
    top-k [nq, k] by (dist, global id)."""
    import torch

    G, nq, k = stacked_ids.shape
    out_i = torch.empty((nq, k), dtype=torch.int32, device=stacked_ids.device)
    out_d = torch.empty((nq, k), dtype=torch.float32, device=stacked_ids.device)
    offs = np.ascontiguousarray(np.asarray(offsets, np.uint64))
    capi.check(capi.lib().cagra_merge_shard_topk_dev(
        capi.ptr(stacked_ids.contiguous()), capi.ptr(stacked_dists.contiguous()), G, nq, k,
        capi.ptr(offs), capi.ptr(out_i), capi.ptr(out_d), device, C.c_void_p(stream)))
    return out_i, out_d


def build_graph_row_sharded(ds: fodg.Dataset, degree: int, device: int = 0, group=None,
                            d_init: Optional[int] = None):
    """Row-sharded multi-process graph build: rank r
    computes the exact kNN rows of its contiguous row range on its GPU
    (cagra_exact_knn_rows — the parallel_for over rows of knn_build.cpp:49,
    split over ranks), ONE all-gather assembles the N x d_init kNN graph on
    every rank, and each rank runs the rank optimize (graph_opt.cpp:211-246)
    locally, so no second collective is needed.  The graph is bit-identical
    to a one-GPU build.  Returns (Graph, info)."""
    import time

    import torch
    import torch.distributed as dist

    d_init = d_init or 2 * degree
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = ds.size()
    bounds = shard_bounds(n, world)
    s, e = bounds[rank]
    t0 = time.perf_counter()
    part = fodg.exact_knn_rows(ds, d_init, s, e, device)
    t_rows = time.perf_counter() - t0
    maxr = max(b - a for a, b in bounds)
    nccl = dist.get_backend(group) == "nccl"
    where = torch.device("cuda", device) if nccl else torch.device("cpu")
    ids = torch.zeros((maxr, d_init), dtype=torch.int32, device=where)
    dists = torch.zeros((maxr, d_init), dtype=torch.float32, device=where)
    ids[:e - s] = torch.from_numpy(part.ids.view(np.int32)).to(where)
    dists[:e - s] = torch.from_numpy(part.dists).to(where)
    gi = [torch.empty_like(ids) for _ in range(world)]
    gd = [torch.empty_like(dists) for _ in range(world)]
    dist.all_gather(gi, ids, group=group)
    dist.all_gather(gd, dists, group=group)
    kid = np.concatenate([gi[r][:b - a].cpu().numpy().view(np.uint32)
                          for r, (a, b) in enumerate(bounds)])
    kd = np.concatenate([gd[r][:b - a].cpu().numpy() for r, (a, b) in enumerate(bounds)])
    t_gather = time.perf_counter() - t0 - t_rows
    st = fodg.OptimizeStats()
    g = fodg.optimize(fodg.KnnGraph(n, d_init, kid, kd), degree,
                      fodg.OptimizeOptions(device=device), stats=st)
    return g, {"knn_rows_seconds": t_rows, "gather_seconds": t_gather,
               "optimize_seconds": st.total_seconds, "rows": e - s}


class ShardedIndex:
    """This rank's shard of a dataset-sharded index (ids local to the shard).

    `build` constructs the shard graph on this rank's GPU (exact kNN + rank
    optimize over the shard's rows only)."""

    def __init__(self, data_shard: np.ndarray, graph: fodg.Graph, offset: int, device: int = 0):
        self.offset = int(offset)
        self.device = device
        self.index = fodg.Index(fodg.Dataset.from_array(data_shard), graph, device)
        self.build_info = {"knn_seconds": 0.0, "optimize_seconds": 0.0}

    @classmethod
    def build(cls, data_shard: np.ndarray, offset: int, degree: int, device: int = 0):
        ds = fodg.Dataset.from_array(data_shard)
        g, info = fodg.build_graph(ds, degree, device=device)
        sh = cls(data_shard, g, offset, device)
        sh.build_info = info
        return sh

    def search_local(self, d_queries, nq: int, params: fodg.SearchParams,
                     opts: Optional[fodg.EngineOptions] = None, stream: Optional[int] = None,
                     stats=None):
        """Per-shard search of device-resident queries (row stride = index.ld),
        asynchronous on `stream` (default: torch's current stream on this
        device, so torch/NCCL work queued after it is ordered after the search).
        `stats`: optional [nq, 6] int32 device tensor for the per-query counters."""
        import torch

        opts = opts or fodg.EngineOptions(device=self.device)
        dev = torch.device("cuda", self.device)
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        ids = torch.empty((nq, params.k), dtype=torch.int32, device=dev)
        dists = torch.empty((nq, params.k), dtype=torch.float32, device=dev)
        self.index.search_dev(d_queries, nq, params, opts, ids, dists, None, stats, stream)
        return ids, dists

    def search(self, d_queries, nq: int, params: fodg.SearchParams, offsets: List[int],
               opts: Optional[fodg.EngineOptions] = None, group=None):
        """Global top-k for every query on every rank: local search, one
        all-gather of the per-shard lists, K8 merge.  Everything is queued on
        torch's current stream: with NCCL the all-gather is stream-ordered after
        the search (no host sync); with gloo (CPU tensors) the copy to the host
        synchronises first."""
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", self.device)
        stream = torch.cuda.current_stream(dev).cuda_stream
        ids, dists = self.search_local(d_queries, nq, params, opts, stream)
        if dist.get_backend(group) == "nccl":
            gi, gd = exchange_topk(ids, dists, group)
        else:
            gi, gd = exchange_topk(ids.cpu(), dists.cpu(), group)
            gi, gd = gi.to(dev), gd.to(dev)
        return merge_shard_topk(gi, gd, offsets, self.device, stream)
