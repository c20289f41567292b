"""Multi-GPU layouts (paper_2308_15136_b200/dist.py).

CPU (gloo, world size 2): shard / query partitioning and the one data-path
collective of the dataset-sharded layout (all-gather of per-shard top-k).
GPU: G dataset shards on one device — per-shard device graphs + searches,
the K8 merge against a host merge of the same lists, recall against the
global ground truth; and query-sharding seeds equal to a 1-GPU run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_15136_b200 import dist as pdist
from paper_2308_15136_b200 import fodg


def test_shard_bounds_cover_and_balance():
    for n, w in [(10, 3), (1000000, 8), (7, 7), (8, 1)]:
        b = pdist.shard_bounds(n, w)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        sizes = [e - s for s, e in b]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(fodg.UsageError):
        pdist.shard_bounds(3, 4)
    assert pdist.query_slice(1, 2, 0) == (0, 1) and pdist.query_slice(1, 2, 1) == (1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nq, k = 5, 4
        # rank r's per-shard result: local ids r*100+q*10+j, dists ascending
        ids = torch.tensor([[rank * 100 + q * 10 + j for j in range(k)] for q in range(nq)],
                           dtype=torch.int32)
        dists = torch.tensor([[float(j + rank) + 0.5 * q for j in range(k)] for q in range(nq)])
        gi, gd = pdist.exchange_topk(ids, dists)
        out[rank] = (gi.numpy().copy(), gd.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_exchange_topk_gloo_world2():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        gi, gd = res[r]
        assert gi.shape == (world, 5, 4) and gd.shape == (world, 5, 4)
        for src in range(world):
            assert gi[src, 2, 1] == src * 100 + 21
            assert gd[src, 3, 0] == pytest.approx(src + 1.5)
    assert np.array_equal(res[0][0], res[1][0])


def _host_merge(ids, dists, offsets, k):
    out = []
    for q in range(ids.shape[1]):
        pool = sorted((float(dists[g, q, j]), int(ids[g, q, j]) + offsets[g])
                      for g in range(ids.shape[0]) for j in range(k)
                      if ids[g, q, j] != -1)
        row, prev = [], None
        for d, i in pool:
            if i == prev:
                continue
            prev = i
            row.append(i)
        out.append(row[:k])
    return np.array(out)


@pytest.mark.gpu
def test_dataset_sharded_search_on_one_device(gpu, oracle):
    n, dim, nq, G, k = 24000, 32, 400, 4, 10
    data = oracle.uniform_dataset(n, dim, 5)
    queries = oracle.uniform_dataset(nq, dim, 6)
    gt, _ = fodg.exact_topk_batch(fodg.Dataset.from_array(data), queries, k)
    bounds = pdist.shard_bounds(n, G)
    offsets = [s for s, _ in bounds]
    prm = fodg.SearchParams(k=k, topm=64, width=2, seed=3)
    per_ids, per_d = [], []
    for s, e in bounds:
        sh = pdist.ShardedIndex.build(np.ascontiguousarray(data[s:e]), s, 16)
        qd = torch.zeros((nq, sh.index.ld), dtype=torch.float32, device="cuda:0")
        qd[:, :dim] = torch.from_numpy(queries).cuda()
        i, d = sh.search_local(qd, nq, prm)
        per_ids.append(i)
        per_d.append(d)
    gi, gd = torch.stack(per_ids), torch.stack(per_d)
    torch.cuda.synchronize()
    mi, md = pdist.merge_shard_topk(gi, gd, offsets)
    torch.cuda.synchronize()
    ids = mi.cpu().numpy().astype(np.int64)
    host = _host_merge(gi.cpu().numpy().astype(np.int64), gd.cpu().numpy(), offsets, k)
    assert np.array_equal(ids, host)
    assert (np.diff(md.cpu().numpy(), axis=1) >= 0).all()
    rec = np.mean([len(set(ids[q]) & set(gt[q].astype(np.int64))) / k for q in range(nq)])
    assert rec >= 0.95, rec
    # distances of the merged ids are the sequential chain of the global rows
    for q in range(0, nq, 37):
        for j in range(k):
            assert md[q, j].item() == fodg.squared_l2(data[ids[q, j]], queries[q])


@pytest.mark.gpu
def test_query_sharding_matches_single_gpu(gpu, oracle):
    n, dim, nq = 8000, 24, 300
    data = oracle.uniform_dataset(n, dim, 8)
    queries = oracle.uniform_dataset(nq, dim, 9)
    ds = fodg.Dataset.from_array(data)
    g, _ = fodg.build_graph(ds, 16)
    ix = fodg.Index(ds, g)
    prm = fodg.SearchParams(k=10, topm=48, width=2, seed=21)
    full = ix.search(queries, prm)[0]
    parts = []
    for r in range(3):
        s, e = pdist.query_slice(nq, 3, r)
        parts.append(ix.search(queries[s:e], prm, query_offset=s)[0])
    assert np.array_equal(np.concatenate(parts), full)


def _sharded_search_worker(rank, world, port, out):
    """One rank of a dataset-sharded index on the (shared) GPU, gloo exchange."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_15136_b200 import capi

        n, dim, nq = 20000, 24, 300
        data = capi.uniform_dataset(n, dim, 41)
        queries = capi.uniform_dataset(nq, dim, 42)
        bounds = pdist.shard_bounds(n, world)
        s, e = bounds[rank]
        sh = pdist.ShardedIndex.build(np.ascontiguousarray(data[s:e]), s, 16)
        qd = torch.zeros((nq, sh.index.ld), dtype=torch.float32, device="cuda:0")
        qd[:, :dim] = torch.from_numpy(queries).cuda()
        prm = fodg.SearchParams(k=10, topm=64, width=2, seed=5)
        mi, md = sh.search(qd, nq, prm, [b[0] for b in bounds])
        torch.cuda.synchronize()
        out[rank] = (mi.cpu().numpy().copy(), md.cpu().numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_index_search_world2_matches_one_process(gpu, oracle):
    # ShardedIndex.search end to end over 2 ranks (gloo all-gather, K8 merge)
    # equals the same shards searched and merged in one process, and reaches
    # the global ground truth
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_sharded_search_worker, args=(world, _free_port(), out), nprocs=world,
                 join=True)
        res = dict(out)
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    from paper_2308_15136_b200 import capi

    n, dim, nq = 20000, 24, 300
    data = capi.uniform_dataset(n, dim, 41)
    queries = capi.uniform_dataset(nq, dim, 42)
    bounds = pdist.shard_bounds(n, world)
    prm = fodg.SearchParams(k=10, topm=64, width=2, seed=5)
    li, ld_ = [], []
    for s, e in bounds:
        sh = pdist.ShardedIndex.build(np.ascontiguousarray(data[s:e]), s, 16)
        qd = torch.zeros((nq, sh.index.ld), dtype=torch.float32, device="cuda:0")
        qd[:, :dim] = torch.from_numpy(queries).cuda()
        i, d = sh.search_local(qd, nq, prm)
        li.append(i)
        ld_.append(d)
    mi, md = pdist.merge_shard_topk(torch.stack(li), torch.stack(ld_), [b[0] for b in bounds])
    torch.cuda.synchronize()
    assert np.array_equal(res[0][0], mi.cpu().numpy())
    assert np.array_equal(res[0][1].view(np.uint32), md.cpu().numpy().view(np.uint32))
    gt, _ = fodg.exact_topk_batch(fodg.Dataset.from_array(data), queries, 10)
    ids = res[0][0].astype(np.int64)
    rec = np.mean([len(set(ids[q]) & set(gt[q].astype(np.int64))) / 10 for q in range(nq)])
    assert rec >= 0.95, rec
