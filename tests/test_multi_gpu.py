"""Multi-GPU layer (csrc/multi.cu, dist.build_graph_row_sharded) against the
one-device engine.

The box has one B200, so device sets repeat device 0 (several parts on one
GPU) and the multi-process paths run two gloo ranks on the same GPU: the code
paths (row ranges, peer copies / stores, slice seeds, gathers, K8 merges) are
the ones an 8-GPU node runs.  Bars: the row-sharded build and the replicated
search are bit-identical to one device; the dataset-sharded search equals the
same shards merged in one process (K8) and reaches the global ground truth.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_15136_b200 import capi, fodg
from paper_2308_15136_b200 import dist as pdist

pytestmark = pytest.mark.gpu


def _data(n, dim, seed):
    return capi.uniform_dataset(n, dim, seed)


def test_exact_knn_rows_equal_full_graph_rows(gpu):
    data = _data(70000, 40, 3)   # two-pass K1 (sample + append) on the row range
    ds = fodg.Dataset.from_array(data)
    full = fodg.exact_knn_graph(ds, 32)
    for a, b in [(0, 1), (1234, 40000), (69990, 70000), (0, 70000)]:
        part = fodg.exact_knn_rows(ds, 32, a, b)
        assert np.array_equal(part.ids, full.ids[a:b])
        assert np.array_equal(part.dists.view(np.uint32), full.dists[a:b].view(np.uint32))
    with pytest.raises(fodg.UsageError):
        fodg.exact_knn_rows(ds, 32, 10, 70001)


@pytest.mark.parametrize("devs", [[0, 0], [0, 0, 0]])
def test_build_graph_multi_bit_identical(gpu, devs):
    data = _data(60000, 48, 5)
    ds = fodg.Dataset.from_array(data)
    g1, _, k1 = fodg.build_graph(ds, 16, 32, return_knn=True)
    gm, info, km = fodg.build_graph_multi(ds, 16, devs, 32, return_knn=True)
    assert np.array_equal(k1.ids, km.ids)
    assert np.array_equal(k1.dists.view(np.uint32), km.dists.view(np.uint32))
    assert np.array_equal(g1.ids, gm.ids)
    assert info["knn_seconds"] > 0


def test_replicated_multi_index_equals_one_device(gpu):
    data = _data(30000, 32, 7)
    queries = _data(1001, 32, 8)
    ds = fodg.Dataset.from_array(data)
    g, _ = fodg.build_graph(ds, 16)
    ix = fodg.Index(ds, g)
    mx = fodg.MultiIndex(ds, [0, 0, 0], graph=g)
    for prm, opt in [(fodg.SearchParams(k=10, topm=64, width=4, seed=3), fodg.EngineOptions()),
                     (fodg.SearchParams(k=10, topm=32, width=1, seed=4),
                      fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers,
                                         team_count=4, exact_distances=True))]:
        a = ix.search(queries, prm, opt)
        b = mx.search(queries, prm, opt)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1].view(np.uint32),
                                                             b[1].view(np.uint32))
        assert np.array_equal(a[2], b[2])
        assert np.array_equal(a[3]["distance_evals"], b[3]["distance_evals"])
    # a batch smaller than the set: the spare parts get no slice
    a = ix.search(queries[:2], prm, opt)
    b = mx.search(queries[:2], prm, opt)
    assert np.array_equal(a[0], b[0])
    # graph built by the set itself (row-sharded, bit-identical) -> same results
    mx2 = fodg.MultiIndex(ds, [0, 0], degree=16)
    assert np.array_equal(mx2.search(queries[:2], prm, opt)[0], a[0])
    with pytest.raises(fodg.UsageError):
        mx.search(queries[:, :31], prm)


def test_dataset_sharded_multi_index(gpu):
    n, dim, nq, G = 24000, 32, 400, 3
    data = _data(n, dim, 11)
    queries = _data(nq, dim, 12)
    ds = fodg.Dataset.from_array(data)
    mx = fodg.MultiIndex(ds, [0] * G, degree=16, shard_mode="dataset")
    prm = fodg.SearchParams(k=10, topm=64, width=2, seed=3)
    ids, dists, counts, st = mx.search(queries, prm)
    # the same shards searched + merged in one process
    bounds = pdist.shard_bounds(n, G)
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
    assert np.array_equal(ids, mi.cpu().numpy().view(np.uint32))
    assert np.array_equal(dists.view(np.uint32), md.cpu().numpy().view(np.uint32))
    assert (counts == 10).all()
    assert (st["distance_evals"] > 0).all()
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    rec = np.mean([len(set(ids[q]) & set(gt[q])) / 10 for q in range(nq)])
    assert rec >= 0.95, rec
    # distances of merged ids are the sequential chain of the global rows
    for q in range(0, nq, 53):
        for j in range(10):
            assert dists[q, j] == fodg.squared_l2(data[ids[q, j]], queries[q])
    with pytest.raises(fodg.UsageError):
        fodg.MultiIndex(ds, [0, 0], graph=fodg.build_graph(ds, 16)[0], shard_mode="dataset")


def _row_sharded_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data = capi.uniform_dataset(50000, 36, 21)
        g, info = pdist.build_graph_row_sharded(fodg.Dataset.from_array(data), 16)
        out[rank] = g.ids.copy()
    finally:
        dist.destroy_process_group()


def test_row_sharded_build_world2_bit_identical(gpu):
    from test_dist import _free_port

    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_row_sharded_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    data = capi.uniform_dataset(50000, 36, 21)
    g1, _ = fodg.build_graph(fodg.Dataset.from_array(data), 16)
    for r in range(world):
        assert np.array_equal(res[r], g1.ids)
