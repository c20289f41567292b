"""Pin the C restatement (oracle/) before trusting it as the GPU checker.

(a) against golden fixtures produced by the unmodified reference
    (tests/golden/make_golden.py), and
(b) against the reference library itself (oracle/_ref) when it was built here,
(c) against the known answers of the reference's own unit tests.
CPU only.
"""
import numpy as np
import pytest

from oracle.bindings import make_params
from golden_util import load_golden

CORPORA = ["small", "accept"]


@pytest.mark.parametrize("name", CORPORA)
def test_generator_matches_reference_fixture_generator(oracle, name):
    g = load_golden(name)
    data = oracle.uniform_dataset(int(g["n"]), int(g["dim"]), int(g["data_seed"]))
    assert np.array_equal(data[:4].view(np.uint32), g["data_head"].view(np.uint32))


def test_generator_matches_engine_host_generator(oracle):
    from paper_2308_15136_b200 import capi

    a = oracle.uniform_dataset(300, 96, 424242)
    b = capi.uniform_dataset(300, 96, 424242)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("name", CORPORA)
def test_oracle_knn_and_optimize_match_golden(oracle, name):
    g = load_golden(name)
    data = oracle.uniform_dataset(int(g["n"]), int(g["dim"]), int(g["data_seed"]))
    ids, dists = oracle.exact_knn_graph(data, int(g["d_init"]))
    assert np.array_equal(ids, g["knn_ids"])
    assert np.array_equal(dists.view(np.uint32), g["knn_dists"].view(np.uint32))
    counts = oracle.count_detourable_routes(ids, dists)
    assert np.array_equal(counts, g["counts"])
    assert np.array_equal(oracle.optimize(ids, dists, int(g["d"])), g["graph"])


@pytest.mark.parametrize("name", CORPORA)
def test_oracle_search_matches_golden(oracle, name):
    g = load_golden(name)
    data = oracle.uniform_dataset(int(g["n"]), int(g["dim"]), int(g["data_seed"]))
    queries = oracle.uniform_dataset(int(g["nq"]), int(g["dim"]), int(g["query_seed"]))
    gt, gtd = oracle.exact_topk_batch(data, queries, 10)
    assert np.array_equal(gt, g["gt_ids"])
    for gi, (mode, m, p, pol, bits, ri, teams, seed) in enumerate(g["grid"].tolist()):
        prm = make_params(k=10, topm=m, width=p, hash_policy=pol, hash_bits=bits,
                          reset_interval=ri, seed=seed)
        ids, dists, cnt, st = oracle.batch_search(g["graph"], data, queries, prm, mode=mode,
                                                  team_count=teams)
        assert np.array_equal(ids, g[f"s{gi}_ids"]), gi
        assert np.array_equal(dists.view(np.uint32), g[f"s{gi}_dists"].view(np.uint32)), gi
        assert np.array_equal(st["distance_evals"], g[f"s{gi}_evals"]), gi
        assert np.array_equal(st["iterations"], g[f"s{gi}_iters"]), gi
        assert np.array_equal(st["hash_resets"], g[f"s{gi}_resets"]), gi
        assert np.array_equal(st["converged"], g[f"s{gi}_conv"]), gi


def test_oracle_matches_reference_library(oracle, reference):
    if reference is None:
        pytest.skip("oracle/_ref not built in this environment (needs /root/reference)")
    for seed, (n, dim, k) in [(5, (700, 7, 12)), (6, (500, 33, 20))]:
        data = oracle.uniform_dataset(n, dim, seed)
        a = oracle.exact_knn_graph(data, k)
        b = reference.exact_knn_graph(data, k)
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
        graph, _ = reference.optimize(b[0], b[1], k // 2)
        assert np.array_equal(oracle.optimize(*a, k // 2), graph)
        q = oracle.uniform_dataset(40, dim, seed + 100)
        ix = reference.index(data, graph)
        for mode in (0, 1):
            prm = make_params(k=5, topm=24, width=1 + mode, seed=seed, hash_policy=0)
            r1 = oracle.batch_search(graph, data, q, prm, mode=mode)
            r2 = ix.batch_search(q, prm, mode=mode)
            assert np.array_equal(r1[0], r2[0])
            assert np.array_equal(r1[3]["distance_evals"], r2[3]["distance_evals"])


# ---- known answers of the reference's unit tests -------------------------

def test_kat_squared_l2(oracle):
    # test_core.cpp:13-20
    assert oracle.squared_l2(np.array([3, 4], np.float32), np.zeros(2, np.float32)) == 25.0


def test_kat_exact_topk_1d(oracle):
    # test_core.cpp:22-46: points {0,1,3,7}
    data = np.array([[0], [1], [3], [7]], np.float32)
    ids, _ = oracle.exact_topk_batch(data, np.array([[2.9]], np.float32), 1)
    assert ids.tolist() == [[2]]
    ids, _ = oracle.exact_topk_batch(data, np.array([[0.4]], np.float32), 2)
    assert ids.tolist() == [[0, 1]]
    tie = np.array([[1], [1], [1], [5]], np.float32)
    ids, _ = oracle.exact_topk_batch(tie, np.array([[1]], np.float32), 3)
    assert ids.tolist() == [[0, 1, 2]]


def test_kat_exact_knn_graph_1d(oracle):
    # test_knn_build.cpp:32-54
    data = np.array([[0], [1], [3], [7]], np.float32)
    ids, _ = oracle.exact_knn_graph(data, 1)
    assert ids.ravel().tolist() == [1, 0, 1, 2]
    ids, d = oracle.exact_knn_graph(data, 2)
    assert ids[3].tolist() == [2, 1] and d[3].tolist() == [16.0, 36.0]
    dup = np.array([[2], [9], [2], [30]], np.float32)
    ids, d = oracle.exact_knn_graph(dup, 1)
    assert ids[0, 0] == 2 and ids[2, 0] == 0 and d[0, 0] == 0.0


def _knn(rows):
    ids = np.array(rows, np.uint32)
    dists = np.tile(np.arange(1, ids.shape[1] + 1, dtype=np.float32), (ids.shape[0], 1))
    return ids, dists


def test_kat_graph_opt(oracle):
    # test_graph_opt.cpp:67-74 two-node example
    ids, dists = _knn([[1, 2], [2, 0], [0, 1]])
    c = oracle.count_detourable_routes(ids, dists)
    assert c[0, 0] == 0 and c[0, 1] == 1
    # :107-122 reorder_and_prune
    ids, dists = _knn([[1, 2, 3], [2, 3, 0], [3, 0, 1], [0, 1, 2]])
    counts = np.zeros((4, 3), np.uint32)
    counts[0, 1] = 1
    pr = oracle.reorder_and_prune(ids, counts, 2)
    assert pr[0].tolist() == [1, 3]
    # :154-190 merge [a,b,c,e] + [w,x,y,z] -> [a,w,b,x]
    a, b, c_, e, w, x, y, z = range(1, 9)
    pr = np.array([[a, b, c_, e]], np.uint32)
    out = oracle.merge_graphs(pr, np.array([4], np.uint32), np.array([[w, x, y, z]], np.uint32))
    assert out[0].tolist() == [a, w, b, x]
    out = oracle.merge_graphs(pr, np.array([1], np.uint32), np.array([[w, 0, 0, 0]], np.uint32))
    assert out[0].tolist() == [a, w, b, c_]
    out = oracle.merge_graphs(pr, np.array([1], np.uint32), np.array([[a, 0, 0, 0]], np.uint32))
    assert out[0].tolist() == [a, b, c_, e]
