"""GPU parity: the sm_100a engine, through the C ABI, against the reference's
own outputs (golden fixtures from the unmodified reference) and the C oracle.

Bar: bit-exact for every integer/id output and for every distance (the engine
reproduces the sequential fp32 chain of squared_l2, dataset.hpp:33-43), and
exact counters (distance_evals, iterations, hash_resets, converged) in
reference-semantics mode.  The fast mode (team-reduced in-loop distances) is
held to recall within 0.5 pp and >= 99% exact-ID match, with reported
distances still bit-exact.
"""
import numpy as np
import pytest

from golden_util import load_golden
from oracle.bindings import make_params
from paper_2308_15136_b200 import capi, fodg

pytestmark = pytest.mark.gpu

CORPORA = ["small", "accept"]


def corpus(oracle, name):
    g = load_golden(name)
    data = oracle.uniform_dataset(int(g["n"]), int(g["dim"]), int(g["data_seed"]))
    queries = oracle.uniform_dataset(int(g["nq"]), int(g["dim"]), int(g["query_seed"]))
    return g, data, queries


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------ kNN / GT ----
@pytest.mark.parametrize("name", CORPORA)
def test_exact_knn_graph_bit_exact(gpu, oracle, name):
    g, data, _ = corpus(oracle, name)
    knn = fodg.exact_knn_graph(fodg.Dataset.from_array(data), int(g["d_init"]))
    assert np.array_equal(knn.ids, g["knn_ids"])
    assert np.array_equal(bits(knn.dists), bits(g["knn_dists"]))


@pytest.mark.parametrize("name", CORPORA)
def test_ground_truth_bit_exact(gpu, oracle, name):
    g, data, queries = corpus(oracle, name)
    ids, dists = fodg.exact_topk_batch(fodg.Dataset.from_array(data), queries, 10)
    assert np.array_equal(ids, g["gt_ids"])
    assert np.array_equal(bits(dists), bits(g["gt_dists"]))


def test_knn_known_answers(gpu):
    # test_knn_build.cpp:32-54, test_core.cpp:22-46
    ds = fodg.Dataset(1, [0, 1, 3, 7])
    assert fodg.exact_knn_graph(ds, 1).ids.ravel().tolist() == [1, 0, 1, 2]
    g2 = fodg.exact_knn_graph(ds, 2)
    assert g2.ids[3].tolist() == [2, 1] and g2.dists[3].tolist() == [16.0, 36.0]
    with pytest.raises(fodg.UsageError):
        fodg.exact_knn_graph(ds, 4)
    dup = fodg.Dataset(1, [2, 9, 2, 30])
    gd = fodg.exact_knn_graph(dup, 1)
    assert gd.ids[0, 0] == 2 and gd.ids[2, 0] == 0 and gd.dists[0, 0] == 0.0
    assert fodg.exact_topk(ds, [2.9], 1).ids.tolist() == [2]
    assert fodg.exact_topk(ds, [0.4], 2).ids.tolist() == [0, 1]
    tie = fodg.Dataset(1, [1, 1, 1, 5])
    assert fodg.exact_topk(tie, [1], 3).ids.tolist() == [0, 1, 2]


def test_knn_odd_dimension_and_ragged_tiles(gpu, oracle):
    # dim not a multiple of 4 / 32, n not a multiple of the 128-point tile
    for n, dim, k, seed in [(333, 5, 7, 3), (1000, 37, 40, 4), (129, 1, 3, 9)]:
        data = oracle.uniform_dataset(n, dim, seed)
        ref_ids, ref_d = oracle.exact_knn_graph(data, k)
        knn = fodg.exact_knn_graph(fodg.Dataset.from_array(data), k)
        assert np.array_equal(knn.ids, ref_ids)
        assert np.array_equal(bits(knn.dists), bits(ref_d))


@pytest.mark.parametrize("split", ["1", "3"])
@pytest.mark.parametrize("n,dim,k,two_pass", [
    (3000, 128, 64, False),    # single pass, D=128
    (70000, 96, 128, True),    # sample pass + append pass (DEEP shape, d_init 128)
    (90000, 37, 40, True),     # odd dim, ragged last tile
    (4000, 200, 32, False),    # K > 512 (bf16x3): query tile streamed with each data tile
    (70000, 960, 128, True),   # GIST shape, streamed query tile, both passes
])
def test_knn_tensor_core_path_bit_exact(gpu, oracle, monkeypatch, n, dim, k, two_pass, split):
    # K1 on tcgen05 (knn_tc.cu) against the SIMT sequential-chain kernel (itself
    # bit-exact vs the reference above) and, on the small case, the oracle;
    # both filter splits (fp16 single term, bf16x3).
    data = oracle.uniform_dataset(n, dim, 1000 + n)
    ds = fodg.Dataset.from_array(data)
    monkeypatch.setenv("CAGRA_KNN_PATH", "auto")
    monkeypatch.setenv("CAGRA_KNN_SPLIT", split)
    tc = fodg.exact_knn_graph(ds, k)
    st = capi.knn_last_stats()
    assert st["rows"] == n and st["reranked"] >= n * k, st   # the tensor-core path ran
    queries = oracle.uniform_dataset(500, dim, 77)
    gt_tc = fodg.exact_topk_batch(ds, queries, 10)
    monkeypatch.setenv("CAGRA_KNN_PATH", "simt")
    simt = fodg.exact_knn_graph(ds, k)
    assert capi.knn_last_stats()["rows"] == 0
    gt_simt = fodg.exact_topk_batch(ds, queries, 10)
    assert np.array_equal(tc.ids, simt.ids)
    assert np.array_equal(bits(tc.dists), bits(simt.dists))
    assert np.array_equal(gt_tc[0], gt_simt[0])
    assert np.array_equal(bits(gt_tc[1]), bits(gt_simt[1]))
    if n <= 5000:
        ref_ids, ref_d = oracle.exact_knn_graph(data, k)
        assert np.array_equal(tc.ids, ref_ids)
        assert np.array_equal(bits(tc.dists), bits(ref_d))


@pytest.mark.parametrize("scale,offset", [(1e6, 3e7), (1e-12, 0.0), (1e-18, 0.0), (1.0, -250.0)])
def test_knn_tensor_core_extreme_magnitudes(gpu, oracle, monkeypatch, scale, offset):
    # the fp16 split scales rows by a power of two chosen from the largest
    # centred norm: huge, tiny and offset data stay bit-exact (the error
    # bound covers fp16 rounding and subnormal operands)
    base = oracle.uniform_dataset(70000, 48, 31)
    data = np.ascontiguousarray((base * np.float32(scale) + np.float32(offset)).astype(np.float32))
    # a few rows far from the rest (large centred norms next to small ones)
    data[::9973] *= np.float32(3.0)
    ds = fodg.Dataset.from_array(data)
    monkeypatch.setenv("CAGRA_KNN_PATH", "auto")
    tc = fodg.exact_knn_graph(ds, 24)
    assert capi.knn_last_stats()["rows"] == 70000
    monkeypatch.setenv("CAGRA_KNN_PATH", "simt")
    simt = fodg.exact_knn_graph(ds, 24)
    assert np.array_equal(tc.ids, simt.ids)
    assert np.array_equal(bits(tc.dists), bits(simt.dists))


def test_knn_tensor_core_single_pass_forced(gpu, oracle, monkeypatch):
    # the single-pass list mode (used for retried rows) on a size that would
    # normally take two passes
    data = oracle.uniform_dataset(70000, 24, 5)
    ds = fodg.Dataset.from_array(data)
    monkeypatch.setenv("CAGRA_KNN_PATH", "auto")
    monkeypatch.setenv("CAGRA_TC_ONEPASS", "1")
    one = fodg.exact_knn_graph(ds, 32)
    monkeypatch.delenv("CAGRA_TC_ONEPASS")
    two = fodg.exact_knn_graph(ds, 32)
    assert np.array_equal(one.ids, two.ids)
    assert np.array_equal(bits(one.dists), bits(two.dists))


# ------------------------------------------------------------ optimize ----
@pytest.mark.parametrize("name", CORPORA)
def test_optimize_stages_bit_exact(gpu, oracle, name):
    g, data, _ = corpus(oracle, name)
    knn = fodg.KnnGraph(int(g["n"]), int(g["d_init"]), g["knn_ids"], g["knn_dists"])
    d = int(g["d"])
    counts = fodg.count_detourable_routes(knn)
    assert np.array_equal(counts, g["counts"])
    pruned = fodg.reorder_and_prune(knn, counts, d)
    assert np.array_equal(pruned.ids, oracle.reorder_and_prune(g["knn_ids"], g["counts"], d))
    rc, ri = fodg._reverse_arrays(pruned, d)
    orc_rc, orc_ri = oracle.build_reverse_graph(pruned.ids, d)
    assert np.array_equal(rc, orc_rc)
    for y in range(len(rc)):
        assert np.array_equal(ri[y, :rc[y]], orc_ri[y, :orc_rc[y]])
    rev = fodg.build_reverse_graph(pruned, d)
    merged = fodg.merge_graphs(pruned, rev, d)
    assert np.array_equal(merged.ids, g["graph"])
    st = fodg.OptimizeStats()
    assert np.array_equal(fodg.optimize(knn, d, stats=st).ids, g["graph"])
    assert st.total_seconds > 0


@pytest.mark.parametrize("name", CORPORA)
def test_build_graph_pipeline_bit_exact(gpu, oracle, name):
    g, data, _ = corpus(oracle, name)
    graph, info, knn = fodg.build_graph(fodg.Dataset.from_array(data), int(g["d"]),
                                        int(g["d_init"]), return_knn=True)
    assert np.array_equal(knn.ids, g["knn_ids"])
    assert np.array_equal(graph.ids, g["graph"])
    assert info["knn_seconds"] > 0 and info["optimize_seconds"] > 0


def _knn(rows):
    ids = np.array(rows, np.uint32)
    dists = np.tile(np.arange(1, ids.shape[1] + 1, dtype=np.float32), (ids.shape[0], 1))
    return fodg.KnnGraph(ids.shape[0], ids.shape[1], ids, dists)


def test_optimize_known_answers(gpu):
    # test_graph_opt.cpp:67-74
    c = fodg.count_detourable_routes(_knn([[1, 2], [2, 0], [0, 1]]))
    assert c[0, 0] == 0 and c[0, 1] == 1
    # :94-105 no 2-hop routes; unsorted input rejected
    g = _knn([[1, 2], [3, 4], [4, 5], [5, 0], [0, 2], [1, 3]])
    ref = np.zeros((6, 2), np.uint32)
    assert fodg.count_detourable_routes(g).shape == ref.shape
    bad = _knn([[1, 2], [2, 0], [0, 1]])
    bad.dists[0, 0], bad.dists[0, 1] = bad.dists[0, 1], bad.dists[0, 0]
    with pytest.raises(fodg.UsageError):
        fodg.count_detourable_routes(bad)
    # :107-132 reorder_and_prune
    k4 = _knn([[1, 2, 3], [2, 3, 0], [3, 0, 1], [0, 1, 2]])
    counts = np.zeros((4, 3), np.uint32)
    counts[0, 1] = 1
    assert fodg.reorder_and_prune(k4, counts, 2).ids[0].tolist() == [1, 3]
    flat = np.full((4, 3), 7, np.uint32)
    assert fodg.reorder_and_prune(k4, flat, 2).ids[0].tolist() == [1, 2]
    with pytest.raises(fodg.UsageError):
        fodg.reorder_and_prune(k4, flat, 4)
    # :134-152 reverse: 2-cycle, smaller rank wins, empty row
    pr = fodg.Graph(2, 1, np.array([[1], [0]], np.uint32))
    assert fodg.build_reverse_graph(pr, 1).rows == [[1], [0]]
    pr3 = fodg.Graph(3, 2, np.array([[1, 2], [2, 0], [1, 0]], np.uint32))
    rev = fodg.build_reverse_graph(pr3, 1)
    assert rev.rows[2] == [1] and rev.rows[0] == [1] and rev.rows[1] == [0]
    # :154-190 merge
    a, b, c_, e, w, x, y, z = range(1, 9)
    p = fodg.Graph(9, 4, np.zeros((9, 4), np.uint32))
    p.ids[0] = [a, b, c_, e]
    rows = [[w, x, y, z]] + [[]] * 8
    for v in range(1, 9):
        p.ids[v] = [(v + j) % 9 if (v + j) % 9 != v else (v + 5) % 9 for j in range(1, 5)]
    out = fodg.merge_graphs(p, fodg.ReverseGraph(9, rows), 4)
    assert out.ids[0].tolist() == [a, w, b, x]
    out = fodg.merge_graphs(p, fodg.ReverseGraph(9, [[w]] + [[]] * 8), 4)
    assert out.ids[0].tolist() == [a, w, b, c_]
    out = fodg.merge_graphs(p, fodg.ReverseGraph(9, [[a]] + [[]] * 8), 4)
    assert out.ids[0].tolist() == [a, b, c_, e]
    # :231-235 2-cycle boundary
    two = fodg.optimize(_knn([[1], [0]]), 1)
    assert two.ids.ravel().tolist() == [1, 0]


def test_optimize_random_vs_oracle(gpu, oracle):
    # test_graph_opt.cpp:76-85 style: random small graphs, several seeds/degrees
    for seed, (n, dim, k, d) in [(1, (60, 4, 10, 5)), (2, (800, 8, 24, 12)), (3, (2048, 32, 48, 16))]:
        data = oracle.uniform_dataset(n, dim, seed)
        ids, dists = oracle.exact_knn_graph(data, k)
        knn = fodg.KnnGraph(n, k, ids, dists)
        assert np.array_equal(fodg.count_detourable_routes(knn),
                              oracle.count_detourable_routes(ids, dists))
        assert np.array_equal(fodg.optimize(knn, d).ids, oracle.optimize(ids, dists, d))
        # reorder only / reverse only ablations (acceptance.cpp:113-116)
        ro = fodg.optimize(knn, d, fodg.OptimizeOptions(reorder=True, add_reverse=False))
        counts = oracle.count_detourable_routes(ids, dists)
        assert np.array_equal(ro.ids, oracle.reorder_and_prune(ids, counts, d))
        rv = fodg.optimize(knn, d, fodg.OptimizeOptions(reorder=False, add_reverse=True))
        trunc = np.ascontiguousarray(ids[:, :d])
        rc, ri = oracle.build_reverse_graph(trunc, d)
        assert np.array_equal(rv.ids, oracle.merge_graphs(trunc, rc, ri))


# -------------------------------------------------------------- search ----
def _golden_search(gpu, oracle, name, exact):
    g, data, queries = corpus(oracle, name)
    ds = fodg.Dataset.from_array(data)
    graph = fodg.Graph(int(g["n"]), int(g["d"]), g["graph"])
    ix = fodg.Index(ds, graph)
    out = []
    for gi, (mode, m, p, pol, hb, ri, teams, seed) in enumerate(g["grid"].tolist()):
        prm = fodg.SearchParams(k=10, topm=m, width=p, hash_policy=fodg.HashPolicy(pol),
                                hash_bits=hb, reset_interval=ri, seed=seed)
        # multi_cta=1: the lockstep team order (multi-CTA has its own test)
        opts = fodg.EngineOptions(mode=fodg.ExecutionMode(mode), team_count=teams,
                                  exact_distances=exact, multi_cta=1)
        ids, dists, counts, st = ix.search(queries, prm, opts)
        out.append((gi, g, ids, dists, counts, st))
    return out


@pytest.mark.parametrize("name", CORPORA)
def test_search_reference_semantics_bit_exact(gpu, oracle, name):
    """exact_distances=1: ids, dists, evals, iterations, resets, converged all
    equal the reference's for every query at every grid point (per-query and
    shared mode; standard and forgettable visited tables incl. Full resets)."""
    for gi, g, ids, dists, counts, st in _golden_search(gpu, oracle, name, True):
        assert np.array_equal(ids, g[f"s{gi}_ids"]), gi
        assert np.array_equal(bits(dists), bits(g[f"s{gi}_dists"])), gi
        assert np.array_equal(counts, g[f"s{gi}_counts"]), gi
        assert np.array_equal(st["distance_evals"], g[f"s{gi}_evals"]), gi
        assert np.array_equal(st["iterations"], g[f"s{gi}_iters"]), gi
        assert np.array_equal(st["hash_resets"], g[f"s{gi}_resets"]), gi
        assert np.array_equal(st["converged"], g[f"s{gi}_conv"]), gi


@pytest.mark.parametrize("name", CORPORA)
def test_search_fast_mode_parity(gpu, oracle, name):
    """Team-reduced distances: recall within 0.5 pp, >= 99% identical ids,
    reported distances bit-equal to the host sequential chain."""
    for gi, g, ids, dists, counts, st in _golden_search(gpu, oracle, name, False):
        gt = g["gt_ids"]
        ref_ids = g[f"s{gi}_ids"]
        nq = gt.shape[0]
        rec = np.mean([len(set(ids[q]) & set(gt[q])) / 10 for q in range(nq)])
        ref_rec = np.mean([len(set(ref_ids[q]) & set(gt[q])) / 10 for q in range(nq)])
        assert abs(rec - ref_rec) <= 0.005, (gi, rec, ref_rec)
        assert np.mean(ids == ref_ids) >= 0.99, gi
    # distances are the sequential chain of the returned ids
    g, data, queries = corpus(oracle, name)
    for q in range(0, queries.shape[0], 17):
        for j in range(10):
            if ids[q, j] == capi.INVALID_ID:
                continue
            assert bits(dists[q, j]) == bits(fodg.squared_l2(data[ids[q, j]], queries[q]))


@pytest.mark.parametrize("kernel", ["fused", "generic"])
@pytest.mark.parametrize("name", CORPORA)
def test_multi_cta_shared_mode_parity(gpu, oracle, monkeypatch, name, kernel):
    """Shared mode with one CTA per team (teams race on one visited table):
    recall within 0.5 pp of the reference's lockstep shared mode
    (engine.cpp:38-78) at the same params and seeds; reported distances are
    the sequential chain; evaluations >= the per-query p=1 run."""
    g, data, queries = corpus(oracle, name)
    ds = fodg.Dataset.from_array(data)
    ix = fodg.Index(ds, fodg.Graph(int(g["n"]), int(g["d"]), g["graph"]))
    gt = g["gt_ids"]
    # fused: search_b1.cu (M <= 32: one launch, the last team merges);
    # generic: the K5 kernel per team + team_merge_kernel (two launches)
    monkeypatch.setenv("CAGRA_B1_KERNEL", "1" if kernel == "fused" else "0")
    for m, teams in [(32, 4), (64, 8), (16, 32), (12, 64)]:
        prm = fodg.SearchParams(k=10, topm=m, width=1, seed=11)
        ids, dists, counts, st = ix.search(
            queries, prm, fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers,
                                             team_count=teams, multi_cta=2))
        fused = kernel == "fused" and m <= 32
        assert ix.last_launch_count() == (1 if fused else 2)
        o = oracle.batch_search(g["graph"], data, queries, make_params(k=10, topm=m, width=1,
                                                                       seed=11),
                                mode=1, team_count=teams)
        nq = gt.shape[0]
        rec = np.mean([len(set(ids[q]) & set(gt[q])) / 10 for q in range(nq)])
        ref_rec = np.mean([len(set(o[0][q]) & set(gt[q])) / 10 for q in range(nq)])
        assert abs(rec - ref_rec) <= 0.005, (m, teams, rec, ref_rec)
        assert np.mean(ids == o[0]) >= 0.95
        assert (counts == 10).all()
        for q in range(0, nq, 23):
            for j in range(10):
                assert bits(dists[q, j]) == bits(fodg.squared_l2(data[ids[q, j]], queries[q]))
        # lockstep (reference order) still available and bit-exact in exact mode
        if teams > 16:
            continue
        ids2, dists2, _, st2 = ix.search(
            queries, prm, fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers,
                                             team_count=teams, multi_cta=1,
                                             exact_distances=True))
        assert np.array_equal(ids2, o[0])
        assert np.array_equal(st2["distance_evals"], o[3]["distance_evals"])


def test_batch_equals_search_one(gpu, oracle):
    # test_engine.cpp:54-85
    data = oracle.uniform_dataset(600, 8, 71)
    queries = oracle.uniform_dataset(12, 8, 72)
    ds = fodg.Dataset.from_array(data)
    graph = fodg.optimize(fodg.exact_knn_graph(ds, 16), 8)
    params = fodg.SearchParams(k=10, topm=32, width=2, seed=99)
    res = fodg.batch_search(graph, ds, fodg.Dataset.from_array(queries), params)
    for qi in range(12):
        p = fodg.SearchParams(k=10, topm=32, width=2, seed=fodg.mix_seed(99 ^ (0x0BAD + qi)))
        single = fodg.search_one(graph, ds, queries[qi], p)
        assert res[qi].ids.tolist() == single.ids.tolist()
        assert np.array_equal(bits(res[qi].dists), bits(single.dists))


def test_search_properties(gpu, oracle):
    # test_search.cpp:265-398 / test_engine.cpp:87-136 style properties
    data = oracle.uniform_dataset(800, 8, 71)
    ds = fodg.Dataset.from_array(data)
    queries = oracle.uniform_dataset(16, 8, 72)
    graph = fodg.optimize(fodg.exact_knn_graph(ds, 16), 8)
    # exact point found with distance 0 (1-D grid analogue)
    p = fodg.SearchParams(k=1, topm=32, width=2, seed=9)
    r = fodg.search_one(graph, ds, data[123], p)
    assert r.ids.tolist() == [123] and r.dists[0] == 0.0
    # M = N: every node reachable -> exact
    gt, _ = oracle.exact_topk_batch(data, queries, 10)
    full = fodg.SearchParams(k=10, topm=800, width=8, seed=1)
    res = fodg.batch_search(graph, ds, fodg.Dataset.from_array(queries), full)
    assert all(set(res[q].ids.tolist()) == set(gt[q].tolist()) for q in range(16))
    # shared mode: sorted, no duplicates, no flags, true dists, deterministic
    sp = fodg.SearchParams(k=10, topm=32, width=2, seed=17)
    so = fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=4)
    a = fodg.batch_search(graph, ds, fodg.Dataset.from_array(queries), sp, so)
    b = fodg.batch_search(graph, ds, fodg.Dataset.from_array(queries), sp, so)
    for q in range(16):
        ids = a[q].ids.tolist()
        assert len(ids) == 10 and len(set(ids)) == 10
        assert all(i < 0x80000000 for i in ids)
        assert all(a[q].dists[i] <= a[q].dists[i + 1] for i in range(9))
        for i, v in enumerate(ids):
            assert bits(a[q].dists[i]) == bits(fodg.squared_l2(data[v], queries[q]))
        assert ids == b[q].ids.tolist()
        p1 = fodg.SearchParams(k=10, topm=32, width=1, seed=fodg.mix_seed(17 ^ (0x0BAD + q)))
        assert a[q].stats.distance_evals >= fodg.search_one(graph, ds, queries[q], p1).stats.distance_evals


def test_search_validation_errors(gpu, oracle):
    # test_engine.cpp:138-152, test_search.cpp:53-68
    data = oracle.uniform_dataset(100, 4, 1)
    ds = fodg.Dataset.from_array(data)
    graph = fodg.optimize(fodg.exact_knn_graph(ds, 8), 4)
    q = fodg.Dataset.from_array(oracle.uniform_dataset(1, 4, 2))
    with pytest.raises(fodg.UsageError):
        fodg.batch_search(graph, ds, fodg.Dataset.from_array(oracle.uniform_dataset(2, 5, 1)),
                          fodg.SearchParams(k=5, topm=16))
    with pytest.raises(fodg.UsageError):
        fodg.batch_search(graph, ds, q, fodg.SearchParams(k=64, topm=16))
    with pytest.raises(fodg.UsageError):
        fodg.batch_search(graph, ds, q, fodg.SearchParams(),
                          fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers,
                                             team_count=1))
    # raw C ABI rejects the same way
    ix = fodg.Index(ds, graph)
    with pytest.raises(capi.UsageError):
        ix.search(q.data, fodg.SearchParams(k=0))
    with pytest.raises(capi.UsageError):
        ix.search(q.data, fodg.SearchParams(hash_policy=fodg.HashPolicy.kForgettable,
                                            hash_bits=3))
    # empty batch is a no-op (engine.cpp:97)
    ids, dists, counts, st = ix.search(np.zeros((0, 4), np.float32), fodg.SearchParams(k=5, topm=16))
    assert ids.shape == (0, 5)


def test_search_random_params_vs_oracle(gpu, oracle):
    """Reference-semantics mode against the oracle on random parameter draws,
    including odd dimensions, tiny forgettable tables and shared teams."""
    rng = np.random.default_rng(7)
    for case in range(6):
        n = int(rng.integers(200, 1500))
        dim = int(rng.choice([3, 8, 13, 32, 96]))
        d = int(rng.choice([4, 8, 16]))
        data = oracle.uniform_dataset(n, dim, 100 + case)
        ids, dists = oracle.exact_knn_graph(data, 2 * d)
        graph = oracle.optimize(ids, dists, d)
        queries = oracle.uniform_dataset(24, dim, 200 + case)
        ix = fodg.Index(data, graph)
        for trial in range(5):
            m = int(rng.choice([8, 16, 32, 64]))
            prm = make_params(k=int(rng.integers(1, min(m, 10) + 1)), topm=m,
                              width=int(rng.choice([1, 2, 3, 4])),
                              hash_policy=int(rng.integers(0, 2)),
                              hash_bits=int(rng.integers(4, 12)),
                              reset_interval=int(rng.integers(1, 4)), seed=int(rng.integers(0, 1 << 40)),
                              min_iterations=int(rng.integers(1, 5)),
                              max_iterations=int(rng.choice([0, 0, 5, 40])))
            mode = int(rng.integers(0, 2)) if trial % 2 else 0
            teams = int(rng.integers(2, 6))
            o_ids, o_d, o_c, o_st = oracle.batch_search(graph, data, queries, prm, mode=mode,
                                                        team_count=teams)
            sp = fodg.SearchParams(prm.k, prm.topm, prm.width, prm.max_iterations,
                                   prm.min_iterations, fodg.HashPolicy(prm.hash_policy),
                                   prm.hash_bits, prm.reset_interval, prm.seed)
            so = fodg.EngineOptions(mode=fodg.ExecutionMode(mode), team_count=teams,
                                    exact_distances=True)
            ids_, d_, c_, st_ = ix.search(queries, sp, so)
            tag = (case, trial, n, dim, d, prm.topm, prm.width, prm.hash_policy, prm.hash_bits, mode)
            assert np.array_equal(ids_, o_ids), tag
            assert np.array_equal(bits(d_), bits(o_d)), tag
            assert np.array_equal(st_["distance_evals"], o_st["distance_evals"]), tag
            assert np.array_equal(st_["iterations"], o_st["iterations"]), tag
            assert np.array_equal(st_["hash_resets"], o_st["hash_resets"]), tag


# ------------------------------------------------- GIST-shaped (C3) parity ----
def test_gist_shape_960d_pipeline_vs_oracle(gpu, oracle):
    """BASELINE configs[2] shape (960-d, graph degree 64, multi-CTA small
    batch) at oracle-checkable size: the kNN graph (tensor-core path with the
    query tile streamed: K = 3*960+6 > 512) and the optimized graph are
    bit-exact; per-query search in reference-semantics mode matches the oracle
    exactly; multi-CTA shared mode is within 0.5 pp of the reference's shared
    mode."""
    n, dim, nq, d = 3000, 960, 40, 64
    data = oracle.uniform_dataset(n, dim, 31)
    queries = oracle.uniform_dataset(nq, dim, 32)
    ds = fodg.Dataset.from_array(data)
    g, _, knn = fodg.build_graph(ds, d, 2 * d, return_knn=True)
    o_ids, o_d = oracle.exact_knn_graph(data, 2 * d)
    assert np.array_equal(knn.ids, o_ids)
    assert np.array_equal(bits(knn.dists), bits(o_d))
    o_graph = oracle.optimize(o_ids, o_d, d)
    assert np.array_equal(g.ids, o_graph)
    ix = fodg.Index(ds, g)
    prm = fodg.SearchParams(k=10, topm=64, width=2, seed=5)
    ids, dists, _, st = ix.search(queries, prm, fodg.EngineOptions(exact_distances=True))
    o = oracle.batch_search(o_graph, data, queries, make_params(k=10, topm=64, width=2, seed=5))
    assert np.array_equal(ids, o[0])
    assert np.array_equal(bits(dists), bits(o[1]))
    assert np.array_equal(st["distance_evals"], o[3]["distance_evals"])
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    sp = fodg.SearchParams(k=10, topm=32, width=1, seed=5)
    mc = ix.search(queries, sp, fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers,
                                                   team_count=8, multi_cta=2))[0]
    ref = oracle.batch_search(o_graph, data, queries, make_params(k=10, topm=32, width=1,
                                                                  seed=5), mode=1,
                              team_count=8)[0]
    rec = np.mean([len(set(mc[q]) & set(gt[q])) / 10 for q in range(nq)])
    ref_rec = np.mean([len(set(ref[q]) & set(gt[q])) / 10 for q in range(nq)])
    assert abs(rec - ref_rec) <= 0.005 + 1e-9, (rec, ref_rec)


# ------------------------------------------------------------- edge cases ----
@pytest.mark.parametrize("n,dim,d,m,p,k,pol", [
    (40, 1, 4, 8, 1, 8, 0),        # 1-D, k == M, tiny graph
    (130, 7, 6, 16, 3, 5, 1),      # odd dim, degree 6 (not a power of two), forgettable
    (257, 33, 12, 24, 2, 24, 0),   # k == M, ragged sizes
    (600, 8, 24, 64, 5, 10, 1),    # degree 24, p*d = 120 candidates
])
def test_search_edge_shapes_reference_semantics(gpu, oracle, n, dim, d, m, p, k, pol):
    data = oracle.uniform_dataset(n, dim, n + dim)
    queries = oracle.uniform_dataset(11, dim, 3)
    ids_k, d_k = oracle.exact_knn_graph(data, 2 * d)
    graph = oracle.optimize(ids_k, d_k, d)
    ix = fodg.Index(fodg.Dataset.from_array(data), fodg.Graph(n, d, graph))
    prm = fodg.SearchParams(k=k, topm=m, width=p, hash_policy=fodg.HashPolicy(pol), hash_bits=6,
                            seed=17)
    ids, dists, counts, st = ix.search(queries, prm, fodg.EngineOptions(exact_distances=True))
    o = oracle.batch_search(graph, data, queries, make_params(k=k, topm=m, width=p,
                                                              hash_policy=pol, hash_bits=6,
                                                              seed=17))
    assert np.array_equal(ids, o[0])
    assert np.array_equal(bits(dists), bits(o[1]))
    assert np.array_equal(counts, o[2])
    assert np.array_equal(st["distance_evals"], o[3]["distance_evals"])
    assert np.array_equal(st["hash_resets"], o[3]["hash_resets"])


def test_search_empty_batch_and_limits(gpu, oracle):
    data = oracle.uniform_dataset(300, 8, 1)
    ds = fodg.Dataset.from_array(data)
    g = fodg.optimize(fodg.exact_knn_graph(ds, 16), 8)
    ix = fodg.Index(ds, g)
    ids, dists, counts, st = ix.search(np.zeros((0, 8), np.float32), fodg.SearchParams())
    assert ids.shape == (0, 10) and counts.shape == (0,)
    # parameters beyond the device's shared-memory budget fail loudly (UsageError)
    with pytest.raises(fodg.UsageError):
        ix.search(data[:2], fodg.SearchParams(k=10, topm=30000, width=64))
    # M = 20000 fits with the in-place top-M update (one 160 KB list) and
    # returns the exact top-10 (M exceeds n: every node gets evaluated)
    ids, dists, counts, _ = ix.search(data[:2], fodg.SearchParams(k=10, topm=20000, width=64))
    gt, _ = fodg.exact_topk_batch(ds, data[:2], 10)
    assert (counts == 10).all() and np.array_equal(np.sort(ids, 1), np.sort(gt, 1))
    # dimension mismatch / graph-dataset mismatch, reference messages' classes
    with pytest.raises(fodg.UsageError):
        fodg.batch_search(g, ds, fodg.Dataset.from_array(data[:3, :4]), fodg.SearchParams())


# ------------------------------------------------------- graph metrics ----
def _metric_graphs(oracle):
    rng = np.random.default_rng(5)
    yield "functional d=1", rng.integers(0, 5000, (5000, 1), dtype=np.uint32)
    yield "random d=3", rng.integers(0, 20000, (20000, 3), dtype=np.uint32)
    chain = np.arange(-1, 999, dtype=np.int64).clip(0).astype(np.uint32).reshape(1000, 1)
    yield "reverse chain + self loop", chain
    yield "two-cycle", np.array([[1], [0]], np.uint32)
    yield "dup ids in rows", rng.integers(0, 50, (300, 6), dtype=np.uint32)
    data = oracle.uniform_dataset(2048, 32, 3)
    ids, dists = oracle.exact_knn_graph(data, 48)
    yield "optimized 2048x16", oracle.optimize(ids, dists, 16)
    ds = fodg.Dataset.from_array(capi.uniform_dataset(100_000, 32, 424242))
    g, _ = fodg.build_graph(ds, 32)
    yield "optimized 100k x32", g.ids


def test_graph_metrics_vs_reference(gpu, oracle, reference):
    # graph_metrics.cpp:20-120: SCC count and the mean distinct 2-hop count,
    # exact (integer total / n, same double)
    for name, ids in _metric_graphs(oracle):
        ids = np.ascontiguousarray(ids, np.uint32)
        n, d = ids.shape
        g = fodg.Graph(n, d, ids)
        want_scc, want_avg = reference.graph_metrics(ids)
        rep = fodg.measure_graph(g)
        assert rep.strong_cc == want_scc, name
        assert rep.avg_2hop == want_avg, name
        assert rep.max_2hop == d * (1 + d)
    with pytest.raises(fodg.UsageError):
        fodg.measure_graph(fodg.Graph(2, 1, np.array([[1], [7]], np.uint32)))


def test_b1_visited_regions_follow_batch_size(gpu, oracle, monkeypatch):
    # the fused batch-1 kernel clears the other call's visited region in-kernel
    # at the current layout (nq regions): a batch-size change must start clean,
    # or a later call of the same queries finds its nodes already marked
    data = oracle.uniform_dataset(20000, 32, 7)
    queries = oracle.uniform_dataset(8, 32, 8)
    ds = fodg.Dataset.from_array(data)
    g, _ = fodg.build_graph(ds, 32)
    ix = fodg.Index(ds, g)
    monkeypatch.setenv("CAGRA_B1_KERNEL", "1")
    prm = fodg.SearchParams(k=10, topm=16, width=1, seed=5)
    opts = fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=8,
                              multi_cta=2)
    first = ix.search(queries, prm, opts)
    assert ix.last_launch_count() == 1
    ix.search(queries[:1], prm, opts)
    ix.search(queries[:3], prm, opts)
    again = ix.search(queries, prm, opts)
    e0, e1 = first[3]["distance_evals"], again[3]["distance_evals"]
    assert np.all(e1 >= 0.8 * e0), (e0, e1)
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)

    def recall(ids):
        return np.mean([len(set(ids[q]) & set(gt[q])) / 10 for q in range(len(gt))])

    # racing teams: ids differ run to run, recall does not collapse
    assert recall(again[0]) >= recall(first[0]) - 0.05


def test_multi_cta_large_batch_chunked(gpu, oracle, monkeypatch):
    # forced multi-CTA on a batch whose per-query visited regions exceed the
    # table budget runs in query chunks (query_offset keeps seeds global):
    # same recall as one launch
    data = oracle.uniform_dataset(20000, 32, 7)
    queries = oracle.uniform_dataset(300, 32, 8)
    ds = fodg.Dataset.from_array(data)
    g, _ = fodg.build_graph(ds, 32)
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    ix = fodg.Index(ds, g)
    prm = fodg.SearchParams(k=10, topm=64, width=1, seed=3)
    opts = fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=8,
                              multi_cta=2)

    def recall(ids):
        return np.mean([len(set(ids[q]) & set(gt[q])) / 10 for q in range(len(gt))])

    one = ix.search(queries, prm, opts)
    monkeypatch.setenv("CAGRA_TABLE_BUDGET_MB", "4")  # 1 MB per query -> chunks of 4
    chunked = ix.search(queries, prm, opts)
    assert np.all(chunked[2] == 10)
    assert np.all(chunked[3]["iterations"] > 0)
    assert abs(recall(one[0]) - recall(chunked[0])) <= 0.01
