"""Device NN-descent at one size: seconds, rounds, graph recall vs the exact
kNN graph (sampled rows), and batch search recall / QPS on the optimized
graph built from it vs from the exact graph.

  python tools/nnd_eval.py [n] [dim] [k]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 128
data = capi.uniform_dataset(n, dim, 424242)
queries = capi.uniform_dataset(10000, dim, 424243)
ds = fodg.Dataset.from_array(data)
for rate in (0.5, 1.0):
    t = time.time()
    nd = fodg.nn_descent(ds, k, fodg.NNDescentParams(seed=1, sample_rate=rate))
    print(f"nn_descent n={n} k={k} rate={rate}: {time.time() - t:.2f}s rounds={nd.rounds} "
          f"converged={nd.converged}", flush=True)
t = time.time()
ex = fodg.exact_knn_graph(ds, k)
print(f"exact kNN {time.time() - t:.2f}s", flush=True)
rows = np.random.default_rng(0).choice(n, 20000, replace=False)
rec = np.mean([len(set(nd.ids[r].tolist()) & set(ex.ids[r].tolist())) / k for r in rows])
print(f"graph recall (20k sampled rows) {rec:.4f}", flush=True)
gt, _ = fodg.exact_topk_batch(ds, queries, 10)
for name, knn in (("nn_descent", nd), ("exact", ex)):
    g = fodg.optimize(knn, k // 2)
    ix = fodg.Index(ds, g)
    for m, p in ((896, 16), (1024, 16)):
        prm = fodg.SearchParams(k=10, topm=m, width=p, hash_policy=fodg.HashPolicy.kForgettable,
                                hash_bits=12, seed=11)
        ix.search(queries[:100], prm)
        t = time.time()
        ids = ix.search(queries, prm)[0]
        el = time.time() - t
        r = np.mean([len(set(ids[i]) & set(gt[i])) / 10 for i in range(len(queries))])
        print(f"{name} graph: M={m} p={p} recall {r:.4f} qps {len(queries) / el:.0f}", flush=True)
