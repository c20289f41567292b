"""Small end-to-end run of every kernel family, for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402

data = capi.uniform_dataset(1500, 20, 1)
q = capi.uniform_dataset(9, 20, 2)
ds = fodg.Dataset.from_array(data)
g, info, knn = fodg.build_graph(ds, 12, 24, return_knn=True)           # TC kNN + optimize
fodg.exact_topk_batch(ds, q, 5)                                         # TC ground truth
os.environ["CAGRA_KNN_PATH"] = "simt"
fodg.exact_knn_graph(ds, 8)                                             # SIMT kNN
os.environ["CAGRA_KNN_PATH"] = "auto"
fodg.count_detourable_routes(knn, fodg.ReorderMode.kRank)
ix = fodg.Index(ds, g)
for pol in (0, 1):
    for exact in (False, True):
        ix.search(q, fodg.SearchParams(k=5, topm=32, width=2, hash_policy=fodg.HashPolicy(pol),
                                       hash_bits=8, seed=3),
                  fodg.EngineOptions(exact_distances=exact))
for mc in (1, 2):
    ix.search(q, fodg.SearchParams(k=5, topm=16, width=1, seed=3),
              fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=4,
                                 multi_cta=mc))
ds2 = fodg.Dataset.from_array(capi.uniform_dataset(700, 200, 4))   # K > 512: streamed query tile
fodg.exact_knn_graph(ds2, 16)
fodg.measure_graph(g)                                                   # graph metrics (SCC + 2-hop)
print("sanitize run ok")
