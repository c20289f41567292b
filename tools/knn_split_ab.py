"""A/B of the K1 filter splits (fp16 single term vs bf16x3) at one size:
build seconds of each and bit-equality of the two kNN graphs (both must equal
the reference; tests/test_gpu_parity.py pins each against the SIMT chain).

  python tools/knn_split_ab.py [n] [dim] [k]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 128
data = capi.uniform_dataset(n, dim, 424242)
ds = fodg.Dataset.from_array(data)
res = {}
for split in ("1", "3", "1"):
    os.environ["CAGRA_KNN_SPLIT"] = split
    t = time.time()
    g, info, knn = fodg.build_graph(ds, k // 2, k, return_knn=True)
    wall = time.time() - t
    st = capi.knn_last_stats()
    print(f"split={split} n={n} dim={dim} k={k} wall {wall:.3f}s knn {info['knn_seconds']:.3f}s "
          f"opt {info['optimize_seconds']:.3f}s reranked/row {st['reranked'] / max(1, st['rows']):.1f} "
          f"retried {st['retried_rows']} fallback {st['fallback_rows']}", flush=True)
    res[split] = (knn.ids.copy(), knn.dists.view(np.uint32).copy(), g.ids.copy())
a, b = res["1"], res["3"]
print("ids equal", np.array_equal(a[0], b[0]), "dist bits equal", np.array_equal(a[1], b[1]),
      "graph equal", np.array_equal(a[2], b[2]), flush=True)
