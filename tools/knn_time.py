"""Time the device graph build (exact kNN + optimize) at one size, 3 builds,
under whatever CAGRA_* knobs the environment sets; prints a digest of the kNN
graph so runs under different knobs can be compared for bit-equality.

  CAGRA_KNN_SPLIT=3 python tools/knn_time.py [n] [dim] [k]
"""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 128
knobs = {kk: v for kk, v in os.environ.items() if kk.startswith("CAGRA_")}
data = capi.uniform_dataset(n, dim, 424242)
ds = fodg.Dataset.from_array(data)
for rep in range(3):
    t = time.time()
    g, info, knn = fodg.build_graph(ds, k // 2, k, return_knn=True)
    wall = time.time() - t
    st = capi.knn_last_stats()
    h = hashlib.sha256(knn.ids.tobytes() + knn.dists.tobytes()).hexdigest()[:16]
    print(f"{knobs} n={n} dim={dim} k={k} wall {wall:.3f}s knn {info['knn_seconds']:.3f}s "
          f"opt {info['optimize_seconds']:.3f}s rerank/row {st['reranked'] / max(1, st['rows']):.1f} "
          f"retried {st['retried_rows']} fallback {st['fallback_rows']} digest {h}", flush=True)
