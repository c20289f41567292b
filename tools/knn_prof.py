"""Time the kNN build kernels at one size (for ncu / quick timing).
With CAGRA_TC_DEBUG set only exact_knn_graph runs (debug epilogues produce
garbage graphs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 128
data = capi.uniform_dataset(n, dim, 424242)
ds = fodg.Dataset.from_array(data)
for rep in range(2):
    t = time.time()
    if os.environ.get("CAGRA_TC_DEBUG"):
        fodg.exact_knn_graph(ds, k)
        info = {}
    else:
        g, info = fodg.build_graph(ds, k // 2, k)
    print(f"n={n} dim={dim} k={k} wall {time.time() - t:.3f}s {info} {capi.knn_last_stats()}",
          flush=True)
