"""Time exact_topk_batch (ground truth, K1 in list mode) at one size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 96
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000
data = capi.uniform_dataset(n, dim, 424242)
q = capi.uniform_dataset(nq, dim, 424243)
ds = fodg.Dataset.from_array(data)
for rep in range(3):
    t = time.time()
    ids, d = fodg.exact_topk_batch(ds, q, 10)
    print(f"gt n={n} dim={dim} nq={nq} {time.time() - t:.3f}s {capi.knn_last_stats()} "
          f"checksum {int(ids.astype(np.int64).sum())}", flush=True)
