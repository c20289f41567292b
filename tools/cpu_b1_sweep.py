"""Batch-1 operating point of the REFERENCE on the host:
sequential single-query fodg_ref::batch_search calls, single-threaded, in
per-query mode and in shared mode (choose_mode's pick for batch 1), over a
grid; prints recall@10 and QPS per point.  The graph is the device-built one
(bit-identical to the reference's optimize of the same exact kNN graph).

  python tools/cpu_b1_sweep.py [n] [queries]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.bindings import load_reference, make_params  # noqa: E402
from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dim = 96
data = capi.uniform_dataset(n, dim, 424242)
queries = capi.uniform_dataset(nq, dim, 424243)
ds = fodg.Dataset.from_array(data)
g, _ = fodg.build_graph(ds, 64)
gt, _ = fodg.exact_topk_batch(ds, queries, 10)
ref = load_reference()
rix = ref.index(data, g.ids)


def rec(ids):
    return np.mean([len(set(ids[i]) & set(gt[i])) / 10 for i in range(nq)])


def run(label, p, mode, teams=4):
    out = np.empty((nq, 10), np.uint32)
    t0 = time.perf_counter()
    for i in range(nq):
        ids, _, _, _ = rix.batch_search(queries[i:i + 1], p, mode=mode, team_count=teams, threads=1)
        out[i] = ids[0]
    el = time.perf_counter() - t0
    print(f"{label:40s} recall {rec(out):.4f}  qps {nq / el:8.1f}  ms/q {el / nq * 1e3:7.2f}",
          flush=True)


for m, p in [(256, 4), (384, 4), (512, 8), (640, 8), (896, 16), (1024, 16)]:
    run(f"per_query M={m} p={p}", make_params(k=10, topm=m, width=p, seed=11), 0)
for m, t in [(64, 4), (128, 4), (192, 4), (256, 4), (128, 8), (64, 16), (16, 64)]:
    run(f"shared x{t} M={m}", make_params(k=10, topm=m, width=1, seed=11), 1, t)
