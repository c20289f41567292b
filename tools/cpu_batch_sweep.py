"""Batch-10k operating point of the REFERENCE on the host:
fodg_ref::batch_search over a query sample with all host threads, over an
(M, p, hash policy, mode) grid; prints recall@10 and QPS per point.

  python tools/cpu_batch_sweep.py [n] [queries]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.bindings import load_reference, make_params  # noqa: E402
from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
dim = 96
data = capi.uniform_dataset(n, dim, 424242)
queries = capi.uniform_dataset(nq, dim, 424243)
ds = fodg.Dataset.from_array(data)
g, _ = fodg.build_graph(ds, 64)
gt, _ = fodg.exact_topk_batch(ds, queries, 10)
ref = load_reference()
rix = ref.index(data, g.ids)
th = ref.hardware_threads()
print(f"host threads {th}", flush=True)


def rec(ids):
    return np.mean([len(set(ids[i]) & set(gt[i])) / 10 for i in range(nq)])


def run(label, p, mode=0, teams=4):
    rix.batch_search(queries[:th], p, mode=mode, team_count=teams, threads=th)
    t0 = time.perf_counter()
    ids, _, _, st = rix.batch_search(queries, p, mode=mode, team_count=teams, threads=th)
    el = time.perf_counter() - t0
    print(f"{label:44s} recall {rec(ids):.4f}  qps {nq / el:8.1f}  evals {st['distance_evals'].mean():9.0f}",
          flush=True)


for hp, hb in [(0, 11), (1, 12)]:
    for m, p in [(768, 16), (896, 16), (1024, 16), (896, 32), (1024, 32), (640, 8), (768, 8)]:
        run(f"per_query M={m} p={p} hash={'std' if hp == 0 else 'forget'}",
            make_params(k=10, topm=m, width=p, hash_policy=hp, hash_bits=hb, seed=11))
for m, t in [(256, 4), (128, 8)]:
    run(f"shared x{t} M={m}", make_params(k=10, topm=m, width=1, seed=11), 1, t)
