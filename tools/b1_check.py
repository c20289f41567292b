"""Batch-1 quick check: sequential single-query cagra_search calls (pinned host
buffers) with the fused team kernel vs the generic multi-CTA kernel, recall
and latency at a few (M, teams) points; device time per call via the index's
launch count is not needed — wall per call is what a caller sees.

  python tools/b1_check.py [n] [queries] [M,T;M,T...]
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 500
grid = [tuple(int(x) for x in t.split(",")) for t in
        (sys.argv[3] if len(sys.argv) > 3 else "16,64;12,96;16,32;32,32;24,48").split(";")]
dim = 96
data = capi.uniform_dataset(n, dim, 424242)
queries = capi.uniform_dataset(10000, dim, 424243)[:nq]
ds = fodg.Dataset.from_array(data)
g, _ = fodg.build_graph(ds, 64)
gt, _ = fodg.exact_topk_batch(ds, queries, 10)
ix = fodg.Index(ds, g)
hq = torch.from_numpy(queries).pin_memory()
oi = torch.empty((1, 10), dtype=torch.int32).pin_memory()
od = torch.empty((1, 10), dtype=torch.float32).pin_memory()
L = capi.lib()
for kern in ("1", "0"):
    os.environ["CAGRA_B1_KERNEL"] = kern
    for (m, t) in grid:
        prm = fodg.SearchParams(k=10, topm=m, width=1, seed=11)
        opt = fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=t)
        pc, oc = prm.c(), opt.c()
        out = np.empty((nq, 10), np.uint32)
        for i in range(3):
            L.cagra_search(ix.h, capi.ptr(hq[i]), 1, dim, C.byref(pc), C.byref(oc),
                           capi.ptr(oi), capi.ptr(od), None, None)
        t0 = time.perf_counter()
        for i in range(nq):
            capi.check(L.cagra_search(ix.h, capi.ptr(hq[i]), 1, dim, C.byref(pc), C.byref(oc),
                                      capi.ptr(oi), capi.ptr(od), None, None))
            out[i] = oi.numpy().view(np.uint32)[0]
        el = time.perf_counter() - t0
        rec = np.mean([len(set(out[i]) & set(gt[i])) / 10 for i in range(nq)])
        print(f"b1_kernel={kern} M={m} teams={t}: recall={rec:.4f} qps={nq / el:.0f} "
              f"lat_us={el / nq * 1e6:.1f} launches={ix.last_launch_count()}", flush=True)
