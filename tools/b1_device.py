"""Batch-1 device time: search_dev with nq = 1 on a private stream, CUDA events
around each call, plus the C-ABI (host buffers) wall time per call."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402

n = int(os.environ.get("B1_N", "1000000"))
nq = 200
m, t = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,64").split(","))
dim = 96
data = capi.uniform_dataset(n, dim, 424242)
queries = capi.uniform_dataset(nq, dim, 424243)
ds = fodg.Dataset.from_array(data)
g, _ = fodg.build_graph(ds, 64)
ix = fodg.Index(ds, g)
prm = fodg.SearchParams(k=10, topm=m, width=1, seed=11)
opt = fodg.EngineOptions(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=t)
st = torch.cuda.Stream()
qd = torch.zeros((nq, ix.ld), dtype=torch.float32, device="cuda")
qd[:, :dim] = torch.from_numpy(queries).cuda()
ids = torch.empty((1, 10), dtype=torch.int32, device="cuda")
ds_ = torch.empty((1, 10), dtype=torch.float32, device="cuda")
stats = torch.empty((1, 6), dtype=torch.int32, device="cuda")
ms, its = [], []
for i in range(nq):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ix.search_dev(qd[i:i + 1], 1, prm, opt, ids, ds_, None, stats, st.cuda_stream, query_offset=i)
    e1.record(st)
    st.synchronize()
    ms.append(e0.elapsed_time(e1))
    its.append(int(stats[0, 0]))
ms = np.array(ms[5:]) * 1e3
print(f"M={m} T={t}: device us/query median {np.median(ms):.1f} p10 {np.percentile(ms, 10):.1f} "
      f"p90 {np.percentile(ms, 90):.1f}; iterations mean {np.mean(its):.1f}; "
      f"us/iteration {np.median(ms) / np.mean(its):.2f}", flush=True)
hq = torch.from_numpy(queries).pin_memory()
oi = torch.empty((1, 10), dtype=torch.int32).pin_memory()
od = torch.empty((1, 10), dtype=torch.float32).pin_memory()
pc, oc = prm.c(), opt.c()
L = capi.lib()
t0 = time.perf_counter()
for i in range(nq):
    capi.check(L.cagra_search(ix.h, capi.ptr(hq[i]), 1, dim, C.byref(pc), C.byref(oc),
                              capi.ptr(oi), capi.ptr(od), None, None))
print(f"C-ABI host-buffer wall us/query {(time.perf_counter() - t0) / nq * 1e6:.1f}", flush=True)
