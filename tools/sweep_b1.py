"""Batch-1 operating-point sweep: sequential single-query cagra_search calls
(pinned host buffers, as a user would call it) over a shared-mode grid."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402


def main():
    n, dim, nq = int(sys.argv[1]), 96, int(sys.argv[2])
    grid = [tuple(int(x) for x in t.split(",")) for t in sys.argv[3].split(";")]
    data = capi.uniform_dataset(n, dim, 424242)
    queries = capi.uniform_dataset(10000, dim, 424243)[:nq]
    ds = fodg.Dataset.from_array(data)
    g, info = fodg.build_graph(ds, 64)
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    ix = fodg.Index(ds, g)
    hq = torch.from_numpy(queries).pin_memory()
    oi = torch.empty((1, 10), dtype=torch.int32).pin_memory()
    od = torch.empty((1, 10), dtype=torch.float32).pin_memory()
    L = capi.lib()
    for (mode, m, p, teams, mc) in grid:
        prm = fodg.SearchParams(k=10, topm=m, width=p, seed=11)
        opt = fodg.EngineOptions(mode=fodg.ExecutionMode(mode), team_count=teams, multi_cta=mc)
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
        print(f"mode={mode} M={m} p={p} teams={teams} mc={mc}: recall={rec:.4f} "
              f"qps={nq / el:.0f} lat_us={el / nq * 1e6:.0f}", flush=True)


if __name__ == "__main__":
    main()
