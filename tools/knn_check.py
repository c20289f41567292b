"""GPU check of the tensor-core kNN path against the SIMT sequential-chain
path (and the C oracle on small cases): ids + dist bits, timings, counters."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402


def run(path, fn):
    os.environ["CAGRA_KNN_PATH"] = path
    t = time.time()
    r = fn()
    return r, time.time() - t, capi.knn_last_stats()


def cmp(name, a, b):
    ia, da = a
    ib, db = b
    same_ids = np.mean(ia == ib)
    same_d = np.mean(da.view(np.uint32) == db.view(np.uint32))
    rows = np.mean(np.all(ia == ib, axis=1))
    print(f"  {name}: id-match {same_ids:.6f} dist-bits {same_d:.6f} rows-identical {rows:.6f}",
          flush=True)
    return rows


def main():
    big = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    cases = [(1000, 37, 40), (333, 5, 7), (5000, 96, 128), (20000, 96, 128), (20000, 128, 64),
             (4096, 64, 64)]
    for n, dim, k in cases:
        data = capi.uniform_dataset(n, dim, 7 + n)
        ds = fodg.Dataset.from_array(data)
        f = lambda: (lambda g: (g.ids, g.dists))(fodg.exact_knn_graph(ds, k))
        tc, ttc, st = run("auto", f)
        si, tsi, _ = run("simt", f)
        print(f"knn n={n} dim={dim} k={k}: tc {ttc:.3f}s simt {tsi:.3f}s stats {st}", flush=True)
        cmp("tc vs simt", tc, si)
        q = capi.uniform_dataset(100, dim, 99)
        g = lambda: fodg.exact_topk_batch(ds, q, 10)
        tc, _, st = run("auto", g)
        si, _, _ = run("simt", g)
        cmp(f"gt k=10 {st}", tc, si)
    if big:
        data = capi.uniform_dataset(big, 96, 424242)
        ds = fodg.Dataset.from_array(data)
        f = lambda: (lambda g: (g.ids, g.dists))(fodg.exact_knn_graph(ds, 128))
        tc, ttc, st = run("auto", f)
        print(f"knn n={big} dim=96 k=128: tc wall {ttc:.2f}s stats {st}", flush=True)
        si, tsi, _ = run("simt", f)
        print(f"  simt wall {tsi:.2f}s", flush=True)
        cmp("tc vs simt", tc, si)
        gg, info = fodg.build_graph(ds, 64)
        print(f"  build_graph {info}", flush=True)


if __name__ == "__main__":
    main()
