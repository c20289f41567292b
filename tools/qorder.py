"""Experiment: does the order in which a batch's queries are handed to the
resident CTAs change the search kernel's L2 reuse (and QPS)?  Builds the C2
index, then times the same batch in several permutations.  Exploration tool.

  python tools/qorder.py [--n 1000000] [--nq 10000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402


def kmeans_order(q, c, iters=10, seed=0):
    rng = np.random.default_rng(seed)
    cent = q[rng.choice(len(q), c, replace=False)].copy()
    for _ in range(iters):
        d = (q * q).sum(1)[:, None] - 2 * q @ cent.T + (cent * cent).sum(1)[None]
        a = d.argmin(1)
        for j in range(c):
            m = a == j
            if m.any():
                cent[j] = q[m].mean(0)
    # order clusters along a greedy nearest-centroid path so neighbours in the
    # schedule are also close
    left = set(range(1, c))
    path = [0]
    while left:
        cur = cent[path[-1]]
        nxt = min(left, key=lambda j: float(((cent[j] - cur) ** 2).sum()))
        path.append(nxt)
        left.remove(nxt)
    rank = np.empty(c, np.int64)
    rank[path] = np.arange(c)
    return np.argsort(rank[a], kind="stable")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    data = capi.uniform_dataset(args.n, args.dim, 424242)
    queries = capi.uniform_dataset(args.nq, args.dim, 424243)
    ds = fodg.Dataset.from_array(data)
    g, _ = fodg.build_graph(ds, 64)
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    ix = fodg.Index(ds, g)
    dev = torch.device("cuda:0")
    prm = fodg.SearchParams(k=10, topm=896, width=16, hash_policy=fodg.HashPolicy(1),
                            hash_bits=12, seed=11)
    opt = fodg.EngineOptions(team_size=8)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    orders = {"natural": np.arange(args.nq), "random": np.random.default_rng(1).permutation(args.nq)}
    for c in (16, 64, 256, 1024):
        t = time.time()
        orders[f"kmeans{c}"] = kmeans_order(queries, c)
        print(f"kmeans{c} {time.time() - t:.1f}s", flush=True)
    # 1-NN id of the query (ids are in generation order: no locality) and a
    # projection on the top principal direction
    orders["gt_nn_id"] = np.argsort(gt[:, 0], kind="stable")
    u = np.linalg.svd(queries - queries.mean(0), full_matrices=False)[2][0]
    orders["pc1"] = np.argsort(queries @ u, kind="stable")
    for name, perm in orders.items():
        qp = queries[perm]
        qd = torch.zeros((args.nq, ix.ld), dtype=torch.float32, device=dev)
        qd[:, :args.dim] = torch.from_numpy(np.ascontiguousarray(qp)).to(dev)
        ids = torch.empty((args.nq, 10), dtype=torch.int32, device=dev)
        dists = torch.empty((args.nq, 10), dtype=torch.float32, device=dev)
        stats = torch.empty((args.nq, 6), dtype=torch.int32, device=dev)
        ix.search_dev(qd, args.nq, prm, opt, ids, dists, None, stats, st.cuda_stream)
        torch.cuda.synchronize()
        ms = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ix.search_dev(qd, args.nq, prm, opt, ids, dists, None, stats, st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        got = ids.cpu().numpy().view(np.uint32)
        rec = np.mean([len(set(got[i]) & set(gt[perm[i]])) / 10 for i in range(args.nq)])
        print(f"{name:10s} ms {np.median(ms):7.2f} qps {args.nq / np.median(ms) * 1e3:9.0f} "
              f"recall {rec:.4f}", flush=True)


if __name__ == "__main__":
    main()
