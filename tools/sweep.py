"""Operating-point sweep on the GPU box: build an N x D synthetic index on
device, exact ground truth, then recall / QPS / evals over a (M, p, policy)
grid.  Prints one line per setting.  Exploration tool, not the bench.

  python tools/sweep.py --n 1000000 --dim 96 --nq 10000
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15136_b200 import capi, fodg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--grid", default="")
    ap.add_argument("--data", default="uniform", choices=["uniform", "lowrank"])
    ap.add_argument("--rank", type=int, default=32)
    args = ap.parse_args()
    t = time.time()
    if args.data == "lowrank":
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from bench import lowrank_dataset
        data = lowrank_dataset(args.n, args.dim, args.rank, 424242)
        queries = lowrank_dataset(args.nq, args.dim, args.rank, 424243)
    else:
        data = capi.uniform_dataset(args.n, args.dim, 424242)
        queries = capi.uniform_dataset(args.nq, args.dim, 424243)
    print(f"gen {time.time()-t:.1f}s", flush=True)
    ds = fodg.Dataset.from_array(data)
    t = time.time()
    g, info = fodg.build_graph(ds, args.d)
    print(f"build wall {time.time()-t:.1f}s {info}", flush=True)
    t = time.time()
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    print(f"gt wall {time.time()-t:.1f}s", flush=True)
    ix = fodg.Index(ds, g)
    dev = torch.device("cuda:0")
    qd = torch.zeros((args.nq, ix.ld), dtype=torch.float32, device=dev)
    qd[:, :args.dim] = torch.from_numpy(queries).to(dev)
    ids = torch.empty((args.nq, 10), dtype=torch.int32, device=dev)
    dists = torch.empty((args.nq, 10), dtype=torch.float32, device=dev)
    stats = torch.empty((args.nq, 6), dtype=torch.int32, device=dev)
    ts_stream = torch.cuda.Stream()
    torch.cuda.set_stream(ts_stream)
    stream = ts_stream.cuda_stream
    grid = []
    if args.grid:
        for tok in args.grid.split(";"):
            # M,p,policy,bits,team_size,reset_interval[,mode,teams,multi_cta]
            defaults = [0, 0, 0, 0, 0, 1, 0, 4, 0]
            vals = [int(x) for x in tok.split(",")]
            grid.append(tuple(vals + defaults[len(vals):]))
    else:
        for m, p in [(512, 8), (768, 16), (896, 16), (1024, 16), (1024, 32)]:
            for pol in (0, 1):
                for ts in (4, 8, 16):
                    grid.append((m, p, pol, 0, ts, 1, 0, 4, 0))
    for (m, p, pol, bits, ts, ri, mode, teams, mc) in grid:
        if not bits:
            need = m + p * args.d
            bits = max(10, int(np.ceil(np.log2(need * 1.6))))
        prm = fodg.SearchParams(k=10, topm=m, width=p, hash_policy=fodg.HashPolicy(pol),
                                hash_bits=bits, seed=11, reset_interval=ri)
        opt = fodg.EngineOptions(team_size=ts, mode=fodg.ExecutionMode(mode), team_count=teams,
                                 multi_cta=mc)
        try:
            ix.search_dev(qd, args.nq, prm, opt, ids, dists, None, stats, stream)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                ix.search_dev(qd, args.nq, prm, opt, ids, dists, None, stats, stream)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
        except Exception as ex:  # noqa: BLE001
            print(f"M={m} p={p} pol={pol} bits={bits}: {ex}", flush=True)
            continue
        hid = ids.cpu().numpy().astype(np.uint32)
        st = stats.cpu().numpy()
        evals = st[:, 2].astype(np.int64) + (st[:, 3].astype(np.int64) << 32)
        iters = st[:, 0]
        rec = np.mean([len(set(hid[i]) & set(gt[i])) / 10 for i in range(args.nq)])
        bytes_q = evals.mean() * args.dim * 4 + iters.mean() * p * args.d * 4
        gbs = bytes_q * args.nq / (ms * 1e-3) / 1e9
        print(f"M={m:5d} p={p:3d} pol={pol} bits={bits:2d} ts={ts} ri={ri} mode={mode} "
              f"teams={teams} mc={mc} recall={rec:.4f} "
              f"qps={args.nq / (ms * 1e-3):10.0f} ms={ms:8.2f} evals={evals.mean():8.0f} "
              f"iters={iters.mean():6.1f} alg_GBs={gbs:7.0f}", flush=True)


if __name__ == "__main__":
    main()
