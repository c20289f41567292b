"""Generate tests/golden/*.npz by running the UNMODIFIED reference
(oracle/_ref/libfodg_ref.so, compiled from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/) and the GPU engine to the
reference's own outputs on seeded inputs (the reference ships no golden files;
its tests generate everything from seeds, proj/tests/test_util.hpp:11-18).
Inputs are regenerated from their seeds at test time, so only outputs are
stored.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bindings import load_oracle, load_reference, make_params  # noqa: E402

# (name, n, dim, d_init, d, data_seed, query_seed, nq)
CORPORA = [
    ("small", 2000, 16, 32, 16, 71, 72, 200),
    ("accept", 3000, 64, 64, 32, 424242, 424243, 100),  # acceptance-corpus shape, smaller N
]

# search grid: (mode, M, p, policy, hash_bits, reset_interval, team_count, seed)
GRID = [
    (0, 32, 1, 0, 11, 1, 4, 11),
    (0, 64, 2, 0, 11, 1, 4, 11),
    (0, 64, 4, 0, 11, 1, 4, 99),
    (0, 128, 4, 0, 11, 1, 4, 11),
    (0, 64, 2, 1, 8, 1, 4, 19),
    (0, 64, 2, 1, 6, 3, 4, 19),   # small table: forces mid-expansion "Full" resets
    (0, 32, 1, 1, 4, 1, 4, 5),    # 16-entry table
    (1, 64, 1, 0, 11, 1, 4, 17),
    (1, 32, 1, 0, 11, 1, 3, 17),
]


def main():
    ref = load_reference()
    if ref is None:
        sys.exit("oracle/_ref/libfodg_ref.so missing: run `make -C oracle` first")
    orc = load_oracle()
    for name, n, dim, d_init, d, ds_seed, q_seed, nq in CORPORA:
        data = orc.uniform_dataset(n, dim, ds_seed)
        queries = orc.uniform_dataset(nq, dim, q_seed)
        kid, kd = ref.exact_knn_graph(data, d_init)
        counts = ref.count_detourable_routes(kid, kd)
        graph, _ = ref.optimize(kid, kd, d)
        gt_ids, gt_d = ref.exact_topk_batch(data, queries, 10)
        out = dict(n=n, dim=dim, d_init=d_init, d=d, data_seed=ds_seed, query_seed=q_seed, nq=nq,
                   data_head=data[:4].copy(), knn_ids=kid, knn_dists=kd, counts=counts,
                   graph=graph, gt_ids=gt_ids, gt_dists=gt_d, grid=np.array(GRID, np.uint64))
        ix = ref.index(data, graph)
        for gi, (mode, m, p, pol, bits, ri, teams, seed) in enumerate(GRID):
            prm = make_params(k=10, topm=m, width=p, hash_policy=pol, hash_bits=bits,
                              reset_interval=ri, seed=seed)
            ids, dists, cnt, st = ix.batch_search(queries, prm, mode=mode, team_count=teams)
            out[f"s{gi}_ids"] = ids
            out[f"s{gi}_dists"] = dists
            out[f"s{gi}_counts"] = cnt
            out[f"s{gi}_evals"] = st["distance_evals"]
            out[f"s{gi}_iters"] = st["iterations"]
            out[f"s{gi}_resets"] = st["hash_resets"]
            out[f"s{gi}_conv"] = st["converged"]
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


if __name__ == "__main__":
    main()
