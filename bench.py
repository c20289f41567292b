"""Benchmark: QPS at recall@10 >= 0.95 of batch beam search (the CAGRA hot
path) on the synthetic DEEP-1M shape (BASELINE.json configs[1]: 1M x 96 fp32,
graph degree 64, batch 10k), one process per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one batch_search of `--batch` queries over the device-resident index.

Our arm (default):
  * the index is built ON DEVICE by this process (exact kNN -> rank optimize,
    both bit-exact to the reference) and its build seconds are reported;
  * `value`    = queries / s with queries already in HBM (CUDA events around
                 each step on the launching stream, max over ranks);
  * `e2e`      = the same through the C-ABI call `cagra_search` with pinned
                 HOST query/result buffers: H2D + kernels + D2H inside the
                 timed region;
  * `roofline` = algorithmic gather bytes (distance rows + graph rows +
                 query + results, from the kernel's own per-query counters)
                 / search-kernel time, against MEASURED_PEAKS.json hbm_gbs;
  * `cpu_baseline` = the reference compiled from its own sources
                 (oracle/_ref, kind "reference") on a bounded query sample,
                 all host threads, rank 0 only.
Multi-GPU (torchrun): queries are sharded over replicated indexes — every rank
searches its own batch of `--batch` queries (weak scaling), no collective on
the data path; value = all ranks' queries / max-over-ranks time.

Reference arm (--impl reference): the unmodified reference's batch_search
(oracle/_ref) on the host cores, same index, same params, a bounded query
sample per step; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "QPS at recall@10=0.95 (batch 10k), 1M x 96 fp32, graph degree 64"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--points", dest="n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--batch", type=int, default=10_000)
    ap.add_argument("--degree", type=int, default=64)
    ap.add_argument("--topm", type=int, default=896)
    ap.add_argument("--width", type=int, default=16)
    ap.add_argument("--hash", default="forgettable", choices=["standard", "forgettable"])
    ap.add_argument("--hash-bits", type=int, default=12)
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="queries in the CPU baseline sample (0 = auto, ~10-30 s of work)")
    ap.add_argument("--batch1", type=int, default=500,
                    help="also time this many sequential batch-1 calls (0 = off)")
    ap.add_argument("--b1-topm", type=int, default=16, help="batch-1 team top-M")
    ap.add_argument("--b1-teams", type=int, default=64, help="batch-1 teams (one CTA each)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--build-once", action="store_true",
                    help="one graph build (large configs): graph_build_s is then the first build")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers --
class Clocks:
    """nvidia-smi sampler running DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_key):
    """dram bytes per search launch from the committed ncu --set full capture
    of this same workload (profiles/search_ncu.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "search_ncu.json")) as f:
            d = json.load(f)
        if d.get("config_key") == cfg_key:
            return float(d["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        pass
    return None


def recall_at_k(ids, gt, k=10):
    hits = 0
    for i in range(ids.shape[0]):
        hits += len(set(ids[i, :k].tolist()) & set(gt[i, :k].tolist()))
    return hits / (ids.shape[0] * k)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------ shared inputs --
def make_inputs(args, world, rank):
    from paper_2308_15136_b200 import capi

    data = capi.uniform_dataset(args.n, args.dim, 424242)
    # every rank owns its own batch of queries (weak scaling); rank 0's batch is
    # the single-GPU batch
    allq = capi.uniform_dataset(args.batch * world, args.dim, 424243)
    queries = np.ascontiguousarray(allq[rank * args.batch:(rank + 1) * args.batch])
    return data, queries


def search_params(args):
    from paper_2308_15136_b200 import fodg

    return fodg.SearchParams(
        k=10, topm=args.topm, width=args.width,
        hash_policy=fodg.HashPolicy.kForgettable if args.hash == "forgettable"
        else fodg.HashPolicy.kStandard,
        hash_bits=args.hash_bits, reset_interval=1, seed=11)


def config(args, world):
    return {"workload": f"synthetic uniform {args.n}x{args.dim} fp32 (DEEP-1M shape), graph "
                        f"degree {args.degree} (kNN {2 * args.degree} -> rank optimize), "
                        f"k=10, batch {args.batch} per GPU",
            "n": args.n, "dim": args.dim, "graph_degree": args.degree, "k": 10,
            "batch_per_gpu": args.batch, "global_batch": args.batch * world,
            "itopk_M": args.topm, "search_width_p": args.width, "hash": args.hash,
            "hash_bits": args.hash_bits, "seed": 11, "data_seed": 424242,
            "query_seed": 424243,
            "parallelism": f"query-sharded x{world} (replicated index)",
            "l2": "inputs larger than L2: dataset 384 MB + graph 256 MB vs 126 MB L2"}


# ------------------------------------------------------------- reference arm --
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch  # noqa: F401  (device for the index build below)

    from oracle.bindings import load_reference, make_params
    from paper_2308_15136_b200 import fodg

    ref = load_reference()
    if ref is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libfodg_ref.so was not built"}))
        return 0
    data, queries = make_inputs(args, 1, 0)
    ds = fodg.Dataset.from_array(data)
    # The reference cannot build a 1M graph on the host in bench time (exact
    # kNN ~4 h, NN-descent ~120 GB RSS), so its index is the graph
    # the device builds, which is bit-identical to what the reference's
    # optimize produces from the same exact kNN graph (tests/test_gpu_parity).
    g, _ = fodg.build_graph(ds, args.degree)
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    rix = ref.index(data, g.ids)
    threads = ref.hardware_threads()
    p = make_params(k=10, topm=args.topm, width=args.width,
                    hash_policy=1 if args.hash == "forgettable" else 0,
                    hash_bits=args.hash_bits, seed=11)
    # size the per-step sample to ~2-6 s of host work
    probe = queries[:max(threads, 8)]
    t0 = time.perf_counter()
    rix.batch_search(probe, p, threads=threads)
    per_q = (time.perf_counter() - t0) / probe.shape[0]
    sample = args.cpu_sample or int(min(args.batch, max(threads, 4.0 / max(per_q, 1e-6))))
    sample = max(1, min(sample, args.batch))
    sq = queries[:sample]
    for _ in range(args.warmup):
        rix.batch_search(sq, p, threads=threads)
    times, rec = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ids, _, _, _ = rix.batch_search(sq, p, threads=threads)
        times.append(time.perf_counter() - t0)
        rec.append(recall_at_k(ids, gt[:sample]))
    tot = sum(times)
    qps = sample * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference fixture generator)",
        "config": config(args, 1), "recall@10": float(np.mean(rec)),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{sample} of the {args.batch} batch queries per step, "
                                   f"fodg::batch_search per-query mode, {threads} threads"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm --
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2308_15136_b200 import capi, fodg

    world, rank, local = dist_env()
    # one process per GPU; CAGRA_BENCH_BACKEND=gloo lets several ranks share a
    # device (exercises the N>1 path on a 1-GPU box; NCCL needs distinct GPUs)
    backend = os.environ.get("CAGRA_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    data, queries = make_inputs(args, world, rank)
    ds = fodg.Dataset.from_array(data)
    # The first build in a process also pays one-time costs (module loading,
    # the driver mapping ~2 GB of fresh device memory): reported as
    # first_build_s; the graph_build_s figures are the steady-state second build.
    t0 = time.perf_counter()
    g, binfo = fodg.build_graph(ds, args.degree, device=local)
    first_build = {"knn": binfo["knn_seconds"], "wall": time.perf_counter() - t0}
    if not args.build_once:
        del g
        t0 = time.perf_counter()
        g, binfo = fodg.build_graph(ds, args.degree, device=local)
    build_wall = time.perf_counter() - t0
    kst = capi.knn_last_stats()
    # tensor work of the kNN build: sample pass (every 16th point) + full
    # pass, 2*N*N*K each, K = the filter GEMM's K (fp16 single term: dim + 2
    # rounded to 16; bf16x3: 3*dim + 6)
    gk = kst["gemm_k"]
    tc_flops = 2.0 * args.n * args.n * gk * (1 + 1 / 16)
    tc = kst["rows"] > 0  # 0 rows: the SIMT sequential-chain kernel ran (dim too large)
    split = {1: "fp16 single-term", 3: "bf16x3"}.get(kst["split_terms"], "?")
    knn_stats = {"path": (f"tcgen05 {split} filter GEMM (K={gk}) + exact re-rank (bit-exact)"
                          if tc else
                          "SIMT sequential-chain fp32 (bit-exact; dim beyond the tensor-core path)"),
                 "tensor_tflops": tc_flops / binfo["knn_seconds"] / 1e12 if tc else None,
                 "fp32_equiv_tflops": 2.0 * args.n * args.n * args.dim / binfo["knn_seconds"] / 1e12,
                 "rows": kst["rows"], "fallback_rows": kst["fallback_rows"],
                 "retried_rows": kst["retried_rows"],
                 "reranked_per_row": kst["reranked"] / max(1, kst["rows"])}
    gt, _ = fodg.exact_topk_batch(ds, queries, 10, device=local)
    ix = fodg.Index(ds, g, device=local)
    prm = search_params(args)
    opt = fodg.EngineOptions(device=local)
    nq, k, ld = args.batch, 10, ix.ld

    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    qd = torch.zeros((nq, ld), dtype=torch.float32, device=dev)
    qd[:, :args.dim] = torch.from_numpy(queries).to(dev)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    stats = torch.empty((nq, 6), dtype=torch.int32, device=dev)
    qoff = rank * nq  # global query index -> the same seeds as a 1-GPU run

    def step():
        ix.search_dev(qd, nq, prm, opt, ids, dists, None, stats, sp, query_offset=qoff)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    clk.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for i in range(args.steps):
        step()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    launches = ix.last_launch_count() * args.steps
    kernel_ms = float(np.mean(step_ms))
    total_ms = evs[0].elapsed_time(evs[-1])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()

    hid = ids.cpu().numpy().view(np.uint32)
    st = stats.cpu().numpy()
    evals = st[:, 2].astype(np.int64) + (st[:, 3].astype(np.int64) << 32)
    iters = st[:, 0].astype(np.int64)
    rec = recall_at_k(hid, gt)
    # algorithmic bytes per query: evaluated rows + expanded graph rows + query + results
    alg_bytes = float(evals.sum() * args.dim * 4 + iters.sum() * args.width * args.degree * 4
                      + nq * (args.dim * 4 + k * 8))

    # ---- e2e through the C-ABI with pinned host buffers
    hq = torch.from_numpy(queries).pin_memory()
    h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    h_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    import ctypes as C
    pc, oc = prm.c(), opt.c(0, qoff)
    L = capi.lib()

    def e2e_step():
        capi.check(L.cagra_search(ix.h, capi.ptr(hq), nq, args.dim, C.byref(pc), C.byref(oc),
                                  capi.ptr(h_ids), capi.ptr(h_d), None, None))

    for _ in range(max(1, args.warmup)):
        e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    e2e_ids = h_ids.numpy().view(np.uint32)
    assert np.array_equal(e2e_ids, hid), "device-resident and host-buffer paths disagree"

    # ---- batch-1 path: sequential single-query calls through the C ABI (host
    # buffers), shared mode as choose_mode picks for batch 1 (engine.cpp:86-93),
    # one CTA per team (multi-CTA)
    b1 = None
    if args.batch1:
        nb = min(args.batch1, nq)
        prm1 = fodg.SearchParams(k=10, topm=args.b1_topm, width=1, seed=11)
        mode = fodg.choose_mode(1, args.b1_topm)
        opt1 = fodg.EngineOptions(device=local, mode=mode, team_count=args.b1_teams)
        pc1, oc1 = prm1.c(), opt1.c(0, qoff)
        one_i = torch.empty((1, k), dtype=torch.int32).pin_memory()
        one_d = torch.empty((1, k), dtype=torch.float32).pin_memory()
        out = np.empty((nb, k), np.uint32)
        for i in range(min(3, nb)):
            capi.check(L.cagra_search(ix.h, capi.ptr(hq[i]), 1, args.dim, C.byref(pc1),
                                      C.byref(oc1), capi.ptr(one_i), capi.ptr(one_d), None, None))
        t0 = time.perf_counter()
        for i in range(nb):
            capi.check(L.cagra_search(ix.h, capi.ptr(hq[i]), 1, args.dim, C.byref(pc1),
                                      C.byref(oc1), capi.ptr(one_i), capi.ptr(one_d), None,
                                      None))
            out[i] = one_i.numpy().view(np.uint32)[0]
        b1s = time.perf_counter() - t0
        b1 = {"qps": nb / b1s, "latency_us": b1s / nb * 1e6, "recall@10": recall_at_k(out, gt[:nb]),
              "queries": nb, "mode": fodg.mode_name(mode), "team_topm": args.b1_topm,
              "teams": args.b1_teams, "launches_per_query": ix.last_launch_count(),
              "path": "C-ABI cagra_search, pinned host buffers, one CTA per team"}

    # ---- max over ranks
    vals = torch.tensor([total_ms, e2e_s, kernel_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        rr = torch.tensor([rec, alg_bytes], dtype=torch.float64, device=dev)
        dist.all_reduce(rr, op=dist.ReduceOp.SUM)
        rec_all = float(rr[0]) / world
        alg_all = float(rr[1])
    else:
        rec_all, alg_all = rec, alg_bytes
    total_ms, e2e_s, kernel_ms = [float(x) for x in vals.tolist()]
    ms_per_step = total_ms / args.steps
    value = world * nq * args.steps / (total_ms * 1e-3)

    peak, peak_src = measured_peak_hbm()
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9  # this rank's kernel, GB/s
    cfg = config(args, world)
    cfg_key = f"{args.n}x{args.dim}/d{args.degree}/b{nq}/M{args.topm}/p{args.width}/" \
              f"{args.hash}{args.hash_bits}"
    traffic = ncu_traffic(cfg_key)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, data, g.ids, queries, gt, hid)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference fixture generator mt19937_64 uniform[0,1))",
            "config": cfg,
            "recall@10": rec_all,
            "mean_distance_evals": float(evals.mean()),
            "mean_iterations": float(iters.mean()),
            "graph_build_s": {"knn": binfo["knn_seconds"], "optimize": binfo["optimize_seconds"],
                              "wall": build_wall, "first_build_s": first_build},
            "knn_build": knn_stats,
            "e2e": {"value": world * nq * args.steps / e2e_s, "unit": "queries/s",
                    "h2d_bytes_per_step": nq * args.dim * 4,
                    "d2h_bytes_per_step": nq * k * 8},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "search_kernel (single-CTA beam search)",
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "peak_source": peak_src},
            "clocks": clocks,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        if b1 is not None:
            line["batch1"] = b1
        if cpu and "parity_vs_gpu" in cpu:
            line["parity"] = cpu["parity_vs_gpu"]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_baseline(args, data, graph, queries, gt, gpu_ids):
    """The reference (oracle/_ref) on the host cores: bounded query sample."""
    try:
        from oracle.bindings import load_reference, make_params
    except Exception as ex:  # noqa: BLE001
        return {"value": None, "unavailable": str(ex)}
    ref = load_reference()
    if ref is None:
        return {"value": None, "unavailable": "oracle/_ref not built"}
    threads = ref.hardware_threads()
    rix = ref.index(data, graph)
    p = make_params(k=10, topm=args.topm, width=args.width,
                    hash_policy=1 if args.hash == "forgettable" else 0,
                    hash_bits=args.hash_bits, seed=11)
    probe = queries[:max(threads, 8)]
    t0 = time.perf_counter()
    rix.batch_search(probe, p, threads=threads)
    per_q = (time.perf_counter() - t0) / probe.shape[0]
    sample = args.cpu_sample or int(min(args.batch, max(threads, 12.0 / max(per_q, 1e-6))))
    sample = max(1, min(sample, args.batch))
    t0 = time.perf_counter()
    ids, _, _, _ = rix.batch_search(queries[:sample], p, threads=threads)
    el = time.perf_counter() - t0
    rix.close()
    # parity on the same queries, same params and seeds: the GPU batch's ids
    # (fast mode: team-reduced in-loop distances) against the reference's
    ref_rec = recall_at_k(ids, gt[:sample])
    gpu_rec = recall_at_k(gpu_ids[:sample], gt[:sample])
    parity = {"queries": sample, "recall_gpu": gpu_rec, "recall_reference": ref_rec,
              "delta_pp": 100.0 * (gpu_rec - ref_rec),
              "exact_id_match": float(np.mean(gpu_ids[:sample] == ids)),
              "set_overlap": float(np.mean([len(set(gpu_ids[i]) & set(ids[i])) / 10
                                            for i in range(sample)]))}
    return {"value": sample / el, "unit": "queries/s", "cores": threads, "kind": "reference",
            "recall@10": ref_rec, "parity_vs_gpu": parity,
            "sample": f"first {sample} of the {args.batch} batch queries, same index and "
                      f"params, fodg::batch_search per-query mode, {threads} threads"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
