"""Benchmark of the CAGRA hot path on B200 (BASELINE.json metric: QPS at
recall@10 = 0.95, batch 10k and batch 1, at 1/2/4/8 GPUs; graph build
seconds), on the synthetic DEEP-1M shape (configs[1]: 1M x 96 fp32, graph
degree 64, batch 10k and batch 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--shard query|data] [--shards-per-rank S] [--points N] ...

A step = one batch search of `--batch` queries over the device-resident index.
`--gpus N` without a torch.distributed environment re-launches itself under
`torch.distributed.run` with N ranks (one process per GPU); inside one, N must
equal WORLD_SIZE.  When N exceeds the visible GPUs the ranks share devices over
gloo (a 1-GPU box exercising the N > 1 code path; not a scaling number).

Our arm (default):
  * the index is built ON DEVICE by this process (exact kNN -> rank optimize,
    both bit-exact to the reference) and its build seconds are reported;
  * `value`    = batch-10k queries / s with queries already in HBM (CUDA events
                 around each step on the launching stream, max over ranks);
  * `e2e`      = the same through the C-ABI call `cagra_search` with pinned
                 HOST query/result buffers: H2D + kernels + D2H timed;
  * `roofline` = algorithmic gather bytes (distance rows + graph rows + query +
                 results, from the kernel's own per-query counters) / search
                 kernel time, against MEASURED_PEAKS.json hbm_gbs;
  * `batch1`   = sequential single-query calls through the C ABI (host
                 buffers), with `parity` against the reference's shared mode at
                 the same params/seeds and its own single-threaded
                 `cpu_baseline` (per-query and shared x4 at the reference's
                 best recall >= 0.95 points, profiles/r02_cpu_batch1_sweep.txt);
  * `cpu_baseline` = the reference (oracle/_ref, kind "reference") at ITS best
                 batch-10k grid point with recall >= 0.95
                 (profiles/r02_cpu_batch10k_sweep.txt), all host threads, on a
                 bounded query sample, rank 0 at N = 1 only; `parity` = the
                 reference at the GPU's params and seeds on the same queries;
  * `optimize_parity` = fodg_ref::optimize run on this build's 1M kNN graph,
                 compared bit for bit with the device graph.
Multi-GPU:
  * --shard query (default; C2 scaling, C4): queries sharded over replicated
    indexes; every rank searches its own batch of `--batch` queries (weak
    scaling), no collective on the data path;
  * --shard data (C5): rank r holds `--shards-per-rank` contiguous id ranges
    with their own graphs; rank 0's queries are broadcast, every rank searches
    them on its shards, one all-gather of the per-shard top-k lists, K8 merge
    (strong scaling: the dataset and the batch are fixed).

Reference arm (--impl reference): the unmodified reference's batch_search
(oracle/_ref) on the host cores at the same params as our arm, a bounded query
sample per step; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = ("QPS at recall@10=0.95 (batch 10k and batch 1) at 1/2/4/8 B200; graph build sec")
# The reference's own best operating points on the box's host cores (recall@10
# >= 0.95, 1M x 96): profiles/r02_cpu_batch10k_sweep.txt (16 threads) and
# profiles/r02_cpu_batch1_sweep.txt (1 thread, sequential calls).
CPU_BATCH_POINT = {"topm": 896, "width": 16, "hash_policy": 0, "hash_bits": 11}
CPU_B1_PER_QUERY = {"topm": 896, "width": 16}
CPU_B1_SHARED = {"topm": 256, "teams": 4}


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
    ap.add_argument("--shard", default="query", choices=["query", "data"])
    ap.add_argument("--data", default="uniform", choices=["uniform", "lowrank"],
                    help="synthetic generator: the reference fixture's uniform[0,1) "
                         "(default) or low-intrinsic-dimension rows (C3)")
    ap.add_argument("--rank", type=int, default=32, help="intrinsic dimension for --data lowrank")
    ap.add_argument("--shards-per-rank", type=int, default=1,
                    help="data-sharded: id-range shards held by each rank (C5 on one GPU: 8)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="queries in the CPU baseline sample (0 = auto, ~10 s of work)")
    ap.add_argument("--batch1", type=int, default=500,
                    help="also time this many sequential batch-1 calls (0 = off)")
    ap.add_argument("--b1-topm", type=int, default=10, help="batch-1 team top-M")
    ap.add_argument("--b1-teams", type=int, default=96, help="batch-1 teams (one CTA each)")
    ap.add_argument("--no-cpu", action="store_true", help="skip every reference (CPU) leg")
    ap.add_argument("--cpu-topm", type=int, default=CPU_BATCH_POINT["topm"],
                    help="the reference's own batch operating point (default: its best "
                         "recall>=0.95 point at 1M x 96)")
    ap.add_argument("--cpu-width", type=int, default=CPU_BATCH_POINT["width"])
    ap.add_argument("--cpu-hash", default="standard", choices=["standard", "forgettable"])
    ap.add_argument("--no-opt-parity", action="store_true",
                    help="skip fodg_ref::optimize on the device-built kNN graph")
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


def host_cpu():
    """CPU model / thread count of this host (lscpu-equivalent, /proc/cpuinfo)."""
    model, sockets = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                elif ln.startswith("physical id"):
                    sockets.add(ln.split(":", 1)[1].strip())
    except OSError:
        pass
    return {"cpu_model": model, "sockets": max(1, len(sockets)), "threads": os.cpu_count()}


def recall_at_k(ids, gt, k=10):
    hits = 0
    for i in range(ids.shape[0]):
        hits += len(set(ids[i, :k].tolist()) & set(gt[i, :k].tolist()))
    return hits / (ids.shape[0] * k)


def id_parity(a, b, gt):
    """recall delta / exact-ID match / set overlap of two [nq, k] id arrays."""
    nq = a.shape[0]
    ra, rb = recall_at_k(a, gt), recall_at_k(b, gt)
    return {"queries": int(nq), "recall_gpu": ra, "recall_reference": rb,
            "delta_pp": 100.0 * (ra - rb), "exact_id_match": float(np.mean(a == b)),
            "set_overlap": float(np.mean([len(set(a[i]) & set(b[i])) / a.shape[1]
                                          for i in range(nq)]))}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args):
    """--gpus N outside torch.distributed: one process per GPU via torchrun."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ------------------------------------------------------------ shared inputs --
def lowrank_dataset(n, dim, rank, seed):
    """Low-intrinsic-dimension synthetic rows (the C3 decision):
    x = z A + e with z ~ U[0,1)^rank per row, one fixed A ~ U[-0.5,0.5)^(rank x
    dim) and e ~ 0.01 U[0,1)^dim (numpy PCG64; A from seed 4242, z / e from
    `seed`).  Uniform 960-d data has no neighbourhood structure (recall
    saturates near 0.8 for both arms); this keeps the GIST shape with a
    structure graph search can use.  Both arms search the same arrays."""
    a = np.random.default_rng(4242).random((rank, dim), dtype=np.float32) - np.float32(0.5)
    rng = np.random.default_rng(seed)
    out = np.empty((n, dim), np.float32)
    step = 1 << 18
    for i in range(0, n, step):
        m = min(step, n - i)
        z = rng.random((m, rank), dtype=np.float32)
        out[i:i + m] = z @ a + np.float32(0.01) * rng.random((m, dim), dtype=np.float32)
    return out


def gen_rows(args, count, seed):
    from paper_2308_15136_b200 import capi

    if args.data == "lowrank":
        return lowrank_dataset(count, args.dim, args.rank, seed)
    return capi.uniform_dataset(count, args.dim, seed)


def make_inputs(args, world, rank):
    data = gen_rows(args, args.n, 424242)
    if args.shard == "data":
        queries = gen_rows(args, args.batch, 424243)
        return data, queries
    # every rank owns its own batch of queries (weak scaling); rank 0's batch is
    # the single-GPU batch
    allq = gen_rows(args, args.batch * world, 424243)
    queries = np.ascontiguousarray(allq[rank * args.batch:(rank + 1) * args.batch])
    return data, queries


def search_params(args, **over):
    from paper_2308_15136_b200 import fodg

    kw = dict(topm=args.topm, width=args.width,
              hash_policy=1 if args.hash == "forgettable" else 0, hash_bits=args.hash_bits)
    kw.update(over)
    return fodg.SearchParams(k=10, topm=kw["topm"], width=kw["width"],
                             hash_policy=fodg.HashPolicy(kw["hash_policy"]),
                             hash_bits=kw["hash_bits"], reset_interval=1, seed=11)


def ref_params(args, **over):
    from oracle.bindings import make_params

    kw = dict(topm=args.topm, width=args.width,
              hash_policy=1 if args.hash == "forgettable" else 0, hash_bits=args.hash_bits)
    kw.update(over)
    return make_params(k=10, topm=kw["topm"], width=kw["width"], hash_policy=kw["hash_policy"],
                       hash_bits=kw["hash_bits"], seed=11)


def config(args, world, shared_devices=False):
    gb = 1e9
    data_b = args.n * args.dim * 4
    graph_b = args.n * args.degree * 4
    shape = {(1_000_000, 96): " (DEEP-1M shape)", (10_000_000, 96): " (DEEP-10M shape)",
             (1_000_000, 960): " (GIST shape)", (100_000_000, 96): " (C5 shape)",
             (100_000, 128): " (SIFT shape)"}.get((args.n, args.dim), "")
    if args.shard == "data":
        nsh = world * args.shards_per_rank
        par = (f"dataset-sharded: {nsh} id-range shards ({args.shards_per_rank} per rank x "
               f"{world} ranks), per-shard top-k all-gathered + K8 merge")
        batch = f"batch {args.batch} (all ranks search every query)"
    else:
        par = f"query-sharded x{world} (replicated index)"
        batch = f"batch {args.batch} per GPU"
    cfg = {"workload": f"synthetic uniform {args.n}x{args.dim} fp32{shape}, graph degree "
                       f"{args.degree} (kNN {2 * args.degree} -> rank optimize), k=10, {batch}",
           "n": args.n, "dim": args.dim, "graph_degree": args.degree, "k": 10,
           "batch_per_gpu": args.batch if args.shard == "query" else None,
           "global_batch": args.batch * (world if args.shard == "query" else 1),
           "itopk_M": args.topm, "search_width_p": args.width, "hash": args.hash,
           "hash_bits": args.hash_bits, "seed": 11, "data_seed": 424242,
           "query_seed": 424243, "parallelism": par,
           "l2": (f"inputs larger than L2: dataset {data_b / gb:.2f} GB + graph "
                  f"{graph_b / gb:.2f} GB vs 0.126 GB L2")}
    if shared_devices:
        cfg["note"] = ("ranks share GPUs (more ranks than visible devices, gloo): exercises the "
                       "N > 1 path, not a scaling measurement")
    return cfg


# ------------------------------------------------------------- reference arm --
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch  # noqa: F401  (device for the index build below)

    from oracle.bindings import load_reference
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
    # optimize produces from the same exact kNN graph (bench optimize_parity,
    # tests/test_gpu_parity).  Outside the timed region.
    g, _ = fodg.build_graph(ds, args.degree)
    gt, _ = fodg.exact_topk_batch(ds, queries, 10)
    rix = ref.index(data, g.ids)
    threads = ref.hardware_threads()
    p = ref_params(args)
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
                         "kind": "reference", **host_cpu(),
                         "sample": f"{sample} of the {args.batch} batch queries per step, "
                                   f"fodg::batch_search per-query mode, {threads} threads"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm --
class Dist:
    """torch.distributed plumbing for N > 1 (NCCL; gloo when ranks share GPUs)."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world, self.rank, local = dist_env()
        ndev = max(1, torch.cuda.device_count())
        self.shared = self.world > ndev
        self.backend = os.environ.get("CAGRA_BENCH_BACKEND",
                                      "gloo" if self.shared else "nccl")
        self.local = local % ndev
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max(self, vals):
        """element-wise max over ranks of a list of floats"""
        if self.world == 1:
            return vals
        t = self.torch.tensor(vals, dtype=self.torch.float64,
                              device=self.dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    def sum(self, vals):
        if self.world == 1:
            return vals
        t = self.torch.tensor(vals, dtype=self.torch.float64,
                              device=self.dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return [float(x) for x in t.tolist()]

    def done(self):
        if self.world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


def build_graph(args, ds, local, want_knn=False):
    """Device build (exact kNN -> optimize); steady-state second build unless
    --build-once.  Returns (graph, info, first_build, wall[, knn])."""
    from paper_2308_15136_b200 import fodg

    t0 = time.perf_counter()
    r = fodg.build_graph(ds, args.degree, device=local, return_knn=want_knn and args.build_once)
    first = {"knn": r[1]["knn_seconds"], "wall": time.perf_counter() - t0}
    if not args.build_once:
        del r
        t0 = time.perf_counter()
        r = fodg.build_graph(ds, args.degree, device=local, return_knn=want_knn)
    wall = time.perf_counter() - t0
    return r, first, wall


def knn_stats(args, n, binfo):
    from paper_2308_15136_b200 import capi

    kst = capi.knn_last_stats()
    # tensor work of the kNN build: sample pass (every 16th point) + full
    # pass, 2*N*N*K each, K = the filter GEMM's K (fp16 single term: dim + 2
    # rounded to 16; bf16x3: 3*dim + 6)
    gk = kst["gemm_k"]
    tc_flops = 2.0 * n * n * gk * (1 + 1 / 16)
    tc = kst["rows"] > 0  # 0 rows: the SIMT sequential-chain kernel ran (dim too large)
    split = {1: "fp16 single-term", 3: "bf16x3"}.get(kst["split_terms"], "?")
    return {"path": (f"tcgen05 {split} filter GEMM (K={gk}) + exact re-rank (bit-exact)"
                     if tc else
                     "SIMT sequential-chain fp32 (bit-exact; dim beyond the tensor-core path)"),
            "tensor_tflops": tc_flops / binfo["knn_seconds"] / 1e12 if tc else None,
            "fp32_equiv_tflops": 2.0 * n * n * args.dim / binfo["knn_seconds"] / 1e12,
            "rows": kst["rows"], "fallback_rows": kst["fallback_rows"],
            "retried_rows": kst["retried_rows"],
            "reranked_per_row": kst["reranked"] / max(1, kst["rows"])}


def run_ours(args):
    world, rank, _ = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    D = Dist()
    if args.shard == "data":
        return run_data_sharded(args, D)
    return run_query_sharded(args, D)


def run_query_sharded(args, D):
    import ctypes as C

    import torch

    from paper_2308_15136_b200 import capi, fodg

    world, rank, local, dev = D.world, D.rank, D.local, D.dev
    data, queries = make_inputs(args, world, rank)
    ds = fodg.Dataset.from_array(data)
    want_knn = rank == 0 and world == 1 and not args.no_cpu and not args.no_opt_parity
    if world > 1:
        # row-sharded build: each rank computes N/world kNN rows, one
        # all-gather, every rank optimizes (bit-identical to a 1-GPU build)
        from paper_2308_15136_b200 import dist as pdist

        D.barrier()
        t0 = time.perf_counter()
        g, rinfo = pdist.build_graph_row_sharded(ds, args.degree, local)
        D.barrier()
        build_wall = time.perf_counter() - t0
        (build_wall,) = D.max([build_wall])
        binfo = {"knn_seconds": rinfo["knn_rows_seconds"] + rinfo["gather_seconds"],
                 "optimize_seconds": rinfo["optimize_seconds"]}
        first_build = {"row_sharded": rinfo}
        knn = None
        kstats = {"path": "row-sharded over ranks: cagra_exact_knn_rows + all-gather + optimize",
                  "rows_per_rank": rinfo["rows"]}
    else:
        r, first_build, build_wall = build_graph(args, ds, local, want_knn)
        g, binfo = r[0], r[1]
        knn = r[2] if want_knn else None
        kstats = knn_stats(args, args.n, binfo)
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
    D.barrier()
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
    D.barrier()
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
    pc, oc = prm.c(), opt.c(0, qoff)
    L = capi.lib()

    def e2e_step():
        capi.check(L.cagra_search(ix.h, capi.ptr(hq), nq, args.dim, C.byref(pc), C.byref(oc),
                                  capi.ptr(h_ids), capi.ptr(h_d), None, None))

    for _ in range(max(1, args.warmup)):
        e2e_step()
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    e2e_ids = h_ids.numpy().view(np.uint32)
    assert np.array_equal(e2e_ids, hid), "device-resident and host-buffer paths disagree"

    # ---- batch-1: sequential single-query calls through the C ABI (host
    # buffers), shared mode as choose_mode picks for batch 1 (engine.cpp:86-93),
    # one CTA per team (multi-CTA)
    b1 = None
    if args.batch1:
        nb = min(args.batch1, nq)
        prm1 = fodg.SearchParams(k=10, topm=args.b1_topm, width=1, seed=11)
        mode = fodg.choose_mode(1, args.b1_topm)
        opt1 = fodg.EngineOptions(device=local, mode=mode, team_count=args.b1_teams)
        pc1, oc1 = prm1.c(), opt1.c(0, qoff)
        # every call gets its own query row and its own result rows of pinned
        # host buffers (argument objects built before the timed loop, so the
        # loop is the C-ABI call and little Python around it)
        b1_i = torch.empty((nb, k), dtype=torch.int32).pin_memory()
        b1_d = torch.empty((nb, k), dtype=torch.float32).pin_memory()
        qrow, rrow = hq.stride(0) * 4, k * 4
        q0, i0, d0 = hq.data_ptr(), b1_i.data_ptr(), b1_d.data_ptr()
        argv = [(C.c_void_p(q0 + i * qrow), C.c_void_p(i0 + i * rrow), C.c_void_p(d0 + i * rrow))
                for i in range(nb)]
        call, h, dim1, ppc, poc = L.cagra_search, ix.h, args.dim, C.byref(pc1), C.byref(oc1)
        for i in range(min(3, nb)):
            capi.check(call(h, argv[i][0], 1, dim1, ppc, poc, argv[i][1], argv[i][2], None, None))
        rcs = [0] * nb
        t0 = time.perf_counter()
        for i in range(nb):
            a = argv[i]
            rcs[i] = call(h, a[0], 1, dim1, ppc, poc, a[1], a[2], None, None)
        b1s = time.perf_counter() - t0
        for rc in rcs:
            capi.check(rc)
        out = b1_i.numpy().view(np.uint32).copy()
        b1 = {"qps": nb / b1s, "latency_us": b1s / nb * 1e6, "recall@10": recall_at_k(out, gt[:nb]),
              "queries": nb, "mode": fodg.mode_name(mode), "team_topm": args.b1_topm,
              "teams": args.b1_teams, "launches_per_query": ix.last_launch_count(),
              "path": "C-ABI cagra_search, pinned host buffers, one CTA per team"}
        b1_ids = out

    # ---- max over ranks
    total_ms, e2e_s, kernel_ms = D.max([total_ms, e2e_s, kernel_ms])
    rec_all, alg_all = D.sum([rec, alg_bytes])
    rec_all /= world
    ms_per_step = total_ms / args.steps
    value = world * nq * args.steps / (total_ms * 1e-3)

    peak, peak_src = measured_peak_hbm()
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9  # this rank's kernel, GB/s
    cfg = config(args, world, D.shared)
    cfg_key = f"{args.n}x{args.dim}/d{args.degree}/b{nq}/M{args.topm}/p{args.width}/" \
              f"{args.hash}{args.hash_bits}"
    traffic = ncu_traffic(cfg_key)

    cpu = parity = opt_par = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, parity = cpu_batch_legs(args, data, g.ids, queries, gt, hid)
        if b1 is not None:
            b1["parity"], b1["cpu_baseline"] = cpu_batch1_legs(args, data, g.ids, queries, gt,
                                                               b1_ids)
        if knn is not None:
            opt_par = optimize_parity(args, knn, g.ids, binfo)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": ("synthetic (reference fixture generator mt19937_64 uniform[0,1))"
                     if args.data == "uniform" else
                     f"synthetic low-rank: z A + 0.01 e, intrinsic dimension {args.rank} "
                     "(numpy PCG64; bench.lowrank_dataset), same arrays for both arms"),
            "config": cfg,
            "value_is": "batch-10k QPS (per GPU batch) at recall@10 >= 0.95; batch 1 in `batch1`",
            "recall@10": rec_all,
            "mean_distance_evals": float(evals.mean()),
            "mean_iterations": float(iters.mean()),
            "graph_build_s": {"knn": binfo["knn_seconds"], "optimize": binfo["optimize_seconds"],
                              "wall": build_wall, "first_build_s": first_build},
            "knn_build": kstats,
            "e2e": {"value": world * nq * args.steps / e2e_s, "unit": "queries/s",
                    "h2d_bytes_per_step": nq * args.dim * 4,
                    "d2h_bytes_per_step": nq * k * 8},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "search_kernel (single-CTA beam search)",
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "peak_source": peak_src,
                         # the access pattern's own ceiling: random whole-row
                         # gathers with nothing else in the loop (committed
                         # measurement, profiles/r02_gather_ceiling.txt)
                         "gather_ceiling": gather_ceiling(args.n, args.dim)},
            "clocks": clocks,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        gc = line["roofline"]["gather_ceiling"]
        if gc:
            gc["frac"] = achieved / gc["gbs"]
        if parity is not None:
            line["parity"] = parity
        if cpu and cpu.get("mean_distance_evals") and args.cpu_hash == "standard" and \
                args.cpu_topm == args.topm and args.cpu_width == args.width:
            # the standard (never-forget) policy's evaluations at the same M, p:
            # the share of this kernel's gathered rows that are not revisits
            std_e = cpu["mean_distance_evals"]
            line["roofline"]["standard_policy_mean_evals"] = std_e
            line["roofline"]["useful_fraction_vs_standard"] = std_e / float(evals.mean())
            line["roofline"]["frac_useful"] = line["roofline"]["frac"] * std_e / float(evals.mean())
        if b1 is not None:
            line["batch1"] = b1
        if opt_par is not None:
            line["optimize_parity"] = opt_par
        print(json.dumps(line), flush=True)
    D.done()
    return 0


def cpu_batch_legs(args, data, graph, queries, gt, gpu_ids):
    """Batch-10k reference legs on the host: (cpu_baseline at the reference's
    own best grid point, parity at the GPU's params on the same queries)."""
    try:
        from oracle.bindings import load_reference
    except Exception as ex:  # noqa: BLE001
        return {"value": None, "unavailable": str(ex)}, None
    ref = load_reference()
    if ref is None:
        return {"value": None, "unavailable": "oracle/_ref not built"}, None
    threads = ref.hardware_threads()
    rix = ref.index(data, graph)
    # parity: the reference at the GPU's params/seeds, ~2 s of host work
    pg = ref_params(args)
    npar = min(args.batch, 2000)
    pids, _, _, _ = rix.batch_search(queries[:npar], pg, threads=threads)
    parity = id_parity(gpu_ids[:npar], pids, gt[:npar])
    parity["params"] = f"M={args.topm} p={args.width} {args.hash} (the GPU's)"
    # baseline: the reference's own best recall >= 0.95 point
    pb = ref_params(args, topm=args.cpu_topm, width=args.cpu_width,
                    hash_policy=1 if args.cpu_hash == "forgettable" else 0,
                    hash_bits=args.hash_bits if args.cpu_hash == "forgettable" else 11)
    probe = queries[:max(threads, 8)]
    t0 = time.perf_counter()
    rix.batch_search(probe, pb, threads=threads)
    per_q = (time.perf_counter() - t0) / probe.shape[0]
    sample = args.cpu_sample or int(min(args.batch, max(threads, 10.0 / max(per_q, 1e-6))))
    sample = max(1, min(sample, args.batch))
    t0 = time.perf_counter()
    ids, _, _, st = rix.batch_search(queries[:sample], pb, threads=threads)
    el = time.perf_counter() - t0
    rix.close()
    cpu = {"value": sample / el, "unit": "queries/s", "cores": threads, "kind": "reference",
           **host_cpu(), "recall@10": recall_at_k(ids, gt[:sample]),
           "mean_distance_evals": float(np.mean(st["distance_evals"])),
           "operating_point": f"per-query M={args.cpu_topm} p={args.cpu_width} {args.cpu_hash} hash "
                              + ("(the reference's best recall>=0.95 grid point at 1M x 96, "
                                 "profiles/r02_cpu_batch10k_sweep.txt)"
                                 if (args.cpu_topm, args.cpu_width) ==
                                 (CPU_BATCH_POINT["topm"], CPU_BATCH_POINT["width"])
                                 else "(--cpu-topm/--cpu-width: the reference's recall>=0.95 "
                                      "point for this configuration)"),
           "sample": f"first {sample} of the {args.batch} batch queries, same index, "
                     f"fodg::batch_search per-query mode, {threads} threads"}
    return cpu, parity


def gather_ceiling(n, dim):
    """Measured random-row-gather ceiling (tools/cpp/gather_peak.cu on one B200,
    best of 1-6 rows in flight per 8-lane team, 4 CTAs/SM) for 384-byte rows:
    8861 GB/s at 1M rows (L2 reuse included), 6961 at 10M, 6824 at 40M.
    None for other row sizes."""
    if dim != 96:
        return None
    gbs = 8861.0 if n <= 2_000_000 else (6961.0 if n <= 20_000_000 else 6824.0)
    return {"gbs": gbs, "source": "profiles/r02_gather_ceiling.txt (tools/cpp/gather_peak.cu)"}


def cpu_batch1_legs(args, data, graph, queries, gt, gpu_b1_ids):
    """Batch-1 reference legs: parity of the GPU's multi-CTA shared mode vs the
    reference's shared mode (engine.cpp:38-78) at the same M, teams and seeds;
    single-threaded sequential batch-1 baselines (per-query and shared x4)."""
    from oracle.bindings import load_reference

    ref = load_reference()
    if ref is None:
        return None, None
    threads = ref.hardware_threads()
    rix = ref.index(data, graph)
    nb = gpu_b1_ids.shape[0]
    p1 = ref_params(args, topm=args.b1_topm, width=1, hash_policy=0, hash_bits=11)
    # parity: same queries, each a batch of one (query index 0 within its call
    # -> seed mix_seed(seed ^ 0x0bad), as the GPU's batch-1 calls); the
    # reference's threads run different queries in parallel (results do not
    # depend on it)
    ref_ids = np.empty_like(gpu_b1_ids)
    lock = threading.Lock()
    nxt = [0]

    def worker():
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= nb:
                return
            r, _, _, _ = rix.batch_search(queries[i:i + 1], p1, mode=1,
                                          team_count=args.b1_teams, threads=1)
            ref_ids[i] = r[0]

    ths = [threading.Thread(target=worker) for _ in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    parity = id_parity(gpu_b1_ids, ref_ids, gt[:nb])
    parity["params"] = f"shared mode, {args.b1_teams} teams, M={args.b1_topm}, p=1"

    def seq(p, mode, teams, budget_s=4.0):
        t0 = time.perf_counter()
        out, i = [], 0
        while i < nb and (time.perf_counter() - t0 < budget_s or i < 20):
            r, _, _, _ = rix.batch_search(queries[i:i + 1], p, mode=mode, team_count=teams,
                                          threads=1)
            out.append(r[0])
            i += 1
        el = time.perf_counter() - t0
        return {"value": i / el, "unit": "queries/s", "queries": i,
                "recall@10": recall_at_k(np.array(out), gt[:i])}

    pq = seq(ref_params(args, topm=CPU_B1_PER_QUERY["topm"], width=CPU_B1_PER_QUERY["width"],
                        hash_policy=0, hash_bits=11), 0, 4)
    sh = seq(ref_params(args, topm=CPU_B1_SHARED["topm"], width=1, hash_policy=0,
                        hash_bits=11), 1, CPU_B1_SHARED["teams"])
    rix.close()
    best = max(pq["value"], sh["value"])
    cpu = {"value": best, "unit": "queries/s", "cores": 1, "kind": "reference", **host_cpu(),
           "per_query": {**pq, "params": "M=896 p=16"},
           "shared_x4": {**sh, "params": "M=256, 4 teams"},
           "sample": "sequential single-query fodg::batch_search calls, single-threaded "
                     "(the reference's batch-1 path), ~4 s per mode; operating points from "
                     "profiles/r02_cpu_batch1_sweep.txt"}
    return parity, cpu


def optimize_parity(args, knn, graph_ids, binfo):
    """fodg_ref::optimize (graph_opt.cpp:211-246) on this build's exact kNN
    graph, all host threads, compared bit for bit with the device graph."""
    from oracle.bindings import load_reference

    ref = load_reference()
    if ref is None:
        return None
    t0 = time.perf_counter()
    out, secs = ref.optimize(knn.ids.reshape(knn.num_nodes, knn.degree),
                             knn.dists.reshape(knn.num_nodes, knn.degree), args.degree)
    el = time.perf_counter() - t0
    g = np.asarray(graph_ids).reshape(out.shape)
    return {"bit_exact": bool(np.array_equal(out, g)),
            "rows_differing": int(np.sum(np.any(out != g, axis=1))),
            "reference_seconds": el, "reference_threads": ref.hardware_threads(),
            "device_optimize_seconds": binfo["optimize_seconds"],
            "what": "fodg_ref::optimize(knn, d=64) on the device-built exact kNN graph vs the "
                    "device graph"}


# -------------------------------------------------------- dataset-sharded --
def run_data_sharded(args, D):
    """C5 layout: every rank holds --shards-per-rank contiguous id ranges with
    their own graphs; all ranks search every query; per-shard top-k lists are
    all-gathered once and merged by K8 (cagra_merge_shard_topk_dev)."""
    import torch

    from paper_2308_15136_b200 import capi, fodg
    from paper_2308_15136_b200 import dist as pdist

    world, rank, local, dev = D.world, D.rank, D.local, D.dev
    S = args.shards_per_rank
    G = world * S
    bounds = pdist.shard_bounds(args.n, G)
    mine = list(range(rank * S, (rank + 1) * S))
    big = args.n > 20_000_000
    if not big:
        full = gen_rows(args, args.n, 424242)
    queries = gen_rows(args, args.batch, 424243)
    nq, k = args.batch, 10
    shards, build_s, knn_s, opt_s = [], 0.0, 0.0, 0.0
    gt_lists = []
    for s in mine:
        a, b = bounds[s]
        # C5 (> 20M points): every shard has its own generator seed
        # (424242 + shard) so no rank materialises the whole 38 GB dataset —
        # NOT the reference generator's sequence (labelled in `data`)
        part = (capi.uniform_dataset(b - a, args.dim, 424242 + s) if big
                else np.ascontiguousarray(full[a:b]))
        t0 = time.perf_counter()
        sh = pdist.ShardedIndex.build(part, a, args.degree, local)
        build_s += time.perf_counter() - t0
        knn_s += sh.build_info["knn_seconds"]
        opt_s += sh.build_info["optimize_seconds"]
        gt_lists.append(fodg.exact_topk_batch(fodg.Dataset.from_array(part), queries, k,
                                              device=local))
        shards.append(sh)
        del part
    if not big:
        del full
    offsets = [bounds[s][0] for s in range(G)]
    prm = search_params(args)
    opt = fodg.EngineOptions(device=local)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ld = shards[0].index.ld
    # rank 0's queries, broadcast (the batch's one H2D happens on rank 0)
    qd = torch.zeros((nq, ld), dtype=torch.float32, device=dev)
    if rank == 0:
        qd[:, :args.dim] = torch.from_numpy(queries).to(dev)
    if world > 1:
        if D.backend == "nccl":
            D.dist.broadcast(qd, 0)
        else:
            qc = qd.cpu()
            D.dist.broadcast(qc, 0)
            qd.copy_(qc)
    # ground truth: exact per-shard top-10 merged the same way (exact)
    gi = torch.from_numpy(np.stack([x[0] for x in gt_lists]).view(np.int32)).to(dev)
    gd = torch.from_numpy(np.stack([x[1] for x in gt_lists])).to(dev)
    gt = merge_over_ranks(D, gi, gd, offsets, local, stream)[0].cpu().numpy().view(np.uint32)
    stats = [torch.empty((nq, 6), dtype=torch.int32, device=dev) for _ in shards]

    def step():
        li, ldd = [], []
        for j, sh in enumerate(shards):
            i_, d_ = sh.search_local(qd, nq, prm, opt, stream.cuda_stream, stats=stats[j])
            li.append(i_)
            ldd.append(d_)
        return merge_over_ranks(D, torch.stack(li), torch.stack(ldd), offsets, local, stream)

    for _ in range(args.warmup):
        step()
    D.barrier()
    clk = Clocks(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out_i, out_d = step()
    e1.record(stream)
    torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    D.barrier()
    clocks = clk.stop()
    ids = out_i.cpu().numpy().view(np.uint32)
    rec = recall_at_k(ids, gt)
    evals = sum(int((st[:, 2].cpu().numpy().astype(np.int64)
                     + (st[:, 3].cpu().numpy().astype(np.int64) << 32)).sum()) for st in stats)
    iters = sum(int(st[:, 0].cpu().numpy().astype(np.int64).sum()) for st in stats)
    alg_bytes = float(evals * args.dim * 4 + iters * args.width * args.degree * 4
                      + S * nq * (args.dim * 4 + k * 8))
    launches = sum(sh.index.last_launch_count() for sh in shards) * args.steps + args.steps
    (total_ms,) = D.max([total_ms])
    alg_all, build_all, knn_all, opt_all = D.sum([alg_bytes, build_s, knn_s, opt_s])
    value = nq * args.steps / (total_ms * 1e-3)
    peak, peak_src = measured_peak_hbm()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": ("synthetic uniform[0,1); per-shard mt19937_64 seeds 424242+shard (C5 size: "
                     "not the reference generator's single sequence)" if big else
                     "synthetic (reference fixture generator mt19937_64 uniform[0,1))"),
            "config": config(args, world, D.shared),
            "value_is": "batch QPS over the whole sharded index (every query answered over all "
                        "shards), recall@10 vs the exact global top-10",
            "recall@10": rec,
            "graph_build_s": {"shards": G, "wall_sum": build_all, "knn_sum": knn_all,
                              "optimize_sum": opt_all,
                              "per_shard_points": bounds[0][1] - bounds[0][0]},
            "roofline": {"bound": "hbm", "achieved": alg_all / (total_ms * 1e-3) / 1e9 / world,
                         "peak": peak, "unit": "GB/s",
                         "frac": alg_all / (total_ms * 1e-3) / 1e9 / world / peak,
                         "traffic": None,
                         "kernel": "search_kernel over every local shard + K8 merge (per GPU)",
                         "algorithmic_bytes_per_step": alg_all / args.steps,
                         "peak_source": peak_src},
            "e2e": None,
            "clocks": clocks, "gpu_launches": launches, "cpu_baseline": None,
            "cpu_baseline_note": "the reference cannot hold or build the sharded index; see the "
                                 "query-sharded line for the CPU baseline",
        }
        print(json.dumps(line), flush=True)
    D.done()
    return 0


def merge_over_ranks(D, li, ldd, offsets, local, stream):
    """[S, nq, k] local shard lists -> all-gather over ranks -> K8 merge."""
    from paper_2308_15136_b200 import dist as pdist

    if D.world > 1:
        if D.backend == "nccl":
            gi, gd = pdist.exchange_topk(li, ldd)
        else:
            gi, gd = pdist.exchange_topk(li.cpu(), ldd.cpu())
            gi, gd = gi.to(li.device), gd.to(li.device)
        li = gi.reshape(-1, *li.shape[1:])
        ldd = gd.reshape(-1, *ldd.shape[1:])
    return pdist.merge_shard_topk(li, ldd, offsets, local, stream.cuda_stream)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
