"""Out-of-bounds write checks without compute-sanitizer (closed on the GPU
pool): every device output of the search entry point is a slice in the
middle of a larger sentinel-filled buffer, and after the call the guard
zones on both sides must be untouched, every id < n and every count <= k.
Covers the per-query kernel (forgettable smem table and standard bitmap),
the lockstep shared kernel, the multi-CTA shared kernel, the fused batch-1
team kernel and the k > 256 team merge."""
import numpy as np
import pytest
import torch

from paper_2308_15136_b200 import capi, fodg

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side
SENT = 0x5A5A5A5A


def guarded(n, dtype):
    buf = torch.full((n + 2 * GUARD,), SENT, dtype=torch.int32, device="cuda:0")
    return buf, buf[GUARD:GUARD + n].view(dtype)


def check_guards(buf, n):
    h = buf.cpu().numpy()
    assert (h[:GUARD] == SENT).all(), "write below the output buffer"
    assert (h[GUARD + n:] == SENT).all(), "write past the end of the output buffer"


CASES = [
    # (label, SearchParams kwargs, EngineOptions kwargs, nq)
    ("per_query_forgettable", dict(k=10, topm=128, width=4, hash_policy=fodg.HashPolicy.kForgettable,
                                   hash_bits=10), dict(), 300),
    ("per_query_standard", dict(k=10, topm=96, width=2), dict(), 300),
    ("per_query_exact", dict(k=16, topm=64, width=1), dict(exact_distances=True), 200),
    ("shared_lockstep", dict(k=10, topm=32, width=1),
     dict(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=4, multi_cta=1), 40),
    ("shared_multi_cta", dict(k=10, topm=64, width=1),
     dict(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=8, multi_cta=2), 40),
    ("shared_b1_team", dict(k=10, topm=16, width=1),
     dict(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=32), 3),
    ("team_merge_k300", dict(k=300, topm=320, width=1),
     dict(mode=fodg.ExecutionMode.kSharedQueryWorkers, team_count=4, multi_cta=2), 5),
]


@pytest.fixture(scope="module")
def index():
    n, dim = 20000, 40
    data = capi.uniform_dataset(n, dim, 7)
    ds = fodg.Dataset.from_array(data)
    g, _ = fodg.build_graph(ds, 32)
    return fodg.Index(ds, g), n, dim


@pytest.mark.parametrize("label,sp,eo,nq", CASES, ids=[c[0] for c in CASES])
def test_search_outputs_stay_in_bounds(gpu, index, label, sp, eo, nq):
    ix, n, dim = index
    params = fodg.SearchParams(seed=3, **sp)
    opts = fodg.EngineOptions(**eo)
    k = params.k
    queries = capi.uniform_dataset(nq, dim, 11)
    q = torch.zeros((nq, ix.ld), dtype=torch.float32, device="cuda:0")
    q[:, :dim] = torch.from_numpy(queries).cuda()
    ib, ids = guarded(nq * k, torch.int32)
    db, dists = guarded(nq * k, torch.float32)
    cb, counts = guarded(nq, torch.int32)
    sb, stats = guarded(nq * 6, torch.int32)
    torch.cuda.synchronize()
    ix.search_dev(q, nq, params, opts, ids, dists, counts, stats,
                  stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for b, m in ((ib, nq * k), (db, nq * k), (cb, nq), (sb, nq * 6)):
        check_guards(b, m)
    c = counts.cpu().numpy()
    assert ((c >= 1) & (c <= k)).all()
    hid = ids.view(nq, k).cpu().numpy()
    for i in range(nq):
        assert (hid[i, :c[i]].astype(np.int64) < n).all()
    # the host-buffer path agrees with the device path
    ids2, _, counts2, _ = ix.search(queries, params, opts)
    if label not in ("shared_multi_cta", "shared_b1_team", "team_merge_k300"):  # racing teams
        assert np.array_equal(counts2, c)
        assert np.array_equal(ids2.astype(np.int64), hid.astype(np.uint32).astype(np.int64))
