"""bench.py's multi-GPU launch contract.

CPU: `--gpus N` inside a torch.distributed environment whose WORLD_SIZE
disagrees fails loudly (exit 2) instead of timing one GPU.
GPU (slow): `python bench.py --gpus 2` re-launches itself as 2 ranks (they
share the one B200 over gloo here) and prints n_gpus 2, in both the
query-sharded and the dataset-sharded layouts.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_disagreeing_with_world_size_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "3"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stderr
    assert "WORLD_SIZE=2" in r.stderr


def _bench_line(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


SMALL = ["--points", "60000", "--batch", "2000", "--steps", "2", "--warmup", "3",
         "--topm", "128", "--width", "4", "--batch1", "0", "--no-cpu"]


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_gpus2_query_sharded(gpu):
    d = _bench_line(["--gpus", "2"] + SMALL)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["global_batch"] == 4000
    assert d["recall@10"] > 0.9 and d["value"] > 0


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_gpus2_data_sharded(gpu):
    d = _bench_line(["--gpus", "2", "--shard", "data", "--shards-per-rank", "2"] + SMALL)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["graph_build_s"]["shards"] == 4
    assert d["recall@10"] > 0.9 and d["value"] > 0
