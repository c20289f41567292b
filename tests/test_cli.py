"""The `fodg` CLI drop-in (paper_2308_15136_b200/lib/fodg): the reference
CLI's subcommands, flags and exit codes (tools/main.cpp:21-23, 231-309)."""
import os
import subprocess

import numpy as np
import pytest

from paper_2308_15136_b200 import fodg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2308_15136_b200", "lib", "fodg")


def run(*args):
    if not os.path.exists(CLI):
        pytest.fail("fodg CLI not built (make)")
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_cli_usage_errors_exit_2():
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("metrics").returncode == 2                      # --graph required
    assert run("build", "--data", "x", "--out", "y", "--bogus", "1").returncode == 2
    assert run("--help").returncode == 0


def test_cli_format_errors_exit_3(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTAGRAPH" + b"\0" * 20)
    assert run("metrics", "--graph", str(bad)).returncode == 3
    assert run("metrics", "--graph", str(tmp_path / "missing.bin")).returncode == 3


def _write_fvecs(path, a):
    a = np.asarray(a, np.float32)
    with open(path, "wb") as f:
        for row in a:
            f.write(np.int32(a.shape[1]).tobytes())
            f.write(row.tobytes())


def _write_ivecs(path, a):
    a = np.asarray(a, np.int32)
    with open(path, "wb") as f:
        for row in a:
            f.write(np.int32(a.shape[1]).tobytes())
            f.write(row.tobytes())


@pytest.mark.gpu
def test_cli_build_metrics_search_bench(gpu, oracle, tmp_path):
    data = oracle.uniform_dataset(3000, 16, 61)
    queries = oracle.uniform_dataset(40, 16, 62)
    dp, qp, gp, tp, csv = (tmp_path / n for n in ("d.fvecs", "q.fvecs", "g.bin", "t.ivecs", "o.csv"))
    _write_fvecs(dp, data)
    _write_fvecs(qp, queries)
    r = run("build", "--data", str(dp), "--out", str(gp), "--d", "16")
    assert r.returncode == 0, r.stderr
    assert "builder=exact" in r.stdout and "degree=16" in r.stdout
    m = run("metrics", "--graph", str(gp))
    assert m.returncode == 0 and "strong_cc=" in m.stdout
    s = run("search", "--graph", str(gp), "--data", str(dp), "--queries", str(qp), "--k", "5")
    assert s.returncode == 0 and s.stdout.count("query ") == 40
    gt, _ = fodg.exact_topk_batch(fodg.Dataset.from_array(data), queries, 10)
    _write_ivecs(tp, gt.astype(np.int32))
    b = run("bench", "--graph", str(gp), "--data", str(dp), "--queries", str(qp), "--truth", str(tp),
            "--grid", "M=16,32", "--grid", "p=1,2", "--k", "10", "--out", str(csv))
    assert b.returncode == 0, b.stderr
    lines = csv.read_text().strip().splitlines()
    assert lines[0] == "dataset,mode,M,p,d,k,iterations,recall,qps" and len(lines) == 5
