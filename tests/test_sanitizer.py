"""compute-sanitizer over a small run of every kernel family (tensor-core kNN
with resident and streamed query tiles, SIMT kNN, rank optimize, graph
metrics, per-query / lockstep / multi-CTA search in both
distance modes and both visited policies): no memory errors, no shared-memory
races, no illegal barrier use, no uninitialised device reads.

The GPU pool has closed compute-sanitizer (runs under it left GPUs needing a
reset), so these run only when CAGRA_RUN_SANITIZER=1 on a box that allows it;
the round-1 record is profiles/r01_compute_sanitizer.txt.  On the pool the
bounds are covered by the parity tests' guard-zone checks instead."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer_clean(gpu, tool):
    if os.environ.get("CAGRA_RUN_SANITIZER") != "1":
        pytest.skip("compute-sanitizer is closed on the GPU pool; set CAGRA_RUN_SANITIZER=1 to run")
    r = subprocess.run([SAN, "--tool", tool, "--print-limit", "20", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer is closed on this pool")
    assert "sanitize run ok" in out, out[-3000:]
    if tool == "racecheck":
        assert "0 hazards displayed (0 errors, 0 warnings)" in out, out[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
