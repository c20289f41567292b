"""compute-sanitizer over a small run of every kernel family (tensor-core kNN
with resident and streamed query tiles, SIMT kNN, rank optimize, graph
metrics, per-query / lockstep / multi-CTA search in both
distance modes and both visited policies): no memory errors, no shared-memory
races, no illegal barrier use, no uninitialised device reads."""
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
    r = subprocess.run([SAN, "--tool", tool, "--print-limit", "20", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "sanitize run ok" in out, out[-3000:]
    if tool == "racecheck":
        assert "0 hazards displayed (0 errors, 0 warnings)" in out, out[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
