"""The C++ drop-in's own behaviour beyond the reference's suites
(tests/cpp/*.cpp, built by `make dropintests`): the device-index cache never
serves a stale copy after an in-place edit (content check by default;
explicit invalidation with CAGRA_INDEX_CACHE=identity)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_dropin_index_cache_sees_in_place_edits(gpu):
    exe = os.path.join(ROOT, "tests", "_dropin", "test_dropin_cache")
    assert os.path.exists(exe), "run `make dropintests`"
    env = {k: v for k, v in os.environ.items() if k != "CAGRA_INDEX_CACHE"}
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
