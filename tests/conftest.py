import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)



def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: multi-second GPU parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import load_oracle

    return load_oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference, or None when oracle/_ref was not built here."""
    from oracle.bindings import load_reference

    return load_reference()


@pytest.fixture(scope="session")
def gpu():
    """GPU tests fail loudly (never skip) when the engine or device is missing."""
    from paper_2308_15136_b200 import capi

    capi.lib()
    n = capi.device_count()
    assert n > 0, "no CUDA device visible: GPU tests must run on the B200 box"
    return n
