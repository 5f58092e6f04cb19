import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def restated():
    from oracle.oracle import Restated
    return Restated()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, REF_SO
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def xt():
    import paper_2311_13693_b200 as xt
    return xt


@pytest.fixture(scope="session")
def gpu(xt):
    """The product library with a live B200; fails loudly otherwise."""
    if not xt.device_ready():
        pytest.fail("no usable sm_100 device: GPU tests must run on a B200 (xtsg has no CPU fallback)")
    return xt
