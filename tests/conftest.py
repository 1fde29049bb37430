import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs the product path through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    import oracle
    oracle.build(ref=False)
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        if os.path.isdir("/root/reference/proj/include"):
            oracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return oracle.Ref()


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(GOLDEN, "golden.npz")
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture(scope="session")
def fd():
    """The product package; on a GPU box the CUDA library must load."""
    import paper_2406_13984_b200 as fd
    fd.featdrive.lib()
    return fd
