import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: larger parity cases")


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def golden_names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


LEVEL_NAMES = ["rd", "cd", "rdd", "cdd", "rqd", "cqd"]


def level_from_name(name):
    """'cdd' -> product PrecisionLevel(dd, complex)"""
    from paper_1402_2626_b200.xprec import precision_level
    return precision_level(name[1:], name[0] == "c")


def oracle_level(name):
    import oracle
    return oracle.Level(name[1:], name[0] == "c")


def same(a, b):
    """Component-wise equality (np.array_equal: == on every component, so
    +0.0 == -0.0 as in the reference's own bit-identity tests)."""
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b)


@pytest.fixture(scope="session")
def gpu():
    from paper_1402_2626_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("GPU test ran without a CUDA device")
    return True
