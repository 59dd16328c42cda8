import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    r = oracle.reference()
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    return r


@pytest.fixture(scope="session")
def stk():
    from paper_2001_07809_b200 import stereotk

    return stereotk


@pytest.fixture(scope="session")
def synth():
    from paper_2001_07809_b200 import synth

    return synth


@pytest.fixture(scope="session")
def dev():
    """The B200 context.  GPU tests must fail (not skip) without it."""
    from paper_2001_07809_b200 import stereotk

    d = stereotk.Device(0, slots=3)
    yield d
    d.close()
