import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "ref: needs the reference build oracle/_ref/libktune_ref.so")


@pytest.fixture(scope="session")
def O():
    """The oracle (test infrastructure): C restatement + reference build."""
    from oracle import pyoracle
    if not os.path.exists(pyoracle.PORT_SO) or (os.path.isdir("/root/reference") and not pyoracle.ref_available()):
        pyoracle.build()
    return pyoracle


@pytest.fixture(scope="session")
def ref_ok(O):
    if not O.ref_available():
        pytest.skip("reference build oracle/_ref not available")
    return True


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_08743_b200.context import Context
    return Context(0)


def rng(seed):
    return np.random.default_rng(seed)
