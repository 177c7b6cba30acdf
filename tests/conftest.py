import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def orc():
    """The C restatement oracle (test infrastructure)."""
    from oracle.refpy import oracle

    return oracle()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference build (oracle/_ref), skipped when absent."""
    from oracle.refpy import have_ref, ref as _ref

    if not have_ref():
        pytest.skip("oracle/_ref/libanyq_ref.so not built")
    return _ref()


@pytest.fixture(scope="session")
def aq():
    """The product API (CUDA library). Fails loudly if it is not built."""
    from paper_2507_04610_b200 import anyq

    anyq.lib()
    return anyq


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test requires a CUDA device")
    return torch
