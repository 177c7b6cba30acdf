"""Test helpers (shared by the test modules)."""
import numpy as np


def cfg(**kw):
    from paper_2507_04610_b200 import _abi

    return _abi.default_config(**kw)


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype == np.float32:
        return np.array_equal(a.view(np.uint32), b.view(np.uint32))
    return np.array_equal(a, b)
