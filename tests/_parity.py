"""Parity metric shared by the tests (tools/verify.cpp:20-33)."""
import numpy as np


def rel_dev(a, ref):
    """max |a - ref| / max(1, |ref|)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - ref) / np.maximum(1.0, np.abs(ref))))
