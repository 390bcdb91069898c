"""Parity metric shared by the tests (tools/verify.cpp:20-33)."""
import numpy as np


def rel_dev(a, ref):
    """max |a - ref| / max(1, |ref|)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - ref) / np.maximum(1.0, np.abs(ref))))


def label_digest(labels):
    """Order-sensitive 64-bit digest of an int label vector, so the labels of a
    5M-row reference run fit in a small committed fixture: sum over rows of
    (label + 1) * w_i mod 2^64 with w_i = splitmix-style odd weights."""
    lab = np.asarray(labels, np.int64).astype(np.uint64) + np.uint64(1)
    i = np.arange(lab.size, dtype=np.uint64)
    w = (i * np.uint64(0x9E3779B97F4A7C15)) ^ (i >> np.uint64(7))
    w |= np.uint64(1)
    with np.errstate(over="ignore"):
        return int(np.sum(lab * w, dtype=np.uint64))
