"""Self-tests of the tcgen05 / TMA plumbing (csrc/tc.cuh via csrc/tcprobe.cu).

These pin the descriptor formats and the numeric behaviour of kind::tf32 MMAs
that the tensor-core kernels rely on (which fp32 bits the tensor core uses).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2007_13552_b200 import _lib

pytestmark = pytest.mark.gpu


def probe(mode, a, b, rows=0, cols=0, x=None, out_elems=128 * 16):
    L = _lib.lib()
    fn = L.dndc_internal_tc_probe
    fn.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    fn.restype = C.c_int
    ta = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b, np.float32)).cuda()
    tx = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda() if x is not None else ta
    d = torch.zeros(out_elems, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    _lib.check(fn(mode, ta.data_ptr(), tb.data_ptr(), d.data_ptr(), tx.data_ptr(), rows, cols))
    return d.cpu().numpy()


def tf32_trunc(v):
    return (np.asarray(v, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def test_kmajor_mma_exact_on_tf32_inputs():
    rng = np.random.default_rng(1)
    a = tf32_trunc(rng.random((128, 8)) - 0.5)
    b = tf32_trunc(rng.random((16, 8)) - 0.5)
    d = probe(0, a, b).reshape(128, 16)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert np.max(np.abs(d - ref)) < 1e-6


def test_tf32_input_conversion_is_truncation_or_rounding():
    """Records how the tensor core treats the low 13 mantissa bits of fp32 inputs."""
    rng = np.random.default_rng(2)
    a = (rng.random((128, 8)) + 0.5).astype(np.float32)
    b = np.zeros((16, 8), np.float32)
    b[:8, :8] = np.eye(8, dtype=np.float32)  # D[:, j] = A[:, j]
    d = probe(0, a, b).reshape(128, 16)[:, :8]
    trunc = tf32_trunc(a)
    rn = (a.view(np.uint32).astype(np.uint64) + 0x1000) & 0xFFFFE000
    rn = rn.astype(np.uint32).view(np.float32)
    is_trunc = np.array_equal(d, trunc)
    is_rn = np.array_equal(d, rn)
    print(f"tf32 input conversion: truncation={is_trunc} round-nearest={is_rn}")
    assert is_trunc or is_rn


def test_mn_major_probe_and_tma_layout():
    """MN-major kind::tf32 operands are recorded, not relied on: on this part they
    read back as zeros, so every tensor-core kernel here stages K-major tiles
    ("tensor-core layout").  The TMA box layout is asserted."""
    rng = np.random.default_rng(3)
    results = {}
    for mode, M in ((1, 128), (3, 64), (4, 128), (5, 64)):
        a = tf32_trunc(rng.random((128, 128)) - 0.5)  # [K rows x M cols]
        b = np.zeros((128, 16), np.float32)           # one-hot [K x N]
        lab = rng.integers(0, 16, 128)
        b[np.arange(128), lab] = 1.0
        raw = probe(mode, a, b).reshape(128, 16)      # TMEM lane-major dump
        ref = a[:, :M].astype(np.float64).T @ b.astype(np.float64)  # [M x 16]
        if M == 128:
            got = raw
        else:  # half-subpartition layout: row m0 + 16 m1 lives in lane m0 + 32 m1
            got = np.stack([raw[(m % 16) + 32 * (m // 16)] for m in range(64)])
        results[mode] = float(np.max(np.abs(got - ref)))
    print("MN-major probe errors by mode", results)
    # TMA: [rows x 36] with box {4, 128} -> 10 boxes of 128 x 16 B (OOB zero)
    x = rng.random((300, 36)).astype(np.float32)
    raw = probe(2, np.zeros(4, np.float32), np.zeros(4, np.float32), rows=300, cols=36, x=x, out_elems=10 * 512)
    boxes = raw.reshape(10, 128, 4)
    for c in range(10):
        for r in (0, 1, 77, 127):
            want = x[r, 4 * c: 4 * c + 4] if 4 * c < 36 else np.zeros(4, np.float32)
            assert np.array_equal(boxes[c, r], want), (c, r)
