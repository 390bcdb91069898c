"""cdist / cdist_xy / row_norms on the GPU vs the oracle.

Mirrors tests/test_pairwise.cpp of the reference case by case.  f64 inputs go
through the bit-exact f64 kernels (tolerances as in the reference tests, most
of them exact); f32 inputs go through the FFMA performance kernel and are held
to BASELINE.json's 1e-5 relative gate (|a-b| / max(1, |ref|), verify.cpp:24-28).
"""
import numpy as np
import pytest
import torch

import paper_2007_13552_b200.api as dnd
from _parity import rel_dev

pytestmark = pytest.mark.gpu


def test_generator_is_bit_identical(comm, oracle):
    for (n, m, seed) in [(4096, 18, 42), (1000, 32, 7), (333, 5, 1)]:
        a = dnd.random_uniform((n, m), 0, seed, comm)
        assert np.array_equal(a.tile.cpu().numpy().view(np.uint32), oracle.uniform_f32(n, m, seed).view(np.uint32))
        b = dnd.random_uniform((n, m), 0, seed, comm, dtype=torch.float64)
        assert np.array_equal(b.tile.cpu().numpy(), oracle.uniform_f64(n, m, seed))


def test_generator_full_cfg1_checksum(comm, golden):
    # the first 4096 rows of the 5M x 18 cfg1 array, generated at full size
    a = dnd.random_uniform((5_000_000, 18), 0, 42, comm)
    assert np.array_equal(a.tile[:4096].cpu().numpy().view(np.uint32), golden["uniform_18_s42_head"].view(np.uint32))


def test_repeated_rows_have_zero_distances(comm):
    # test_pairwise.cpp:16-21
    x = dnd.from_global(np.tile([1.0, 2.0, 3.0], 5), (5, 3), 0, comm, dtype=torch.float32)
    assert np.all(dnd.gather(dnd.cdist(x)) == 0.0)
    x64 = dnd.from_global(np.tile([1.0, 2.0, 3.0], 5), (5, 3), 0, comm)
    assert np.all(dnd.gather(dnd.cdist(x64)) == 0.0)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_three_four_five_triangle(comm, dtype):
    # test_pairwise.cpp:23-28, exact
    x = dnd.from_global([0.0, 0.0, 3.0, 4.0], (2, 2), 0, comm, dtype=dtype)
    assert np.array_equal(dnd.gather(dnd.cdist(x)), np.array([[0, 5], [5, 0]]))


def test_cdist_f64_is_bit_exact(comm, golden):
    # test_pairwise.cpp:30-45 (1e-8 there; the f64 kernel reproduces the
    # reference's operation order, so the golden matrix is matched bitwise)
    x = dnd.from_global(golden["cdist_x"], golden["cdist_x"].shape, 0, comm)
    assert np.array_equal(dnd.gather(dnd.cdist(x)), golden["cdist_p1"])
    assert np.array_equal(dnd.row_norms(x.tile).cpu().numpy(), golden["row_norms_x"])
    y = dnd.from_global(golden["cdist_y"], golden["cdist_y"].shape, None, comm)
    assert np.array_equal(dnd.gather(dnd.cdist_xy(x, y)), golden["cdist_xy"])


def test_cdist_xy_split_y_f64_is_bit_exact(comm, golden):
    # y split=0 in f64: the device ring (dndc_cdist_xy_ring_f64) instead of the
    # reference's allgather (pairwise.cpp:94); same bits as y replicated
    x = dnd.from_global(golden["cdist_x"], golden["cdist_x"].shape, 0, comm)
    y = dnd.from_global(golden["cdist_y"], golden["cdist_y"].shape, 0, comm)
    assert np.array_equal(dnd.gather(dnd.cdist_xy(x, y)), golden["cdist_xy"])


def test_cdist_f32_within_gate(comm, golden):
    xd = golden["cdist_x"]  # fp32-valued data widened to f64
    x = dnd.from_global(xd, xd.shape, 0, comm, dtype=torch.float32)
    d = dnd.gather(dnd.cdist(x))
    assert rel_dev(d, golden["cdist_p1"]) <= 1e-5
    assert np.all(np.diag(d) == 0.0) and np.all(d >= 0.0)
    y = dnd.from_global(golden["cdist_y"], golden["cdist_y"].shape, None, comm, dtype=torch.float32)
    assert rel_dev(dnd.gather(dnd.cdist_xy(x, y)), golden["cdist_xy"]) <= 1e-5


@pytest.mark.parametrize("n,m", [(1, 1), (3, 2), (129, 18), (255, 7), (1000, 33), (600, 64), (300, 130)])
def test_cdist_f32_shapes(comm, oracle, n, m):
    # ragged tiles (not multiples of 128), feature counts across the K-chunking
    xh = oracle.uniform_f32(n, m, 1000 + n)
    x = dnd.from_global(xh, (n, m), 0, comm)
    d = dnd.gather(dnd.cdist(x))
    ref = oracle.cdist(xh.astype(np.float64))
    dev = rel_dev(d, ref)
    print(f"cdist f32 n={n} m={m}: rel dev {dev:.3e}")
    assert dev <= 1e-5
    assert np.all(np.diag(d) == 0.0)


@pytest.mark.parametrize("n,ny,m", [(1000, 700, 1024), (333, 129, 260), (128, 300, 256), (517, 517, 1000)])
def test_cdist_tensor_core_path(comm, oracle, n, ny, m):
    # m >= 256: the tcgen05 3xTF32 kernel (cdist_tc.cu).  Duplicate rows must
    # cancel to exactly 0 as in the reference (norms come from the same MMA path).
    xh = oracle.uniform_f32(n, m, 2000 + n)
    xh[5] = xh[77]
    yh = oracle.uniform_f32(ny, m, 3000 + ny)
    yh[3] = xh[9]
    x = dnd.from_global(xh, (n, m), 0, comm)
    y = dnd.from_global(yh, (ny, m), None, comm)
    tol = 1e-5  # BASELINE's distance gate, independent of m
    d = dnd.gather(dnd.cdist(x))
    dev = rel_dev(d, oracle.cdist(xh.astype(np.float64)))
    print(f"cdist tc n={n} ny={ny} m={m}: self rel dev {dev:.3e}")
    assert dev <= tol
    assert np.all(np.diag(d) == 0.0) and d[5, 77] == 0.0 and d[77, 5] == 0.0
    dxy = dnd.gather(dnd.cdist_xy(x, y))
    dev = rel_dev(dxy, oracle.cdist_xy(xh.astype(np.float64), yh.astype(np.float64)))
    print(f"cdist tc n={n} ny={ny} m={m}: xy rel dev {dev:.3e}")
    assert dev <= tol
    assert dxy[9, 3] == 0.0


def test_metric_axioms(comm, oracle):
    # test_pairwise.cpp:60-82 (60 x 7): zero diagonal, >= 0, symmetry, triangle
    xh = oracle.uniform_f32(60, 7, 79)
    d = dnd.gather(dnd.cdist(dnd.from_global(xh, (60, 7), 0, comm)))
    assert np.all(np.diag(d) == 0.0) and np.all(d >= 0.0)
    assert np.max(np.abs(d - d.T)) <= 1e-6
    rng = np.random.default_rng(83)
    for _ in range(200):
        i, j, k = rng.integers(0, 60, 3)
        assert d[i, j] <= d[i, k] + d[k, j] + 1e-5


def test_distances_to_zero_row_are_norms(comm, oracle):
    # test_pairwise.cpp:116-133
    xh = oracle.uniform_f32(17, 4, 89).astype(np.float64)
    x = dnd.from_global(xh, (17, 4), 0, comm)
    y = dnd.from_global(np.zeros(4), (1, 4), None, comm)
    d = dnd.gather(dnd.cdist_xy(x, y))[:, 0]
    assert np.allclose(d, np.sqrt((xh * xh).sum(1)), rtol=1e-12, atol=0)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_cdist_xy_self_equals_cdist_bitwise(comm, oracle, dtype):
    # test_pairwise.cpp:135-144: the f32 norm chain equals the dot chain, so
    # the diagonal cancels to exactly 0 and the matrices are identical
    xh = oracle.uniform_f32(25, 6, 97)
    x = dnd.from_global(xh, (25, 6), 0, comm, dtype=dtype)
    y = dnd.from_global(xh, (25, 6), None, comm, dtype=dtype)
    assert np.array_equal(dnd.gather(dnd.cdist_xy(x, y)), dnd.gather(dnd.cdist(x)))


def test_cdist_xy_is_communication_free(comm, oracle):
    # test_pairwise.cpp:146-166
    xh = oracle.uniform_f32(100, 5, 101)
    yh = oracle.uniform_f32(8, 5, 102)
    x = dnd.from_global(xh, (100, 5), 0, comm)
    y = dnd.from_global(yh, (8, 5), None, comm)
    before = comm.counters()
    d = dnd.gather(dnd.cdist_xy(x, y))
    after = comm.counters()
    assert after == before
    assert rel_dev(d, oracle.cdist_xy(xh.astype(np.float64), yh.astype(np.float64))) <= 1e-5


def test_cdist_validation(comm):
    # test_pairwise.cpp:107-114, :168-174
    with pytest.raises(ValueError):
        dnd.cdist(dnd.from_global(np.zeros((0, 3)), (0, 3), 0, comm))
    x = dnd.from_global(np.zeros((4, 3)), (4, 3), 0, comm)
    y = dnd.from_global(np.zeros((2, 2)), (2, 2), None, comm)
    with pytest.raises(ValueError):
        dnd.cdist_xy(x, y)


def test_tile_column_window_and_diag_offset(comm, oracle):
    # distance_block + place_chunk: write a window of a wider row block
    xh = oracle.uniform_f32(50, 18, 5)
    yh = oracle.uniform_f32(70, 18, 6)
    x = torch.from_numpy(xh).cuda()
    y = torch.from_numpy(yh).cuda()
    out = torch.full((50, 203), -1.0, device="cuda")
    from paper_2007_13552_b200 import _lib

    xn, yn = dnd.row_norms(x), dnd.row_norms(y)
    _lib.check(_lib.lib().dndc_cdist_tile_f32(comm.handle, x.data_ptr(), xn.data_ptr(), 50, y.data_ptr(),
                                              yn.data_ptr(), 70, 18, out.data_ptr(), 203, 61, 3))
    o = out.cpu().numpy()
    ref = oracle.cdist_xy(xh.astype(np.float64), yh.astype(np.float64))
    assert np.all(o[:, :61] == -1.0) and np.all(o[:, 131:] == -1.0)
    win = o[:, 61:131]
    for i in range(50):
        if i + 3 < 70:
            assert win[i, i + 3] == 0.0
            win[i, i + 3] = ref[i, i + 3]
    assert rel_dev(win, ref) <= 1e-5


@pytest.mark.slow
def test_cfg2_panels_full_size(comm, oracle):
    """BASELINE config 2 at full size on one GPU: X(200k x 18) vs Y(200k x 18)
    = 160 GB of fp32 output; sampled row panels checked against the oracle,
    plus on-device non-negativity and a checksum of the full matrix."""
    n, m = 200_000, 18
    free = torch.cuda.mem_get_info()[0]
    if free < n * n * 4 + (2 << 30):
        pytest.skip("not enough HBM for the 160 GB output")
    x = dnd.random_uniform((n, m), 0, 42, comm)
    y = dnd.random_uniform((n, m), 0, 43, comm)
    d = dnd.cdist_xy(x, dnd.DndArray((n, m), None, comm, y.tile))
    rows = np.array([0, 1, 12345, 99_999, 150_001, n - 1])
    xh = oracle.uniform_f32(n, m, 42)
    yh = oracle.uniform_f32(n, m, 43).astype(np.float64)
    ref = oracle.cdist_xy(xh[rows].astype(np.float64), yh)
    got = d.tile[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert rel_dev(got, ref) <= 1e-5
    assert float(d.tile.min()) >= 0.0
    del d
    torch.cuda.empty_cache()
