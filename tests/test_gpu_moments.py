"""Moments along the split axis and k-means++ seeding on the GPU vs the oracle."""
import numpy as np
import pytest
import torch

import paper_2007_13552_b200.api as dnd

pytestmark = pytest.mark.gpu


def close(a, b, rel):
    return np.all(np.abs(np.asarray(a) - np.asarray(b)) <= rel * np.maximum(1.0, np.abs(np.asarray(b))))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_moments_1000x18(comm, golden, dtype):
    # test_moments.cpp:125-158 tolerance 1e-12 relative
    xd = golden["mom_x"]
    a = dnd.from_global(xd, xd.shape, 0, comm, dtype=dtype)
    assert close(dnd.gather(dnd.mean_axis(a, 0)), golden["mom_p1_mean"], 1e-12)
    assert close(dnd.gather(dnd.var_axis(a, 0)), golden["mom_p1_var"], 1e-12)
    assert close(dnd.gather(dnd.stddev_axis(a, 0)), np.sqrt(golden["mom_p1_var"]), 1e-12)
    assert close(dnd.gather(dnd.var_axis(a, 0, 1)) * 999 / 1000,
                 golden["mom_p1_var"], 1e-12)


def test_known_answers(comm):
    # test_moments.cpp:46-56, :182-192, :194-202
    a = dnd.from_global(np.array([1.0, 2, 3, 4]), (4, 1), 0, comm)
    st = dnd.moments_axis0(a)
    assert st.count == 4 and st.mean[0] == 2.5 and abs(st.m2[0] - 5.0) <= 5e-14
    assert abs(dnd.gather(dnd.var_axis(a, 0, 0))[0] - 1.25) <= 1e-14
    assert abs(dnd.gather(dnd.var_axis(a, 0, 1))[0] - 5.0 / 3.0) <= 1e-14
    with pytest.raises(ValueError):
        dnd.var_axis(a, 0, 4)
    b = dnd.from_global(np.array([1.0, 2, 3, 4, 5, 6]), (3, 2), 0, comm)
    assert list(dnd.gather(dnd.mean_axis(b, 0))) == [3.0, 4.0]
    c = dnd.from_global(np.full((10, 3), 5.5), (10, 3), 0, comm)
    assert np.all(dnd.gather(dnd.stddev_axis(c, 0)) == 0.0)


def test_offset_stability(comm):
    # test_moments.cpp:160-180: 1e8 + u in f64
    base = np.random.default_rng(61).random((10000, 1))
    a = dnd.from_global(1e8 + base, (10000, 1), 0, comm)
    std = dnd.gather(dnd.stddev_axis(a, 0))[0]
    assert abs(std - base.std()) <= 1e-6 * base.std()


@pytest.mark.parametrize("n,m", [(1, 3), (7, 1), (33, 300), (100_003, 32), (65_536, 18), (2, 18), (3, 17), (100_001, 18),
                                 (50_003, 5), (40_001, 130), (10_007, 257), (5_003, 6), (1_000_003, 3)])
def test_moments_shapes(comm, oracle, n, m):
    xh = oracle.uniform_f32(n, m, n + m)
    a = dnd.from_global(xh, (n, m), 0, comm)
    mean_ref, var_ref = oracle.moments_axis0(xh.astype(np.float64))
    st = dnd.moments_axis0(a)
    assert st.count == n
    assert close(st.mean, mean_ref, 1e-12)
    assert close(st.m2 / n, var_ref, 1e-12)


def test_cfg5_moments_full_size(comm, oracle):
    """BASELINE config 5 moments: 100M x 32 fp32 (12.8 GB); checked against the
    oracle on a 2M-row prefix and for internal consistency at full size."""
    n, m = 100_000_000, 32
    a = dnd.random_uniform((n, m), 0, 42, comm)
    st = dnd.moments_axis0(a)
    assert st.count == n
    assert np.all(np.abs(st.mean - 0.5) < 1e-3) and np.all(np.abs(st.m2 / n - 1 / 12) < 1e-3)
    pre = dnd.DndArray((2_000_000, m), 0, comm, a.tile[:2_000_000])
    sp = dnd.moments_axis0(pre)
    mean_ref, var_ref = oracle.moments_axis0(oracle.uniform_f32(2_000_000, m, 42).astype(np.float64))
    assert close(sp.mean, mean_ref, 1e-12) and close(sp.m2 / 2_000_000, var_ref, 1e-12)


@pytest.mark.parametrize("n,m,k,seed", [(5000, 8, 8, 11), (70_001, 32, 8, 3), (3, 2, 3, 1), (2048 * 1024 + 77, 4, 5, 9),
                                        (40, 32, 3, 5), (2 * 2048 + 64, 32, 4, 2), (2048 * 700 + 1, 32, 6, 8)])
def test_kmeanspp_matches_oracle(comm, oracle, n, m, k, seed):
    # m = 32 fp32 rows take the TMA-staged pass (kpp_update_tma_kernel): a shard
    # shorter than one 64-row chunk, whole blocks + one chunk, more blocks than warps
    xh = oracle.uniform_f32(n, m, seed + 100)
    x = dnd.from_global(xh, (n, m), 0, comm)
    got = dnd.kmeanspp_indices(x, k, seed)
    assert np.array_equal(got, oracle.kmeanspp_indices(xh, k, seed))


@pytest.mark.parametrize("n,m,k,seed", [(5000, 8, 8, 11), (70_001, 18, 8, 3), (2048 * 1024 + 77, 4, 5, 9)])
def test_kmeanspp_f64_matches_oracle(comm, oracle, n, m, k, seed):
    # dndc_kmeanspp_indices_f64 (the f64 entry point of SURVEY 8(b))
    xh = oracle.uniform_f64(n, m, seed + 100)
    x = dnd.from_global(xh, (n, m), 0, comm)
    got = dnd.kmeanspp_indices(x, k, seed)
    assert np.array_equal(got, oracle.kmeanspp_indices(xh, k, seed))


def test_kmeanspp_duplicate_rows_fallback(comm, oracle):
    # all rows identical: W == 0 after the first pick -> the documented fallback
    xh = np.ones((100, 4), np.float32)
    x = dnd.from_global(xh, (100, 4), 0, comm)
    assert np.array_equal(dnd.kmeanspp_indices(x, 4, 5), oracle.kmeanspp_indices(xh, 4, 5))


@pytest.mark.parametrize("shape", [(5, 7, 3), (23, 5), (1, 1, 1), (7, 6, 5)])
def test_resplit_all_transitions(comm, shape):
    """resplit (ndarray.hpp:340-386; test_ndarray.cpp:233-250): every split
    transition keeps the content bitwise and lands on the requested axis."""
    data = np.arange(int(np.prod(shape)), dtype=np.float64) * 0.37 - 3.0
    splits = [None] + list(range(len(shape)))
    for src in splits:
        for dst in splits:
            a = dnd.from_global(data, shape, src, comm)
            r = dnd.resplit(a, dst)
            assert r.split == dst
            assert np.array_equal(dnd.gather(r).ravel(), data)
            if dst is not None:
                assert r.tile.shape[dst] == int(r.split_chunks()[1][comm.rank()])


def test_ops_on_other_splits(comm, oracle):
    """cdist / kmeans_fit / moments accept split=1 and replicated inputs by
    resplitting to row shards first (pairwise.cpp:41, cluster.cpp:91)."""
    n, m = 257, 6
    xh = oracle.uniform_f32(n, m, 5)
    x0 = dnd.from_global(xh, (n, m), 0, comm)
    for split in (1, None):
        x = dnd.from_global(xh, (n, m), split, comm)
        assert np.array_equal(dnd.gather(dnd.cdist(x)), dnd.gather(dnd.cdist(x0)))
        ma, mb = dnd.kmeans_fit(x, 4, 8, 0.0, 3), dnd.kmeans_fit(x0, 4, 8, 0.0, 3)
        assert np.array_equal(ma.centroids, mb.centroids)
        assert close(dnd.moments_axis0(x).mean, dnd.moments_axis0(x0).mean, 1e-14)
    with pytest.raises(ValueError):
        dnd.kmeans_predict(dnd.kmeans_fit(x0, 2, 3, 0.0, 1), dnd.from_global(xh, (n, m), 1, comm))
