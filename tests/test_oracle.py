"""Pins the oracle (oracle/dnd_oracle.c) before it is trusted as the checker.

Against (a) the reference's own known answers (tests/test_*.cpp fixtures),
(b) golden vectors written by the unmodified reference (tests/golden, made by
make_golden.py through oracle/_ref), and (c) the live reference library when
oracle/_ref is built here.  Everything is bit-exact: the oracle restates the
reference's operation order.
"""
import numpy as np
import pytest


def test_uniform_matches_reference_golden(oracle, golden):
    # ndarray.hpp:154-169 via common.hpp:14-27; split/rank-independent content
    assert np.array_equal(oracle.uniform_f32(4096, 18, 42).view(np.uint32),
                          golden["uniform_18_s42_head"].view(np.uint32))
    assert np.array_equal(oracle.uniform_f32(1024, 32, 7).view(np.uint32),
                          golden["uniform_32_s7_head"].view(np.uint32))
    # a shard starting at row0 is the same slice of the global array
    full = oracle.uniform_f32(100, 18, 42)
    assert np.array_equal(oracle.uniform_f32(40, 18, 42, row0=33), full[33:73])


def test_splitmix_known_answer(oracle):
    # splitmix64(0) is the published first output of the SplitMix64 generator
    assert oracle.lib.dno_splitmix64(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("n,p", [(5, 3), (3, 5), (5_000_000, 8), (200_000, 3), (100_000_000, 8)])
def test_chunk_map(oracle, golden, n, p):
    off, ext = oracle.chunk_map(n, p)
    assert np.array_equal(np.stack([off, ext]), golden[f"chunk_{n}_{p}"])
    assert ext.sum() == n and ext.max() - ext.min() <= 1


def test_chunk_map_known_answer(oracle):
    # test_chunking.cpp:10-14 / acceptance.cpp:62-63
    off, ext = oracle.chunk_map(5, 3)
    assert list(ext) == [2, 2, 1] and list(off) == [0, 2, 4]
    with pytest.raises(ValueError):
        oracle.chunk_map(5, 0)


def test_cdist_golden(oracle, golden):
    x = golden["cdist_x"]
    assert np.array_equal(oracle.row_norms(x), golden["row_norms_x"])
    assert np.array_equal(oracle.cdist(x, 1), golden["cdist_p1"])
    assert np.array_equal(oracle.cdist(x, 3), golden["cdist_p3"])
    assert np.array_equal(oracle.cdist_xy(x, golden["cdist_y"]), golden["cdist_xy"])
    assert int(golden["cdist_p3_sendrecvs"][0]) == 2  # p - 1 ring exchanges


def test_cdist_known_answers(oracle):
    # test_pairwise.cpp:23-28: the 3-4-5 triangle, exactly
    assert np.array_equal(oracle.cdist(np.array([[0.0, 0.0], [3.0, 4.0]]), 2), [[0, 5], [5, 0]])
    # :16-21 repeated rows -> all zero
    x = np.tile(np.array([[1.0, 2.0, 3.0]]), (5, 1))
    assert np.all(oracle.cdist(x, 3) == 0.0)
    # :116-133 distance to a zero row is the row norm
    x = np.random.default_rng(89).random((17, 4))
    d = oracle.cdist_xy(x, np.zeros((1, 4)))
    assert np.allclose(d[:, 0], np.sqrt((x * x).sum(1)), rtol=1e-12, atol=0)
    # :135-144 cdist_xy(x, x) == cdist(x) bitwise on one rank
    x = np.random.default_rng(97).random((25, 6))
    assert np.array_equal(oracle.cdist_xy(x, x), oracle.cdist(x, 1))
    with pytest.raises(ValueError):
        oracle.cdist(np.zeros((0, 3)))


@pytest.mark.parametrize("n,k,s", [(100, 8, 21), (6, 6, 77), (5_000_000, 8, 42), (100_000_000, 8, 42),
                                   (50_000_000, 64, 42)])
def test_init_indices_golden(oracle, golden, n, k, s):
    assert np.array_equal(oracle.kmeans_init_indices(n, k, s), golden[f"init_{n}_{k}_{s}"])


def test_init_indices_properties(oracle):
    # test_cluster.cpp:195-219
    assert sorted(oracle.kmeans_init_indices(6, 6, 77)) == list(range(6))
    a = oracle.kmeans_init_indices(100, 8, 21)
    assert np.array_equal(a, oracle.kmeans_init_indices(100, 8, 21))
    assert not np.array_equal(a, oracle.kmeans_init_indices(100, 8, 22))
    with pytest.raises(ValueError):
        oracle.kmeans_init_indices(3, 4, 1)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_kmeans_golden(oracle, golden, p):
    c, t, it = oracle.kmeans_fit(golden["km600_x"], 8, 30, 0.0, 42, p)
    assert it == 30
    assert np.array_equal(c, golden[f"km600_p{p}_centroids"])
    assert np.array_equal(t, golden[f"km600_p{p}_trace"])


def test_kmeans_tol_and_predict_golden(oracle, golden):
    x = golden["km600_x"]
    c, t, it = oracle.kmeans_fit(x, 8, 100, 1e-3, 42, 3)
    assert it == int(golden["km600_tol_iters"][0])
    assert np.array_equal(c, golden["km600_tol_centroids"])
    assert np.array_equal(t, golden["km600_tol_trace"])
    assert np.array_equal(oracle.kmeans_predict(x, golden["km600_p1_centroids"]), golden["km600_labels"])


def test_kmeans_known_answers(oracle):
    # test_cluster.cpp:221-241 own labels and the tie rule
    x = np.array([[0, 0], [5, 5], [9, 0]], np.float64)
    assert list(oracle.kmeans_predict(x, x)) == [0, 1, 2]
    assert list(oracle.kmeans_predict(np.array([[1.0]]), np.array([[0.0], [2.0]]))) == [0]
    # :275-283 more ranks than samples
    c, _, _ = oracle.kmeans_fit(np.array([[0.0], [0.1], [10.0]]), 2, 4, 0.0, 7, 5)
    assert abs(min(c[:, 0]) - 0.05) <= 1e-12 and abs(max(c[:, 0]) - 10.0) <= 1e-12
    # :119-132 k = 1 is the global mean after one iteration
    x = np.random.default_rng(107).random((50, 4))
    c, _, _ = oracle.kmeans_fit(x, 1, 1, 0.0, 9, 2)
    assert np.allclose(c[0], x.mean(0), rtol=1e-12, atol=0)
    # :292-300 non-finite input
    with pytest.raises(ValueError):
        oracle.kmeans_fit(np.array([[1.0, 2.0], [np.nan, 4.0]]), 1, 5, 0.0, 1, 2)


@pytest.mark.parametrize("p", [1, 3, 5])
def test_moments_golden(oracle, golden, p):
    mean, var = oracle.moments_axis0(golden["mom_x"], p)
    assert np.array_equal(mean, golden[f"mom_p{p}_mean"])
    assert np.array_equal(var, golden[f"mom_p{p}_var"])
    _, var1 = oracle.moments_axis0(golden["mom_x"], 2, 1)
    assert np.array_equal(var1, golden["mom_p2_ddof1_var"])


def test_moments_known_answers(oracle):
    # test_moments.cpp:46-56 and :182-192
    c, mean, m2 = oracle.local_moments_axis0(np.array([[1.0], [2.0], [3.0], [4.0]]))
    assert c == 4 and mean[0] == 2.5 and abs(m2[0] - 5.0) <= 5e-14
    _, v0 = oracle.moments_axis0(np.array([[1.0], [2.0], [3.0], [4.0]]), 2, 0)
    _, v1 = oracle.moments_axis0(np.array([[1.0], [2.0], [3.0], [4.0]]), 2, 1)
    assert abs(v0[0] - 1.25) <= 1e-14 and abs(v1[0] - 5.0 / 3.0) <= 1e-14
    with pytest.raises(ValueError):
        oracle.moments_axis0(np.array([[1.0], [2.0], [3.0], [4.0]]), 2, 4)
    # :160-180 the 1e8 offset: Welford keeps the spread
    base = np.random.default_rng(61).random((10000, 1))
    _, var = oracle.moments_axis0(1e8 + base, 3)
    assert abs(np.sqrt(var[0]) - base.std()) <= 1e-6 * base.std()


def test_oracle_matches_live_reference(oracle, reference):
    rng = np.random.default_rng(5)
    x = rng.random((150, 10))
    for p in (1, 4):
        assert np.array_equal(oracle.cdist(x, p), reference.cdist(x, p)[0])
    c1, t1, i1 = oracle.kmeans_fit(x, 5, 12, 0.0, 17, 3)
    c2, t2, i2 = reference.kmeans_fit(x, 5, 12, 0.0, 17, 3)
    assert i1 == i2 and np.array_equal(c1, c2) and np.array_equal(t1, t2)
    m1, v1 = oracle.moments_axis0(x, 4)
    m2, v2 = reference.moments_axis0(x, 4)
    assert np.array_equal(m1, m2) and np.array_equal(v1, v2)


def test_kmeanspp_oracle_properties(oracle):
    # the repo's own definition: deterministic, distinct picks,
    # first pick = kmeans_init_indices(n, 1, seed)
    x = oracle.uniform_f32(5000, 8, 3)
    a = oracle.kmeanspp_indices(x, 8, 11)
    assert np.array_equal(a, oracle.kmeanspp_indices(x, 8, 11))
    assert len(set(a.tolist())) == 8
    assert a[0] == oracle.kmeans_init_indices(5000, 1, 11)[0]
    # rank layout changes the summation blocks only
    assert len(set(oracle.kmeanspp_indices(x, 8, 11, p=3).tolist())) == 8
    # the f64 entry point runs the same chain on the doubles: f32-valued rows
    # give the same picks, other doubles a valid distinct set
    assert np.array_equal(oracle.kmeanspp_indices(x.astype(np.float64), 8, 11), a)
    x64 = oracle.uniform_f64(5000, 8, 3)
    assert len(set(oracle.kmeanspp_indices(x64, 8, 11).tolist())) == 8


def _lasso_problem(n, m, seed):
    rng = np.random.default_rng(seed)
    x = np.hstack([np.ones((n, 1)), rng.normal(size=(n, m - 1))])
    y = x @ rng.normal(size=m) + 0.1 * rng.normal(size=n)
    return x, y


@pytest.mark.parametrize("n,m,lam,sweeps,tol,p", [(301, 7, 2.0, 30, 0.0, 1), (301, 7, 2.0, 30, 0.0, 3),
                                                   (120, 8, 1e4, 5, 0.0, 2), (200, 12, 30.0, 500, 1e-12, 3),
                                                   (3, 2, 0.0, 50, 1e-15, 5)])
def test_lasso_oracle_matches_reference(oracle, reference, n, m, lam, sweeps, tol, p):
    """F4: the C restatement of lasso_fit (regression.cpp:25-102) is bit-exact
    with the compiled reference, every rank count, tol stop included."""
    x, y = _lasso_problem(n, m, n + m)
    a, b = oracle.lasso_fit(x, y, lam, sweeps, tol, p), reference.lasso_fit(x, y, lam, sweeps, tol, p)
    assert a[2] == b[2]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_lasso_oracle_edge_cases(oracle):
    """soft_threshold hand values, zero column skipped, bias column enforced
    (test_regression.cpp:83-89, :172-179, :214-230)."""
    st = oracle.lib.dno_soft_threshold
    assert (st(0.5, 1.0), st(2.0, 0.5), st(-2.0, 0.5), st(0.0, 0.0), st(3.0, 0.0)) == (0.0, 1.5, -1.5, 0.0, 3.0)
    x, y = _lasso_problem(40, 6, 167)
    x[:, 3] = 0.0
    w, trace, _ = oracle.lasso_fit(x, y, 0.5, 50, 0.0, 2)
    assert w[3] == 0.0 and np.all(np.diff(trace) <= 1e-9)
    x[5, 0] = 2.0
    with pytest.raises(ValueError):
        oracle.lasso_fit(x, y, 0.5, 5)
