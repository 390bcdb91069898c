"""F4 LASSO on the GPU (dndc_lasso_fit_f64) against the oracle restatement of
regression.cpp:25-102, itself pinned bit-exact to the compiled reference in
tests/test_oracle.py.  Tolerance: weights 1e-9 relative, objective 1e-10
relative (the GPU sums rho over CTAs in a fixed tree, the reference in row
order); predict is bit-exact."""
import numpy as np
import pytest
import torch

import paper_2007_13552_b200.api as dnd

pytestmark = pytest.mark.gpu


def problem(n, m, seed):
    rng = np.random.default_rng(seed)
    x = np.hstack([np.ones((n, 1)), rng.normal(size=(n, m - 1))])
    y = x @ rng.normal(size=m) + 0.1 * rng.normal(size=n)
    return x, y


def rel_ok(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b)))


@pytest.mark.parametrize("n,m,lam,sweeps", [(301, 7, 2.0, 30), (5000, 18, 50.0, 40), (120, 8, 1e4, 5),
                                            (200, 12, 0.0, 60), (1, 1, 0.0, 3), (100_003, 33, 5.0, 10)])
def test_lasso_matches_oracle(comm, oracle, n, m, lam, sweeps):
    x, y = problem(n, m, n + m)
    w_ref, t_ref, run_ref = oracle.lasso_fit(x, y, lam, sweeps)
    model = dnd.lasso_fit(dnd.from_global(x, x.shape, 0, comm), dnd.from_global(y, y.shape, 0, comm), lam, sweeps)
    assert model.sweeps_run == run_ref
    assert rel_ok(model.weights, w_ref, 1e-9)
    assert rel_ok(model.objective_trace, t_ref, 1e-10)


def test_lasso_tol_stop_and_zero_column(comm, oracle):
    x, y = problem(2000, 9, 5)
    x[:, 4] = 0.0
    w_ref, t_ref, run_ref = oracle.lasso_fit(x, y, 1.0, 500, 1e-10)
    model = dnd.lasso_fit(dnd.from_global(x, x.shape, 0, comm), dnd.from_global(y, y.shape, 0, comm), 1.0, 500,
                          1e-10)
    assert model.sweeps_run == run_ref < 500
    assert model.weights[4] == 0.0 and rel_ok(model.weights, w_ref, 1e-9)


def test_lasso_predict_bit_exact_and_validation(comm):
    x, y = problem(1000, 6, 9)
    xa = dnd.from_global(x, x.shape, 0, comm)
    model = dnd.LassoModel(np.linspace(-1.0, 2.0, 6))
    got = dnd.gather(dnd.lasso_predict(model, xa))
    want = np.zeros(1000)
    for j in range(6):  # row loop in column order, products rounded first
        want = want + x[:, j] * model.weights[j]
    assert np.array_equal(got, want)
    bad = x.copy()
    bad[7, 0] = 0.5
    with pytest.raises(ValueError, match="bias"):
        dnd.lasso_fit(dnd.from_global(bad, bad.shape, 0, comm), dnd.from_global(y, y.shape, 0, comm), 1.0, 3)
    with pytest.raises(ValueError):
        dnd.lasso_fit(xa, dnd.from_global(y[:-1], (999,), 0, comm), 1.0, 3)
    with pytest.raises(ValueError):
        dnd.lasso_fit(xa, dnd.from_global(y, y.shape, 0, comm), -1.0, 3)
