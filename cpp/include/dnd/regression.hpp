// dnd/regression.hpp -- B200 drop-in for proj/include/dnd/regression.hpp
// (regression.cpp:19-127): LASSO by cyclic coordinate descent on the HBM
// shards, one kernel per coordinate with the cross-GPU scalar sum done over
// NVLink inside it (dndc_lasso_fit_f64); predict is bit-identical.
#pragma once

#include <vector>

#include "dnd/ndarray.hpp"

namespace dnd {

/// weights[0] is the unpenalised bias (all-ones column 0); objective_trace
/// holds |y - Xw|^2 + lambda |w_1..|_1 once per sweep (regression.hpp:10-19).
struct LassoModel {
    std::vector<double> weights;
    double lambda = 0.0;
    std::vector<double> objective_trace;
    int sweeps_run = 0;
};

/// sign(rho) max(|rho| - threshold, 0) (regression.cpp:19-23).
inline double soft_threshold(double rho, double threshold) {
    if (rho > threshold) return rho - threshold;
    if (rho < -threshold) return rho + threshold;
    return 0.0;
}

/// Cyclic coordinate descent (regression.cpp:25-102).  x: n x m with the
/// all-ones first column, y: n targets; other layouts are resplit to row
/// shards first.  The bias check raises on every rank.
inline LassoModel lasso_fit(const DndArray<double>& x, const DndArray<double>& y, double lambda, int sweeps,
                            double tol = 0.0) {
    if (x.ndim() != 2) throw ValueError("lasso_fit: design matrix must be 2-D");
    if (y.ndim() != 1) throw ValueError("lasso_fit: targets must be 1-D");
    if (x.shape()[0] != y.shape()[0])
        throw ValueError("lasso_fit: " + std::to_string(x.shape()[0]) + " rows vs " + std::to_string(y.shape()[0]) +
                         " targets");
    if (x.shape()[0] < 1) throw ValueError("lasso_fit: need at least one sample");
    if (x.shape()[1] < 1) throw ValueError("lasso_fit: design matrix needs at least the bias column");
    if (lambda < 0.0) throw ValueError("lasso_fit: lambda must be nonnegative");
    if (sweeps < 1) throw ValueError("lasso_fit: sweeps must be positive");
    if (x.split() != std::optional<int>(0) || y.split() != std::optional<int>(0))
        return lasso_fit(x.split() == std::optional<int>(0) ? x : resplit(x, 0),
                         y.split() == std::optional<int>(0) ? y : resplit(y, 0), lambda, sweeps, tol);
    const index_t m = x.shape()[1];
    LassoModel model;
    model.lambda = lambda;
    model.weights.assign(static_cast<std::size_t>(m), 0.0);
    model.objective_trace.assign(static_cast<std::size_t>(sweeps), 0.0);
    detail::check(dndc_lasso_fit_f64(x.comm().handle(), x.device_data(), x.lshape()[0], x.shape()[0], m,
                                     y.device_data(), lambda, sweeps, tol, model.weights.data(),
                                     model.objective_trace.data(), &model.sweeps_run));
    model.objective_trace.resize(static_cast<std::size_t>(model.sweeps_run));
    return model;
}

/// Xw per local row (regression.cpp:105-127): split=0 in -> split=0 out,
/// replicated in -> replicated out; no communication.
inline DndArray<double> lasso_predict(const LassoModel& model, const DndArray<double>& x) {
    if (x.ndim() != 2) throw ValueError("lasso_predict: input must be 2-D");
    if (x.shape()[1] != static_cast<index_t>(model.weights.size()))
        throw ValueError("lasso_predict: input has " + std::to_string(x.shape()[1]) + " columns, model expects " +
                         std::to_string(model.weights.size()));
    if (x.split() && *x.split() != 0) throw ValueError("lasso_predict: input must be split=0 or replicated");
    const index_t rows = x.lshape()[0];
    auto out = detail::device_alloc<double>(x.comm(), rows);
    detail::check(dndc_lasso_predict_f64(x.comm().handle(), x.device_data(), rows, x.shape()[1],
                                         model.weights.data(), out.get()));
    return DndArray<double>({x.shape()[0]}, x.split() ? std::optional<int>(0) : std::nullopt, x.comm(), {rows},
                            out);
}

}  // namespace dnd
