// dnd/cluster.hpp -- B200 drop-in for proj/include/dnd/cluster.hpp
// (cluster.cpp:13-172): Lloyd's k-means over row shards in HBM.
#pragma once

#include <cstdint>
#include <type_traits>
#include <vector>

#include "dnd/ndarray.hpp"
#include "dnd/pairwise.hpp"

namespace dnd {

struct KMeansModel {
    int k = 0;
    index_t n_features = 0;
    std::vector<double> centroids;  // k x n_features, row-major, f64 master copy
    std::vector<double> inertia_trace;
    int iterations_run = 0;
    std::uint64_t seed = 0;
};

/// k distinct global row indices, a pure function of (n, k, seed) (cluster.cpp:60-75).
inline std::vector<index_t> kmeans_init_indices(index_t n, int k, std::uint64_t seed) {
    std::vector<index_t> out(static_cast<std::size_t>(k > 0 ? k : 0));
    detail::check(dndc_kmeans_init_indices(n, k, seed, out.data()));
    return out;
}

/// Rows of x at the sampled indices, replicated (cluster.cpp:77-81).
template <typename T>
std::vector<double> kmeans_init_centroids(const DndArray<T>& x, int k, std::uint64_t seed) {
    detail::require_2d(x, "kmeans_init_centroids");
    const index_t n = x.shape()[0], m = x.shape()[1];
    if (k < 1 || k > n) throw ValueError("kmeans_init_centroids: k=" + std::to_string(k) + " out of range");
    if (x.split() && *x.split() != 0) return kmeans_init_centroids(resplit(x, 0), k, seed);  // cluster.cpp:79
    std::vector<double> c(static_cast<std::size_t>(k * m), 0.0);
    if constexpr (std::is_same_v<T, float>) {
        index_t rows = 0;
        const T* xl = detail::rank_rows(x, rows);
        detail::check(dndc_kmeans_init_centroids_f32(x.comm().handle(), xl, rows, n, m, k, seed, c.data()));
    } else {
        // gather_rows (cluster.cpp:27-42): owned rows into a zero-filled
        // buffer, then an exact allreduce-sum
        const auto idx = kmeans_init_indices(n, k, seed);
        const index_t lo = x.row_offset(), hi = lo + (x.split() ? x.lshape()[0] : n);
        for (int j = 0; j < k; ++j)
            if (idx[j] >= lo && idx[j] < hi)
                detail::check(dndc_memcpy(x.comm().handle(), c.data() + j * m, x.device_data() + (idx[j] - lo) * m,
                                          m * sizeof(double), DNDC_COPY_D2H));
        if (x.split()) {
            auto d = detail::device_alloc<double>(x.comm(), k * m);
            detail::check(dndc_memcpy(x.comm().handle(), d.get(), c.data(), c.size() * sizeof(double), DNDC_COPY_H2D));
            detail::check(dndc_allreduce_f64(x.comm().handle(), d.get(), k * m));
            detail::check(dndc_memcpy(x.comm().handle(), c.data(), d.get(), c.size() * sizeof(double), DNDC_COPY_D2H));
        }
    }
    return c;
}

/// Lloyd's algorithm (cluster.cpp:83-153): the whole loop runs on the GPUs,
/// one fused kernel per iteration (NVLink peer exchange of the stats across
/// ranks); validation, seeding and the model are the reference's.
template <typename T>
KMeansModel kmeans_fit(const DndArray<T>& x, int k, int max_iter, double tol, std::uint64_t seed) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "kmeans_fit: float or double");
    detail::require_2d(x, "kmeans_fit");
    if ((x.split() && *x.split() != 0) || (!x.split() && x.comm().size() > 1))
        return kmeans_fit(resplit(x, 0), k, max_iter, tol, seed);  // cluster.cpp:91
    const index_t n = x.shape()[0], m = x.shape()[1];
    KMeansModel model;
    model.k = k;
    model.n_features = m;
    model.seed = seed;
    model.centroids.assign(static_cast<std::size_t>(k > 0 ? k * m : 0), 0.0);
    model.inertia_trace.assign(static_cast<std::size_t>(max_iter > 0 ? max_iter : 0), 0.0);
    const index_t rows = x.lshape()[0];
    int iters = 0;
    if constexpr (std::is_same_v<T, float>)
        detail::check(dndc_kmeans_fit_f32(x.comm().handle(), x.device_data(), rows, n, m, k, max_iter, tol, seed,
                                          nullptr, model.centroids.data(), model.inertia_trace.data(), &iters));
    else
        detail::check(dndc_kmeans_fit_f64(x.comm().handle(), x.device_data(), rows, n, m, k, max_iter, tol, seed,
                                          nullptr, model.centroids.data(), model.inertia_trace.data(), &iters));
    model.iterations_run = iters;
    model.inertia_trace.resize(static_cast<std::size_t>(iters));
    return model;
}

/// Nearest-centroid label per row, ties to the lowest index (cluster.cpp:155-172).
template <typename T>
DndArray<std::int32_t> kmeans_predict(const KMeansModel& model, const DndArray<T>& x) {
    detail::require_2d(x, "kmeans_predict");
    if (x.split() && *x.split() != 0)
        throw ValueError("kmeans_predict: input must be split=0 or replicated");  // cluster.cpp:160-161
    if (x.shape()[1] != model.n_features)
        throw ValueError("kmeans_predict: model has " + std::to_string(model.n_features) + " features, input " +
                         std::to_string(x.shape()[1]));
    const index_t rows = x.lshape()[0];
    auto labels = detail::device_alloc<std::int32_t>(x.comm(), rows);
    if (rows > 0) {
        if constexpr (std::is_same_v<T, float>)
            detail::check(dndc_kmeans_predict_f32(x.comm().handle(), x.device_data(), rows, x.shape()[1],
                                                  model.centroids.data(), model.k, labels.get()));
        else
            detail::check(dndc_kmeans_predict_f64(x.comm().handle(), x.device_data(), rows, x.shape()[1],
                                                  model.centroids.data(), model.k, labels.get()));
    }
    return DndArray<std::int32_t>({x.shape()[0]}, x.split(), x.comm(), {rows}, labels);
}

}  // namespace dnd
