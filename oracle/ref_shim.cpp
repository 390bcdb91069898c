// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE.  oracle/Makefile compiles this file together
// with /root/reference/proj/src/*.cpp (in place, read-only) into
// oracle/_ref/libdndref.so.  It is used (a) to pin the C restatement
// (oracle/dnd_oracle.c) and generate tests/golden fixtures, and (b) as the
// reference arm of bench.py (`--impl reference`) and its cpu_baseline leg.
// No reference source is copied into this repository; this file only calls
// the reference's public API (proj/include/dnd/*.hpp).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dnd/chunking.hpp"
#include "dnd/cluster.hpp"
#include "dnd/moments.hpp"
#include "dnd/ndarray.hpp"
#include "dnd/pairwise.hpp"
#include "dnd/regression.hpp"
#include "dnd/transport.hpp"

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const dnd::ValueError& e) {
        g_error = e.what();
        return -1;
    } catch (const dnd::TransportError& e) {
        g_error = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -3;
    }
}

// Rank-local split=0 shard of a replicated row-major n x m buffer, built
// directly (DndArray's public constructor, ndarray.hpp:63-65) so large inputs
// are not copied p times by from_global.
dnd::DndArray<double> shard_rows(const double* x, std::int64_t n, std::int64_t m,
                                 const dnd::Communicator& comm) {
    const auto map = dnd::chunk_map(n, comm.size());
    const auto lo = map.offset(comm.rank()), ext = map.extent(comm.rank());
    std::vector<double> data(x + lo * m, x + (lo + ext) * m);
    return dnd::DndArray<double>({n, m}, 0, comm, dnd::Tile<double>{{ext, m}, std::move(data)});
}

dnd::DndArray<double> synthetic_f32_as_f64(std::int64_t n, std::int64_t m, std::uint64_t seed,
                                           const dnd::Communicator& comm) {
    // What the parity contract feeds the reference: random_uniform<float>
    // values, widened exactly.
    return dnd::astype<double>(dnd::random_uniform<float>({n, m}, 0, seed, comm));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

int ref_chunk_map(std::int64_t n, int p, std::int64_t* offsets, std::int64_t* extents) {
    return guarded([&] {
        const auto map = dnd::chunk_map(n, p);
        for (int r = 0; r < p; ++r) {
            offsets[r] = map.offset(r);
            extents[r] = map.extent(r);
        }
    });
}

int ref_fill_uniform_f32(std::int64_t n, std::int64_t m, std::uint64_t seed, int p, float* out) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = dnd::random_uniform<float>({n, m}, 0, seed, comm);
            auto all = dnd::gather(a);
            if (comm.rank() == 0) std::memcpy(out, all.data(), all.size() * sizeof(float));
        });
    });
}

int ref_row_norms(const double* x, std::int64_t rows, std::int64_t m, double* out) {
    return guarded([&] {
        dnd::Tile<double> t{{rows, m}, std::vector<double>(x, x + rows * m)};
        auto v = dnd::detail::row_norms(t);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int ref_cdist(const double* x, std::int64_t n, std::int64_t m, int p, double* out,
              std::uint64_t* sendrecvs_rank0) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = shard_rows(x, n, m, comm);
            const auto before = comm.counters().sendrecvs;
            auto d = dnd::cdist(a);
            const auto delta = comm.counters().sendrecvs - before;
            auto all = dnd::gather(d);
            if (comm.rank() == 0) {
                std::memcpy(out, all.data(), all.size() * sizeof(double));
                if (sendrecvs_rank0) *sendrecvs_rank0 = delta;
            }
        });
    });
}

int ref_cdist_xy(const double* x, std::int64_t nx, const double* y, std::int64_t ny,
                 std::int64_t m, int p, double* out) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = shard_rows(x, nx, m, comm);
            auto b = dnd::from_global(std::vector<double>(y, y + ny * m), {ny, m}, std::nullopt, comm);
            auto all = dnd::gather(dnd::cdist_xy(a, b));
            if (comm.rank() == 0) std::memcpy(out, all.data(), all.size() * sizeof(double));
        });
    });
}

int ref_kmeans_init_indices(std::int64_t n, int k, std::uint64_t seed, std::int64_t* out) {
    return guarded([&] {
        auto v = dnd::kmeans_init_indices(n, k, seed);
        std::memcpy(out, v.data(), v.size() * sizeof(std::int64_t));
    });
}

static void copy_model(const dnd::KMeansModel& model, double* centroids, double* inertia_trace,
                       int* iterations_run) {
    std::memcpy(centroids, model.centroids.data(), model.centroids.size() * sizeof(double));
    std::memcpy(inertia_trace, model.inertia_trace.data(),
                model.inertia_trace.size() * sizeof(double));
    *iterations_run = model.iterations_run;
}

int ref_kmeans_fit(const double* x, std::int64_t n, std::int64_t m, int p, int k, int max_iter,
                   double tol, std::uint64_t seed, double* centroids, double* inertia_trace,
                   int* iterations_run) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = shard_rows(x, n, m, comm);
            auto model = dnd::kmeans_fit(a, k, max_iter, tol, seed);
            if (comm.rank() == 0) copy_model(model, centroids, inertia_trace, iterations_run);
        });
    });
}

// kmeans_fit on the synthetic fp32 input generated inside every rank
// (random_uniform<float>(seed=data_seed) -> astype<double>), for golden runs at
// full BASELINE sizes.
int ref_kmeans_fit_synthetic(std::int64_t n, std::int64_t m, std::uint64_t data_seed, int p, int k,
                             int max_iter, double tol, std::uint64_t seed, double* centroids,
                             double* inertia_trace, int* iterations_run) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = synthetic_f32_as_f64(n, m, data_seed, comm);
            auto model = dnd::kmeans_fit(a, k, max_iter, tol, seed);
            if (comm.rank() == 0) copy_model(model, centroids, inertia_trace, iterations_run);
        });
    });
}

int ref_kmeans_predict(const double* x, std::int64_t n, std::int64_t m, int p,
                       const double* centroids, int k, std::int32_t* labels) {
    return guarded([&] {
        dnd::KMeansModel model;
        model.k = k;
        model.n_features = m;
        model.centroids.assign(centroids, centroids + k * m);
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = shard_rows(x, n, m, comm);
            auto all = dnd::gather(dnd::kmeans_predict(model, a));
            if (comm.rank() == 0) std::memcpy(labels, all.data(), all.size() * sizeof(std::int32_t));
        });
    });
}

int ref_moments_axis0(const double* x, std::int64_t n, std::int64_t m, int p, std::int64_t ddof,
                      double* mean_out, double* var_out) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = shard_rows(x, n, m, comm);
            auto mean = dnd::gather(dnd::mean_axis(a, 0));
            auto var = dnd::gather(dnd::var_axis(a, 0, ddof));
            if (comm.rank() == 0) {
                std::memcpy(mean_out, mean.data(), mean.size() * sizeof(double));
                std::memcpy(var_out, var.data(), var.size() * sizeof(double));
            }
        });
    });
}

// The reference's bench protocol (tools/bench.cpp:84-112): per rank the
// synthetic dataset, `warmup` untimed runs, then `runs` timed runs each
// bracketed by barriers and reported as the max over ranks.  algo: 0 =
// kmeans_fit(k, iters, tol 0, seed), 1 = cdist(x), 2 = mean_axis + var_axis.
int ref_bench(int algo, std::int64_t n, std::int64_t m, int k, int iters, std::uint64_t seed,
              int p, int warmup, int runs, double* run_seconds, double* checksum) {
    return guarded([&] {
        std::mutex mu;
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto x = synthetic_f32_as_f64(n, m, seed, comm);
            double sink = 0.0;
            auto once = [&]() {
                if (algo == 0) {
                    auto model = dnd::kmeans_fit(x, k, iters, 0.0, seed);
                    sink += model.inertia_trace.back();
                } else if (algo == 1) {
                    auto d = dnd::cdist(x);
                    sink += d.tile().data.empty() ? 0.0 : d.tile().data.back();
                } else {
                    auto mu_ = dnd::mean_axis(x, 0);
                    auto var = dnd::var_axis(x, 0);
                    sink += mu_.tile().data[0] + var.tile().data[0];
                }
            };
            for (int w = 0; w < warmup; ++w) once();
            for (int r = 0; r < runs; ++r) {
                comm.barrier();
                const auto t0 = std::chrono::steady_clock::now();
                once();
                comm.barrier();
                const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
                const double worst =
                    comm.allreduce(el.count(), [](double a, double b) { return a > b ? a : b; }, 0.0);
                if (comm.rank() == 0) run_seconds[r] = worst;
            }
            if (comm.rank() == 0) {
                std::lock_guard<std::mutex> lock(mu);
                *checksum = sink;
            }
        });
    });
}

// lasso_fit (regression.cpp:25-102) on p ranks: x n x m row-major with the
// bias column, y n targets, both split=0
int ref_lasso_fit(const double* x, const double* y, std::int64_t n, std::int64_t m, int p, double lambda,
                  int sweeps, double tol, double* weights, double* trace, int* sweeps_run) {
    return guarded([&] {
        dnd::run_world(p, [&](const dnd::Communicator& comm) {
            auto a = shard_rows(x, n, m, comm);
            auto b = shard_rows(y, n, 1, comm);
            auto t = dnd::DndArray<double>({n}, 0, comm, dnd::Tile<double>{{b.tile().extents[0]}, b.tile().data});
            auto model = dnd::lasso_fit(a, t, lambda, sweeps, tol);
            if (comm.rank() == 0) {
                std::memcpy(weights, model.weights.data(), sizeof(double) * model.weights.size());
                std::memcpy(trace, model.objective_trace.data(), sizeof(double) * model.objective_trace.size());
                *sweeps_run = model.sweeps_run;
            }
        });
    });
}

}  // extern "C"
