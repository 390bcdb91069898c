/*
 * dnd_oracle.h -- CPU restatement of the reference `dnd` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This header and dnd_oracle.c are the checker the
 * parity tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg use.
 * Nothing in the product path (paper_2007_13552_b200/, include/dndc.h) may
 * include, link or call it.
 *
 * Every function restates one reference function (file:line into
 * /root/reference/proj) with the same floating-point operation order, so the
 * oracle reproduces the reference bit for bit; tests/test_oracle.py pins it
 * against golden vectors produced by the reference itself (oracle/_ref,
 * tests/golden/make_golden.py).
 *
 * "p" arguments simulate the reference's loopback world of p rank-threads:
 * rows are split by chunk_map, per-rank partial results are folded in rank
 * order 0..p-1 exactly as Communicator::allreduce does (transport.hpp:136-148).
 */
#ifndef DND_ORACLE_H
#define DND_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* common.hpp:14-19 */
uint64_t dno_splitmix64(uint64_t x);
/* common.hpp:24-27 */
double dno_uniform01(uint64_t seed, uint64_t counter);

/* random_uniform<float>/<double> (ndarray.hpp:154-169): element (r, f) of a
 * rows x m array whose first global row is row0. */
void dno_fill_uniform_f32(uint64_t seed, int64_t row0, int64_t rows, int64_t m, float* out);
void dno_fill_uniform_f64(uint64_t seed, int64_t row0, int64_t rows, int64_t m, double* out);

/* chunking.cpp:9-30; returns 0, or -1 on invalid arguments (ValueError). */
int dno_chunk_map(int64_t n, int p, int64_t* offsets, int64_t* extents);

/* pairwise.cpp:10-20 */
void dno_row_norms(const double* x, int64_t rows, int64_t m, double* out);
/* pairwise.cpp:22-33 with matmul_local (ndarray.hpp:400-418); out is rows x cols */
void dno_distance_block(const double* a, const double* na, int64_t rows, const double* b,
                        const double* nb, int64_t cols, int64_t m, double* out);
/* pairwise.cpp:37-85: ring cdist over p simulated ranks; out is n x n.
 * returns 0 or -1 (ValueError: n == 0). sendrecvs_per_rank (optional) gets p-1. */
int dno_cdist(const double* x, int64_t n, int64_t m, int p, double* out,
              int64_t* sendrecvs_per_rank);
/* pairwise.cpp:87-100 */
int dno_cdist_xy(const double* x, int64_t nx, const double* y, int64_t ny, int64_t m,
                 double* out);

/* cluster.cpp:60-75 (sparse restatement of the iota-pool Fisher-Yates) */
int dno_kmeans_init_indices(int64_t n, int k, uint64_t seed, int64_t* out);
/* cluster.cpp:83-153.  centroids: k*m, inertia_trace: max_iter entries.
 * returns 0, -1 (ValueError: bad k / max_iter), -2 (non-finite input). */
int dno_kmeans_fit(const double* x, int64_t n, int64_t m, int p, int k, int max_iter,
                   double tol, uint64_t seed, double* centroids, double* inertia_trace,
                   int* iterations_run);
/* Same Lloyd loop from caller-provided initial centroids (used to restate
 * single iterations; kmeans_fit == init + this). */
int dno_kmeans_lloyd(const double* x, int64_t n, int64_t m, int p, int k, int max_iter,
                     double tol, double* centroids, double* inertia_trace, int* iterations_run);
/* cluster.cpp:155-172 */
void dno_kmeans_predict(const double* x, int64_t n, int64_t m, const double* centroids, int k,
                        int32_t* labels);

/* moments.cpp:100-114 (axis 0 of a rows x m tile) */
void dno_local_moments_axis0(const double* x, int64_t rows, int64_t m, int64_t* count,
                             double* mean, double* m2);
/* moments.cpp:100-114 continued over fp32 row blocks (state in/out) */
void dno_welford_axis0_f32_continue(const float* x, int64_t rows, int64_t m, int64_t* count,
                                    double* mean, double* m2);
/* moments.cpp:91-98 (flattened tile) */
void dno_local_moments_flat(const double* x, int64_t numel, int64_t* count, double* mean,
                            double* m2);
/* moments.cpp:69-89, in place: (ca, ma, m2a) <- combine(a, b) */
void dno_combine(int64_t* ca, double* ma, double* m2a, int64_t cb, const double* mb,
                 const double* m2b, int64_t arity);
/* moments.cpp:33-52 + :126-140 along the split axis 0 over p simulated ranks.
 * mean_out / var_out may be NULL.  returns 0 or -1 (ValueError: count <= ddof). */
int dno_moments_axis0(const double* x, int64_t n, int64_t m, int p, int64_t ddof,
                      double* mean_out, double* var_out);

/* k-means++ seeding (BASELINE config 5; NOT in the reference).
 * Definition owned by this repo -- see DESIGN.md "k-means++" and the CUDA
 * kernel it pins.  indices: k global row ids. x is fp32 (the device dtype). */
int dno_kmeanspp_indices_f32(const float* x, int64_t n, int64_t m, int p, int k, uint64_t seed,
                             int64_t* indices);
int dno_kmeanspp_indices_f64(const double* x, int64_t n, int64_t m, int p, int k, uint64_t seed,
                             int64_t* indices);

/* LASSO coordinate descent (regression.cpp:19-102) */
double dno_soft_threshold(double rho, double t);
int dno_lasso_fit(const double* x, const double* y, int64_t n, int64_t m, int p, double lambda, int sweeps,
                  double tol, double* weights, double* trace, int* sweeps_run);

#ifdef __cplusplus
}
#endif

#endif
