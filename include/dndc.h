/*
 * dndc.h -- C ABI of the B200-native cdist / k-means / moments hot path.
 *
 * This is the drop-in boundary below the reference's C++ API (proj/include/dnd):
 * plain pointers, sizes and status codes, no torch or C++ types.  The C++
 * surface in cpp/include/dnd/ and the Python mirror in paper_2007_13552_b200/
 * both sit on top of it; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *  - Array arguments are DEVICE pointers (row-major, contiguous) unless the
 *    name ends in `_host`.  The library borrows them and never frees caller
 *    memory; scratch lives in the context's workspace.
 *  - Every call is issued on the context's stream (dndc_set_stream) and is
 *    asynchronous unless it returns host results (those synchronise the stream).
 *  - "Collective" calls must be entered by every rank of the context's world in
 *    the same program order (the reference's rule, transport.hpp:79-84).
 *  - Status: 0 ok; DNDC_EVALUE maps to dnd::ValueError, DNDC_ETRANSPORT to
 *    dnd::TransportError, DNDC_ECUDA to a device failure.  The message of the
 *    last failure on the calling thread is dndc_last_error().
 *  - `split=0` shards: rank r owns global rows [off(r), off(r)+ext(r)) of
 *    chunk_map(n, world) (chunking.cpp:9-30); x_local points at those rows.
 */
#ifndef DNDC_H
#define DNDC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DNDC_OK 0
#define DNDC_EVALUE 1     /* dnd::ValueError (errors.hpp:14-18) */
#define DNDC_ETRANSPORT 2 /* dnd::TransportError (errors.hpp:21-25) */
#define DNDC_ECUDA 3      /* CUDA runtime / launch failure */
#define DNDC_EINTERNAL 4
#define DNDC_EDATA 5      /* dnd::DataError (errors.hpp:40): file I/O and container format */
#define DNDC_ETIMEOUT 6   /* dnd::TimeoutError (errors.hpp:27-31): a rank did not arrive (DND_TIMEOUT_SECS) */
#define DNDC_EORDERING 7  /* dnd::OrderingError (errors.hpp:33-37): ranks entered different collectives */

#define DNDC_UNIQUE_ID_BYTES 128

typedef struct dndc_ctx dndc_ctx;

/* Per-rank tally of transport calls; mirrors dnd::TransportCounters
 * (transport.hpp:19-27) so tests can pin "p-1 ring exchanges" and
 * "cdist_xy is communication-free" (test_pairwise.cpp:84-94, :146-166). */
typedef struct {
    uint64_t sends, recvs, sendrecvs, allreduces, allgathers, alltoalls, barriers;
} dndc_counters;

/* ------------------------------------------------------------- runtime */
int dndc_version(void);
const char* dndc_last_error(void);

/* Rank handle: one per GPU.  world == 1 needs no unique id.  For world > 1
 * every rank passes the same id from dndc_unique_id() (exchanged by the host,
 * e.g. over torch.distributed); the handle then owns an NCCL communicator over
 * NVLink.  Replaces run_world's per-rank Communicator (transport.hpp:85-217,
 * transport.cpp:166-193). */
int dndc_unique_id(void* id_out /* DNDC_UNIQUE_ID_BYTES */);
int dndc_create(int device, int rank, int world, const void* unique_id, dndc_ctx** out);
int dndc_destroy(dndc_ctx* ctx);

/* Ranks that share GPUs (world > visible GPUs, e.g. the reference's tests run
 * run_world(3..5) on one GPU; transport.hpp:222-223): the ranks are threads of
 * one process joined by a host loopback group instead of NCCL.  Device
 * collectives are staged through host memory with the reference's loopback
 * semantics (transport.cpp:64-150): rank-order folds, DNDC_EORDERING when
 * ranks enter different collectives at the same call index, DNDC_ETIMEOUT
 * after timeout_ms (DND_TIMEOUT_SECS), DNDC_ETRANSPORT after
 * dndc_group_abort (a failing rank wakes its peers, transport.cpp:174-192).
 * The group outlives its contexts; destroy it after them. */
typedef struct dndc_group dndc_group;
int dndc_group_create(int world, int64_t timeout_ms, dndc_group** out);
int dndc_group_destroy(dndc_group* g);
int dndc_group_abort(dndc_group* g);
int dndc_create_in_group(int device, int rank, dndc_group* group, int world, dndc_ctx** out);
int dndc_set_stream(dndc_ctx* ctx, void* cuda_stream);
int dndc_rank(const dndc_ctx* ctx);
/* How the k-means stats exchange travels for world > 1: "nvlink peer exchange"
 * (stats stored by the fused kernel straight into every peer over NVLink,
 * CUDA IPC mappings) or why it fell back to the NCCL allgather path. */
const char* dndc_transport_status(const dndc_ctx* ctx);
int dndc_world(const dndc_ctx* ctx);
int dndc_synchronize(dndc_ctx* ctx);
int dndc_get_counters(const dndc_ctx* ctx, dndc_counters* out);
/* Device kernel launches issued by this context since creation (evidence for
 * bench.py's gpu_launches). */
uint64_t dndc_launch_count(const dndc_ctx* ctx);

/* chunk_map (chunking.cpp:9-30), host only. */
int dndc_chunk_map(int64_t n, int world, int64_t* offsets_host, int64_t* extents_host);

/* ---------------------------------------------- device memory and copies */
/* What a host layer needs to own device tiles without CUDA headers (the C++
 * drop-in in cpp/include/dnd keeps DndArray shards in HBM through these).
 * Copies are synchronous with respect to the handle's stream. */
#define DNDC_COPY_H2D 1
#define DNDC_COPY_D2H 2
#define DNDC_COPY_D2D 3
int dndc_device_count(int* out);
/* Communicator::barrier (transport.hpp:150-153), collective. */
int dndc_barrier(dndc_ctx* ctx);
int dndc_alloc(dndc_ctx* ctx, size_t bytes, void** out);
int dndc_free(dndc_ctx* ctx, void* p);
int dndc_memcpy(dndc_ctx* ctx, void* dst, const void* src, size_t bytes, int kind);

/* gather of a split=0 array (ndarray.hpp:389-393 via resplit :354-368),
 * collective: every rank's device rows (row_bytes each) concatenated in rank
 * order into out_host; *total_rows receives the global row count. */
int dndc_allgather_rows(dndc_ctx* ctx, const void* local, int64_t rows, int64_t row_bytes, void* out_host,
                        int64_t* total_rows);

/* resplit (ndarray.hpp:340-386, F1), collective: move a row-major N-D array
 * (ndim <= 8, elem_bytes 1/2/4/8) from src_split to dst_split (-1 = replicated)
 * without changing its global content.  src_local / dst_local are this rank's
 * device shards under the chunk map of the respective axis; replicated ->
 * split slices locally, split -> anything is one grouped NCCL send/recv of the
 * intersection blocks.  Returns after the stream has drained. */
int dndc_resplit(dndc_ctx* ctx, const void* src_local, int ndim, const int64_t* shape, int64_t elem_bytes,
                 int src_split, int dst_split, void* dst_local);

/* DNB container I/O straight between a file and HBM (dataio.hpp:61-142, F2):
 * the byte range [byte_offset, byte_offset + bytes) of `path` is streamed
 * through two pinned chunks (positioned reads overlapped with the H2D copy)
 * into dev_dst, or from dev_src into an existing file.  The DNB header itself
 * (magic, dtype, extents) is parsed by the host layer.  Local, not
 * collective; DNDC_EDATA on open/short-read/write failures. */
int dndc_file_read_to_device(dndc_ctx* ctx, const char* path, uint64_t byte_offset, size_t bytes, void* dev_dst);
int dndc_file_write_from_device(dndc_ctx* ctx, const char* path, uint64_t byte_offset, const void* dev_src,
                                size_t bytes);

/* lasso_fit (regression.cpp:25-102, F4), collective: cyclic coordinate descent
 * on this rank's rows x_local (rows x m, f64, column 0 all ones) and targets
 * y_local (rows); weights_out[m] and trace_out[sweeps] (objective per sweep)
 * in host memory, identical on every rank; *sweeps_run <= sweeps (stops when
 * the largest coordinate change < tol).  DNDC_EVALUE for bad arguments or a
 * bias column that is not all ones on any rank (raised on every rank). */
int dndc_lasso_fit_f64(dndc_ctx* ctx, const double* x_local, int64_t rows, int64_t n_global, int64_t m,
                       const double* y_local, double lambda, int sweeps, double tol, double* weights_out,
                       double* trace_out, int* sweeps_run);
/* lasso_predict (regression.cpp:105-127): out_local[i] = sum_j x[i,j] w[j] in
 * column order without FMA contraction (bit-identical to the reference);
 * weights in host memory, out_local on the device; local, no communication. */
int dndc_lasso_predict_f64(dndc_ctx* ctx, const double* x_local, int64_t rows, int64_t m, const double* weights,
                           double* out_local);

/* Communicator::allreduce(plus) (transport.hpp:136-148, A15), collective, in
 * place on a device buffer: sum over ranks folded in rank order 0..p-1 from
 * the zero identity, bit-identical on every rank. */
int dndc_allreduce_f64(dndc_ctx* ctx, double* buf, int64_t count);

/* ------------------------------------------------------- A1: generator */
/* random_uniform<float>/<double> (ndarray.hpp:154-169, common.hpp:14-27): the
 * rows x m block starting at global row row0, bit-identical to the reference. */
int dndc_fill_uniform_f32(dndc_ctx* ctx, uint64_t seed, int64_t row0, int64_t rows, int64_t m,
                          float* out);
int dndc_fill_uniform_f64(dndc_ctx* ctx, uint64_t seed, int64_t row0, int64_t rows, int64_t m,
                          double* out);

/* ----------------------------------------------------- A3-A7: pairwise */
/* detail::row_norms (pairwise.cpp:10-20).  f32: sequential fmaf chain, the
 * same op order as the distance kernel's dot products, so a row's distance to
 * itself cancels exactly.  f64: bit-identical to the reference. */
int dndc_row_norms_f32(dndc_ctx* ctx, const float* x, int64_t rows, int64_t m, float* out);
int dndc_row_norms_f64(dndc_ctx* ctx, const double* x, int64_t rows, int64_t m, double* out);

/* distance_block + place_chunk (pairwise.cpp:22-33, :69; tile.hpp:90-107):
 * out[i*ld_out + col_off + j] = sqrt(max(xn[i] + yn[j] - 2 x_i.y_j, 0)) for
 * i < nx, j < ny; with diag_offset >= 0 the entries j == i + diag_offset are
 * written as 0 (the self block, pairwise.cpp:63-68). */
int dndc_cdist_tile_f32(dndc_ctx* ctx, const float* x, const float* xn, int64_t nx,
                        const float* y, const float* yn, int64_t ny, int64_t m, float* out,
                        int64_t ld_out, int64_t col_off, int64_t diag_offset);
int dndc_cdist_tile_f64(dndc_ctx* ctx, const double* x, const double* xn, int64_t nx,
                        const double* y, const double* yn, int64_t ny, int64_t m, double* out,
                        int64_t ld_out, int64_t col_off, int64_t diag_offset);

/* cdist(x) (pairwise.cpp:37-85), collective: the ring of row blocks with
 * exactly world-1 NCCL send/recv exchanges per rank, overlapped with the
 * distance tiles.  out: n_local x n_global (this rank's row block, split=0).
 * DNDC_EVALUE when n_global == 0 (pairwise.cpp:39). */
int dndc_cdist_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, int64_t n_global,
                   int64_t m, float* out);
int dndc_cdist_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, int64_t n_global,
                   int64_t m, double* out);

/* cdist_xy(x, y) with y replicated (pairwise.cpp:87-100): communication-free. */
int dndc_cdist_xy_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, const float* y,
                      int64_t ny, int64_t m, float* out);
int dndc_cdist_xy_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, const double* y,
                      int64_t ny, int64_t m, double* out);

/* cdist_xy(x, y) with BOTH split=0 (BASELINE config 2): instead of the
 * reference's allgather of y (pairwise.cpp:94 -> ndarray.hpp:354-368), y's
 * shards travel the ring like cdist's blocks; world-1 exchanges per rank.
 * out: n_local x ny_global. */
int dndc_cdist_xy_ring_f32(dndc_ctx* ctx, const float* x_local, int64_t nx_local,
                           const float* y_local, int64_t ny_local, int64_t ny_global, int64_t m,
                           float* out);
int dndc_cdist_xy_ring_f64(dndc_ctx* ctx, const double* x_local, int64_t nx_local,
                           const double* y_local, int64_t ny_local, int64_t ny_global, int64_t m,
                           double* out);

/* ------------------------------------------------------ A8-A12: k-means */
/* kmeans_init_indices (cluster.cpp:60-75), host only, O(k) memory. */
int dndc_kmeans_init_indices(int64_t n, int k, uint64_t seed, int64_t* out_host);

/* kmeans_init_centroids (cluster.cpp:77-81, gather_rows :27-42), collective:
 * the rows at the sampled indices, replicated (k x m, f64, host). */
int dndc_kmeans_init_centroids_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local,
                                   int64_t n_global, int64_t m, int k, uint64_t seed,
                                   double* centroids_host);

/* kmeans_fit (cluster.cpp:83-153), collective.  Validates like the reference
 * (k range, max_iter >= 1, non-finite input -> DNDC_EVALUE on every rank),
 * seeds with kmeans_init_indices(seed) unless init_centroids_host != NULL,
 * then runs fused assign/accumulate kernels with one f64 exchange of
 * k*m + k values per iteration folded in rank order.  Outputs (host):
 * centroids k x m (f64 master copy), inertia_trace (max_iter entries, the
 * first *iterations_run valid).  With tol == 0 the whole loop is one CUDA graph. */
int dndc_kmeans_fit_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, int64_t n_global,
                        int64_t m, int k, int max_iter, double tol, uint64_t seed,
                        const double* init_centroids_host, double* centroids_host,
                        double* inertia_trace_host, int* iterations_run);
int dndc_kmeans_fit_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local,
                        int64_t n_global, int64_t m, int k, int max_iter, double tol,
                        uint64_t seed, const double* init_centroids_host,
                        double* centroids_host, double* inertia_trace_host,
                        int* iterations_run);

/* kmeans_predict (cluster.cpp:155-172): nearest centroid, ties to the lowest
 * index; labels is a device int32 array of n rows.  Communication-free. */
int dndc_kmeans_predict_f32(dndc_ctx* ctx, const float* x, int64_t n, int64_t m,
                            const double* centroids_host, int k, int32_t* labels);
int dndc_kmeans_predict_f64(dndc_ctx* ctx, const double* x, int64_t n, int64_t m,
                            const double* centroids_host, int k, int32_t* labels);

/* One Lloyd assignment/accumulation step on this rank's rows (cluster.cpp:
 * 108-122, A8/A9) against given centroids (k x m f64, host): the LOCAL
 * (not reduced) stats, k*m sums then k counts, then the local inertia
 * (sum of squared distances of the rows to their centroid), k*m + k + 1
 * doubles on the host; labels (device int32, n) when non-NULL.
 * Communication-free: reduce with dndc_allreduce_f64 for the global step. */
int dndc_kmeans_step_f32(dndc_ctx* ctx, const float* x, int64_t n, int64_t m, const double* centroids_host,
                         int k, double* stats_host, int32_t* labels);
int dndc_kmeans_step_f64(dndc_ctx* ctx, const double* x, int64_t n, int64_t m, const double* centroids_host,
                         int k, double* stats_host, int32_t* labels);

/* Statistics of the most recent kmeans_fit/predict on this context: rows whose
 * fp32 top-2 gap fell inside the error bound and were re-decided in f64. */
int dndc_kmeans_last_refined(const dndc_ctx* ctx, int64_t* rows_refined);

/* Name of the kernel that ran the Lloyd loop of the most recent kmeans_fit
 * ("" when it was the per-iteration launch sequence); static storage. */
const char* dndc_kmeans_last_kernel(const dndc_ctx* ctx);
/* Diagnostics: %globaltimer marks of the last persistent fit run with the
 * environment variable DNDC_PERSIST_TRACE set ([iteration][2*grid + 2]:
 * per-CTA tiles-done, per-CTA barrier-passed, CTA 0 start, CTA 0 update-done);
 * returns the number of marks copied (0 when none were recorded). */
int64_t dndc_kmeans_persist_trace(dndc_ctx* ctx, unsigned long long* out_host, int64_t cap, int* grid);

/* Measurement hook for bench.py's roofline: average duration of `reps`
 * back-to-back launches of the fused assign/accumulate kernel alone (CUDA
 * events on the context's stream) and its algorithmic bytes per launch
 * (n * m * 4: X read once). */
int dndc_kmeans_time_assign_f32(dndc_ctx* ctx, const float* x, int64_t n, int64_t m, int k, int reps,
                                double* ms_per_launch, double* algorithmic_bytes);

/* Measurement hook: with timing enabled, kmeans_fit records a CUDA event pair
 * around every assign/accumulate launch inside its graph; last_assign_ms then
 * returns the summed kernel time of the last fit and the launches it covers
 * (iterations that ran).  For bench.py's roofline; off by default. */
int dndc_kmeans_assign_timing(dndc_ctx* ctx, int enable);
int dndc_kmeans_last_assign_ms(const dndc_ctx* ctx, double* total_ms, int* launches);

/* -------------------------------------------------- A13-A14: moments */
/* local_moments_axis + combine + mean_axis/var_axis along split axis 0
 * (moments.cpp:33-52, :69-114, :126-140), collective.  Outputs (host, f64):
 * count, mean[m], m2[m] of the whole array, folded in rank order; the
 * caller derives var = m2 / (count - ddof) exactly like variance_from. */
int dndc_moments_axis0_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, int64_t m,
                           int64_t* count_host, double* mean_host, double* m2_host);
int dndc_moments_axis0_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, int64_t m,
                           int64_t* count_host, double* mean_host, double* m2_host);

/* ------------------------------------------------- A16: k-means++ seeding */
/* D^2 seeding as defined in DESIGN.md (not in the reference),
 * collective; k global row indices (host). */
int dndc_kmeanspp_indices_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local,
                              int64_t n_global, int64_t m, int k, uint64_t seed,
                              int64_t* indices_host);
int dndc_kmeanspp_indices_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local,
                              int64_t n_global, int64_t m, int k, uint64_t seed,
                              int64_t* indices_host);

#ifdef __cplusplus
}
#endif

#endif /* DNDC_H */
