/*
 * dnd_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load the
 * shared library built from this file (oracle/liboracle.so), and only as the
 * checker.  The product path never links it.
 *
 * Build: oracle/Makefile, `-O2 -ffp-contract=off` so that no multiply-add is
 * fused: the reference is built for baseline x86-64 (no FMA), so every
 * `acc += a * b` below must round the product before the add, as it does there.
 *
 * Citations are file:line into /root/reference/proj.
 */
#include "dnd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- common.hpp */

/* common.hpp:14-19 */
uint64_t dno_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* common.hpp:24-27 */
double dno_uniform01(uint64_t seed, uint64_t counter) {
    const uint64_t z = dno_splitmix64(seed ^ dno_splitmix64(counter));
    return (double)(z >> 11) * 0x1.0p-53;
}

/* ndarray.hpp:154-169: the flat index is i*stride0 + f with stride0 = m;
 * static_cast<float>(double) rounds to nearest (and may round up to 1.0f). */
void dno_fill_uniform_f32(uint64_t seed, int64_t row0, int64_t rows, int64_t m, float* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t f = 0; f < m; ++f) {
            const uint64_t flat = (uint64_t)(row0 + i) * (uint64_t)m + (uint64_t)f;
            out[i * m + f] = (float)dno_uniform01(seed, flat);
        }
}

void dno_fill_uniform_f64(uint64_t seed, int64_t row0, int64_t rows, int64_t m, double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t f = 0; f < m; ++f) {
            const uint64_t flat = (uint64_t)(row0 + i) * (uint64_t)m + (uint64_t)f;
            out[i * m + f] = dno_uniform01(seed, flat);
        }
}

/* ------------------------------------------------------------- chunking.cpp */

/* chunking.cpp:9-30: extent = n/p + (r < n%p); larger chunks on low ranks. */
int dno_chunk_map(int64_t n, int p, int64_t* offsets, int64_t* extents) {
    if (n < 0 || p < 1) return -1;
    const int64_t base = n / p, rem = n % p;
    int64_t off = 0;
    for (int r = 0; r < p; ++r) {
        const int64_t e = base + (r < rem ? 1 : 0);
        offsets[r] = off;
        extents[r] = e;
        off += e;
    }
    return 0;
}

/* ------------------------------------------------------------- pairwise.cpp */

/* pairwise.cpp:10-20: sequential acc += v*v from 0.0. */
void dno_row_norms(const double* x, int64_t rows, int64_t m, double* out) {
    for (int64_t i = 0; i < rows; ++i) {
        double acc = 0.0;
        const double* row = x + i * m;
        for (int64_t k = 0; k < m; ++k) acc += row[k] * row[k];
        out[i] = acc;
    }
}

/* matmul_local(a, transpose2d(b)) (ndarray.hpp:400-418): the i-k-j loop adds
 * a[i][k]*b[j][k] into out[i][j] for k = 0..m-1 starting from 0.0, i.e. a
 * sequential dot product per (i, j).  distance_block (pairwise.cpp:22-33):
 * sq = na + nb - 2.0 * g; g = sqrt(sq > 0 ? sq : 0). */
static double ref_dot(const double* a, const double* b, int64_t m) {
    double g = 0.0;
    for (int64_t k = 0; k < m; ++k) g += a[k] * b[k];
    return g;
}

static double ref_distance(double na, double nb, double g) {
    const double sq = na + nb - 2.0 * g;
    return sqrt(sq > 0.0 ? sq : 0.0);
}

void dno_distance_block(const double* a, const double* na, int64_t rows, const double* b,
                        const double* nb, int64_t cols, int64_t m, double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j)
            out[i * cols + j] = ref_distance(na[i], nb[j], ref_dot(a + i * m, b + j * m, m));
}

/* pairwise.cpp:37-85.  Round t on rank r holds the block that originated at
 * (r - t) mod p and fills that origin's column window; the self block has its
 * diagonal zeroed (:63-68).  Values do not depend on the round schedule, so
 * the simulation walks the ranks and rounds in order. */
int dno_cdist(const double* x, int64_t n, int64_t m, int p, double* out,
              int64_t* sendrecvs_per_rank) {
    if (n == 0 || p < 1) return -1;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    double* norms = (double*)malloc(sizeof(double) * (size_t)n);
    dno_chunk_map(n, p, off, ext);
    dno_row_norms(x, n, m, norms);
    for (int r = 0; r < p; ++r) {
        int origin = r;
        for (int round = 0; round < p; ++round) {
            for (int64_t i = 0; i < ext[r]; ++i) {
                const int64_t gi = off[r] + i;
                for (int64_t j = 0; j < ext[origin]; ++j) {
                    const int64_t gj = off[origin] + j;
                    double d = ref_distance(norms[gi], norms[gj], ref_dot(x + gi * m, x + gj * m, m));
                    if (origin == r && i == j) d = 0.0;
                    out[gi * n + gj] = d;
                }
            }
            origin = (origin + p - 1) % p;
        }
    }
    if (sendrecvs_per_rank) *sendrecvs_per_rank = p - 1;
    free(off);
    free(ext);
    free(norms);
    return 0;
}

/* pairwise.cpp:87-100: no diagonal handling, no communication. */
int dno_cdist_xy(const double* x, int64_t nx, const double* y, int64_t ny, int64_t m,
                 double* out) {
    double* xn = (double*)malloc(sizeof(double) * (size_t)(nx > 0 ? nx : 1));
    double* yn = (double*)malloc(sizeof(double) * (size_t)(ny > 0 ? ny : 1));
    dno_row_norms(x, nx, m, xn);
    dno_row_norms(y, ny, m, yn);
    dno_distance_block(x, xn, nx, y, yn, ny, m, out);
    free(xn);
    free(yn);
    return 0;
}

/* -------------------------------------------------------------- cluster.cpp */

/* cluster.cpp:60-75.  The reference shuffles an iota pool of n entries; only
 * positions touched by the k swaps differ from identity, so a sparse map of
 * touched positions reproduces pool[0..k) exactly in O(k) memory. */
typedef struct {
    int64_t* keys;
    int64_t* vals;
    size_t cap;
} sparse_pool;

static size_t sp_slot(const sparse_pool* sp, int64_t key) {
    size_t h = (size_t)(dno_splitmix64((uint64_t)key) & (sp->cap - 1));
    while (sp->keys[h] != -1 && sp->keys[h] != key) h = (h + 1) & (sp->cap - 1);
    return h;
}

static int64_t sp_get(const sparse_pool* sp, int64_t key) {
    const size_t h = sp_slot(sp, key);
    return sp->keys[h] == key ? sp->vals[h] : key;
}

static void sp_set(sparse_pool* sp, int64_t key, int64_t val) {
    const size_t h = sp_slot(sp, key);
    sp->keys[h] = key;
    sp->vals[h] = val;
}

int dno_kmeans_init_indices(int64_t n, int k, uint64_t seed, int64_t* out) {
    if (k < 1 || (int64_t)k > n) return -1;
    sparse_pool sp;
    sp.cap = 16;
    while (sp.cap < (size_t)k * 4) sp.cap <<= 1;
    sp.keys = (int64_t*)malloc(sizeof(int64_t) * sp.cap);
    sp.vals = (int64_t*)malloc(sizeof(int64_t) * sp.cap);
    for (size_t i = 0; i < sp.cap; ++i) sp.keys[i] = -1;
    for (int j = 0; j < k; ++j) {
        const uint64_t draw = dno_splitmix64(seed ^ dno_splitmix64(0x6b8b4567u + (uint64_t)j));
        const int64_t pick = j + (int64_t)(draw % (uint64_t)(n - j));
        const int64_t a = sp_get(&sp, j), b = sp_get(&sp, pick);
        sp_set(&sp, j, b);
        sp_set(&sp, pick, a);
    }
    for (int j = 0; j < k; ++j) out[j] = sp_get(&sp, j);
    free(sp.keys);
    free(sp.vals);
    return 0;
}

/* assign_local (cluster.cpp:44-56): strict <, lowest index wins ties.  The
 * distances are distance_block's, so the row norm and centroid norms enter
 * exactly as in pairwise.cpp:96-97. */
static int ref_assign(const double* row, double rn, const double* c, const double* cn, int k,
                      int64_t m, double* best_d) {
    int best = 0;
    double bd = ref_distance(rn, cn[0], ref_dot(row, c, m));
    for (int j = 1; j < k; ++j) {
        const double d = ref_distance(rn, cn[j], ref_dot(row, c + (int64_t)j * m, m));
        if (d < bd) {
            bd = d;
            best = j;
        }
    }
    *best_d = bd;
    return best;
}

/* Lloyd body of kmeans_fit, cluster.cpp:105-151, over p simulated ranks. */
int dno_kmeans_lloyd(const double* x, int64_t n, int64_t m, int p, int k, int max_iter,
                     double tol, double* centroids, double* inertia_trace, int* iterations_run) {
    if (k < 1 || (int64_t)k > n || max_iter < 1 || p < 1) return -1;
    const size_t km = (size_t)k * (size_t)m;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    double* stats = (double*)malloc(sizeof(double) * (km + (size_t)k));
    double* acc = (double*)malloc(sizeof(double) * (km + (size_t)k));
    double* next = (double*)malloc(sizeof(double) * km);
    double* cn = (double*)malloc(sizeof(double) * (size_t)k);
    dno_chunk_map(n, p, off, ext);
    int iters = 0;
    for (int iter = 0; iter < max_iter; ++iter) {
        dno_row_norms(centroids, k, m, cn); /* pairwise.cpp:97 on the replicated centroids */
        for (size_t i = 0; i < km + (size_t)k; ++i) acc[i] = 0.0; /* allreduce identity */
        double inertia = 0.0;
        for (int r = 0; r < p; ++r) {
            for (size_t i = 0; i < km + (size_t)k; ++i) stats[i] = 0.0;
            double local_inertia = 0.0;
            for (int64_t i = 0; i < ext[r]; ++i) {
                const double* row = x + (off[r] + i) * m;
                double rn;
                dno_row_norms(row, 1, m, &rn);
                double d;
                const int j = ref_assign(row, rn, centroids, cn, k, m, &d);
                double* dst = stats + (size_t)j * (size_t)m;
                for (int64_t f = 0; f < m; ++f) dst[f] += row[f];
                stats[km + (size_t)j] += 1.0;
                local_inertia += d * d;
            }
            /* plus_vec fold in rank order (cluster.cpp:21-24, transport.hpp:140-146) */
            for (size_t i = 0; i < km + (size_t)k; ++i) acc[i] += stats[i];
            inertia = inertia + local_inertia; /* cluster.cpp:135-136 */
        }
        memcpy(next, centroids, sizeof(double) * km);
        for (int j = 0; j < k; ++j) { /* cluster.cpp:125-133 */
            const double count = acc[km + (size_t)j];
            if (count > 0.0)
                for (int64_t f = 0; f < m; ++f)
                    next[(size_t)j * (size_t)m + (size_t)f] = acc[(size_t)j * (size_t)m + (size_t)f] / count;
        }
        inertia_trace[iter] = inertia;
        iters = iter + 1;
        double displacement = 0.0; /* cluster.cpp:139-150 */
        for (int j = 0; j < k; ++j) {
            double sq = 0.0;
            for (int64_t f = 0; f < m; ++f) {
                const double d = next[(size_t)j * (size_t)m + (size_t)f] - centroids[(size_t)j * (size_t)m + (size_t)f];
                sq += d * d;
            }
            const double s = sqrt(sq);
            displacement = displacement > s ? displacement : s;
        }
        memcpy(centroids, next, sizeof(double) * km);
        if (displacement < tol) break;
    }
    if (iterations_run) *iterations_run = iters;
    free(off);
    free(ext);
    free(stats);
    free(acc);
    free(next);
    free(cn);
    return 0;
}

/* kmeans_fit, cluster.cpp:83-153: validate (:85-89), init via
 * kmeans_init_indices + gather_rows (:100; the zero-filled allreduce-sum of
 * gather_rows replicates the rows exactly), then the Lloyd loop. */
int dno_kmeans_fit(const double* x, int64_t n, int64_t m, int p, int k, int max_iter,
                   double tol, uint64_t seed, double* centroids, double* inertia_trace,
                   int* iterations_run) {
    if (k < 1 || (int64_t)k > n || max_iter < 1 || p < 1) return -1;
    for (int64_t i = 0; i < n * m; ++i)
        if (!isfinite(x[i])) return -2;
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    dno_kmeans_init_indices(n, k, seed, idx);
    for (int j = 0; j < k; ++j) memcpy(centroids + (size_t)j * (size_t)m, x + idx[j] * m, sizeof(double) * (size_t)m);
    free(idx);
    return dno_kmeans_lloyd(x, n, m, p, k, max_iter, tol, centroids, inertia_trace, iterations_run);
}

/* cluster.cpp:155-172 */
void dno_kmeans_predict(const double* x, int64_t n, int64_t m, const double* centroids, int k,
                        int32_t* labels) {
    double* cn = (double*)malloc(sizeof(double) * (size_t)k);
    dno_row_norms(centroids, k, m, cn);
    for (int64_t i = 0; i < n; ++i) {
        double rn, d;
        dno_row_norms(x + i * m, 1, m, &rn);
        labels[i] = ref_assign(x + i * m, rn, centroids, cn, k, m, &d);
    }
    free(cn);
}

/* -------------------------------------------------------------- moments.cpp */

/* moments.cpp:10-14 */
static void welford_update(double x, double* mean, double* m2, int64_t n_after) {
    const double delta = x - *mean;
    *mean += delta / (double)n_after;
    *m2 += delta * (x - *mean);
}

/* moments.cpp:100-114 with AxisView(tile, 0): outer = 1, extent = rows, inner = m */
void dno_local_moments_axis0(const double* x, int64_t rows, int64_t m, int64_t* count,
                             double* mean, double* m2) {
    for (int64_t i = 0; i < m; ++i) mean[i] = m2[i] = 0.0;
    *count = rows;
    for (int64_t k = 0; k < rows; ++k)
        for (int64_t i = 0; i < m; ++i) welford_update(x[k * m + i], &mean[i], &m2[i], k + 1);
}

/* moments.cpp:100-114 fed in row blocks: the same sequential welford_update
 * chain as dno_local_moments_axis0 over rows [0, count_in + rows), continued
 * from the state (count, mean, m2) of the rows already seen.  Lets a test run
 * the reference's single-rank Welford over an array too large for host f64
 * (cfg5, 100M x 32) one fp32 block at a time; the values are widened exactly. */
void dno_welford_axis0_f32_continue(const float* x, int64_t rows, int64_t m, int64_t* count,
                                    double* mean, double* m2) {
    int64_t c = *count;
    for (int64_t k = 0; k < rows; ++k) {
        ++c;
        for (int64_t i = 0; i < m; ++i) welford_update((double)x[k * m + i], &mean[i], &m2[i], c);
    }
    *count = c;
}

/* moments.cpp:91-98 */
void dno_local_moments_flat(const double* x, int64_t numel, int64_t* count, double* mean,
                            double* m2) {
    int64_t c = 0;
    *mean = *m2 = 0.0;
    for (int64_t i = 0; i < numel; ++i) {
        ++c;
        welford_update(x[i], mean, m2, c);
    }
    *count = c;
}

/* moments.cpp:69-89 */
void dno_combine(int64_t* ca, double* ma, double* m2a, int64_t cb, const double* mb,
                 const double* m2b, int64_t arity) {
    if (*ca == 0) {
        *ca = cb;
        memcpy(ma, mb, sizeof(double) * (size_t)arity);
        memcpy(m2a, m2b, sizeof(double) * (size_t)arity);
        return;
    }
    if (cb == 0) return;
    const int64_t c = *ca + cb;
    const double na = (double)*ca, nb = (double)cb, nn = (double)c;
    for (int64_t i = 0; i < arity; ++i) {
        const double delta = mb[i] - ma[i];
        const double mean = ma[i] + delta * nb / nn;
        const double m2 = m2a[i] + m2b[i] + delta * delta * na * nb / nn;
        ma[i] = mean;
        m2a[i] = m2;
    }
    *ca = c;
}

/* axis_statistic split == axis branch (moments.cpp:41-52): local state (the
 * identity for an empty tile), allreduce(combine) folded in rank order from
 * the identity, then mean[i] or variance_from (:24-30). */
int dno_moments_axis0(const double* x, int64_t n, int64_t m, int p, int64_t ddof,
                      double* mean_out, double* var_out) {
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    double* lm = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double* lm2 = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double* gm = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    double* gm2 = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    int64_t gc = 0;
    dno_chunk_map(n, p, off, ext);
    for (int r = 0; r < p; ++r) {
        int64_t lc = 0;
        if (ext[r] * m > 0) {
            dno_local_moments_axis0(x + off[r] * m, ext[r], m, &lc, lm, lm2);
        } else {
            for (int64_t i = 0; i < m; ++i) lm[i] = lm2[i] = 0.0;
        }
        dno_combine(&gc, gm, gm2, lc, lm, lm2, m);
    }
    int rc = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (mean_out) mean_out[i] = gm[i];
        if (var_out) {
            if (gc - ddof <= 0) {
                rc = -1;
                break;
            }
            var_out[i] = gm2[i] / (double)(gc - ddof);
        }
    }
    free(off);
    free(ext);
    free(lm);
    free(lm2);
    free(gm);
    free(gm2);
    return rc;
}

/* ------------------------------------------------------------ k-means++ (A16)
 *
 * NOT in the reference (SPEC.md:413 defers k-means++).  This is the repo's own
 * definition, restated here so the CUDA kernels (csrc/kmeanspp.cu) have a
 * bit-exact checker; it reuses the reference's counter-based draws
 * (common.hpp:24-27) and its first pick (kmeans_init_indices(n, 1, seed)).
 *
 *   D2[i]   = min over chosen c of  sum_f ((double)x[i][f] - (double)c[f])^2
 *             (sequential over f, product rounded before the add)
 *   block   = 2048 consecutive rows; lane l (0..31) sums rows l, l+32, ...
 *             sequentially from 0.0, then a butterfly v += v[l ^ o] for
 *             o = 16, 8, 4, 2, 1 -> S_b
 *   group   = 1024 consecutive blocks; the same lane/butterfly scheme over S_b
 *             -> T_g
 *   W       = sequential sum of T_g over all groups
 *   draw j  : u = uniform01(seed ^ KPP_SALT, j); target = u * W
 *   pick    : first group with P + T_g > target (P = running sequential sum);
 *             then inside it the first block with Q + S_b > target - P; then
 *             inside it the first row with R + D2 > target - P - Q; when
 *             rounding leaves no candidate at a level, the last candidate with
 *             a positive weight is taken.  W == 0 picks row floor(u * n).
 */
#define KPP_BLOCK 2048
#define KPP_GROUP 1024
#define KPP_SALT 0x5851f42d4c957f2dULL

static double kpp_lane_sum(const double* v, int64_t count, int64_t stride_elems) {
    double lanes[32];
    for (int l = 0; l < 32; ++l) {
        double acc = 0.0;
        for (int64_t i = l; i < count; i += 32) acc += v[i * stride_elems];
        lanes[l] = acc;
    }
    for (int o = 16; o >= 1; o >>= 1) {
        double nxt[32];
        for (int l = 0; l < 32; ++l) nxt[l] = lanes[l] + lanes[l ^ o];
        memcpy(lanes, nxt, sizeof(lanes));
    }
    return lanes[0];
}

/* D2 of rows i and j of x (f32 or f64 elements, the same f64 chain) */
static double kpp_dist2(const void* x, int f64, int64_t i, int64_t j, int64_t m) {
    double acc = 0.0;
    for (int64_t f = 0; f < m; ++f) {
        const double d = f64 ? ((const double*)x)[i * m + f] - ((const double*)x)[j * m + f]
                             : (double)((const float*)x)[i * m + f] - (double)((const float*)x)[j * m + f];
        acc += d * d;
    }
    return acc;
}

static int kmeanspp_indices(const void* x, int f64, int64_t n, int64_t m, int p, int k, uint64_t seed,
                            int64_t* indices) {
    if (k < 1 || (int64_t)k > n || p < 1) return -1;
    /* blocks and groups are laid out per rank shard (chunk_map), concatenated
     * in rank order; p = 1 is one shard covering all rows. */
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    dno_chunk_map(n, p, off, ext);
    int64_t nblocks = 0, ngroups = 0;
    for (int r = 0; r < p; ++r) {
        const int64_t nb = (ext[r] + KPP_BLOCK - 1) / KPP_BLOCK;
        nblocks += nb;
        ngroups += (nb + KPP_GROUP - 1) / KPP_GROUP;
    }
    int64_t* blo = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nblocks + 1));
    int64_t* bcnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nblocks + 1));
    int64_t* g0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ngroups + 1));
    int64_t* g1 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ngroups + 1));
    {
        int64_t b = 0, g = 0;
        for (int r = 0; r < p; ++r) {
            const int64_t nb = (ext[r] + KPP_BLOCK - 1) / KPP_BLOCK;
            const int64_t first = b;
            for (int64_t i = 0; i < nb; ++i, ++b) {
                blo[b] = off[r] + i * KPP_BLOCK;
                bcnt[b] = (ext[r] - i * KPP_BLOCK) < KPP_BLOCK ? (ext[r] - i * KPP_BLOCK) : KPP_BLOCK;
            }
            for (int64_t s0 = first; s0 < b; s0 += KPP_GROUP, ++g) {
                g0[g] = s0;
                g1[g] = (s0 + KPP_GROUP) < b ? (s0 + KPP_GROUP) : b;
            }
        }
    }
    double* d2 = (double*)malloc(sizeof(double) * (size_t)n);
    double* S = (double*)malloc(sizeof(double) * (size_t)(nblocks + 1));
    double* T = (double*)malloc(sizeof(double) * (size_t)(ngroups + 1));
    dno_kmeans_init_indices(n, 1, seed, &indices[0]);
    for (int64_t i = 0; i < n; ++i) d2[i] = kpp_dist2(x, f64, i, indices[0], m);
    for (int j = 1; j < k; ++j) {
        for (int64_t b = 0; b < nblocks; ++b) S[b] = kpp_lane_sum(d2 + blo[b], bcnt[b], 1);
        double W = 0.0;
        for (int64_t g = 0; g < ngroups; ++g) {
            T[g] = kpp_lane_sum(S + g0[g], g1[g] - g0[g], 1);
            W += T[g];
        }
        const double u = dno_uniform01(seed ^ KPP_SALT, (uint64_t)j);
        int64_t pick;
        if (!(W > 0.0)) {
            pick = (int64_t)(u * (double)n);
            if (pick >= n) pick = n - 1;
        } else {
            const double target = u * W;
            double P = 0.0, Plast = 0.0;
            int64_t g = -1, glast = -1;
            for (int64_t gg = 0; gg < ngroups; ++gg) {
                if (T[gg] > 0.0) { glast = gg; Plast = P; }
                if (P + T[gg] > target) { g = gg; break; }
                P += T[gg];
            }
            if (g < 0) { g = glast; P = Plast; }
            const double t1 = target - P;
            double Q = 0.0, Qlast = 0.0;
            int64_t b = -1, blast = -1;
            for (int64_t bb = g0[g]; bb < g1[g]; ++bb) {
                if (S[bb] > 0.0) { blast = bb; Qlast = Q; }
                if (Q + S[bb] > t1) { b = bb; break; }
                Q += S[bb];
            }
            if (b < 0) { b = blast; Q = Qlast; }
            const double t2 = t1 - Q;
            double R = 0.0;
            int64_t row = -1, rlast = -1;
            for (int64_t i = blo[b]; i < blo[b] + bcnt[b]; ++i) {
                if (d2[i] > 0.0) rlast = i;
                if (R + d2[i] > t2) { row = i; break; }
                R += d2[i];
            }
            pick = row >= 0 ? row : rlast;
        }
        indices[j] = pick;
        for (int64_t i = 0; i < n; ++i) {
            const double d = kpp_dist2(x, f64, i, pick, m);
            if (d < d2[i]) d2[i] = d;
        }
    }
    free(off); free(ext); free(blo); free(bcnt); free(g0); free(g1);
    free(d2); free(S); free(T);
    return 0;
}

int dno_kmeanspp_indices_f32(const float* x, int64_t n, int64_t m, int p, int k, uint64_t seed,
                             int64_t* indices) {
    return kmeanspp_indices(x, 0, n, m, p, k, seed, indices);
}

int dno_kmeanspp_indices_f64(const double* x, int64_t n, int64_t m, int p, int k, uint64_t seed,
                             int64_t* indices) {
    return kmeanspp_indices(x, 1, n, m, p, k, seed, indices);
}

/* ------------------------------------------------------------ LASSO (F4)
 *
 * Cyclic coordinate descent, regression.cpp:25-102: every rank owns the
 * chunk-map rows of x (bias column 0 all ones) and their residual; column
 * squared norms and, per coordinate, the correlation rho are summed over
 * ranks in rank order from 0.0 (allreduce(plus), transport.hpp:140-146);
 * w_0 = rho / sq_0, w_j = soft_threshold(rho, lambda / 2) / sq_j; columns with
 * zero norm are skipped; one objective |r|^2 + lambda sum_{j>0} |w_j| per
 * sweep; stop when the largest change < tol.  Returns -1 on invalid
 * arguments, -2 when column 0 is not all ones. */

/* regression.cpp:19-23 */
double dno_soft_threshold(double rho, double t) {
    if (rho > t) return rho - t;
    if (rho < -t) return rho + t;
    return 0.0;
}

int dno_lasso_fit(const double* x, const double* y, int64_t n, int64_t m, int p, double lambda, int sweeps,
                  double tol, double* weights, double* trace, int* sweeps_run) {
    if (n < 1 || m < 1 || lambda < 0.0 || sweeps < 1 || p < 1) return -1;
    for (int64_t i = 0; i < n; ++i)
        if (x[i * m] != 1.0) return -2;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    dno_chunk_map(n, p, off, ext);
    double* sq = (double*)calloc((size_t)m, sizeof(double));
    double* sql = (double*)malloc(sizeof(double) * (size_t)m);
    double* res = (double*)malloc(sizeof(double) * (size_t)n);
    for (int r = 0; r < p; ++r) { /* regression.cpp:52-60 per rank, then the fold */
        for (int64_t j = 0; j < m; ++j) sql[j] = 0.0;
        for (int64_t i = off[r]; i < off[r] + ext[r]; ++i)
            for (int64_t j = 0; j < m; ++j) sql[j] += x[i * m + j] * x[i * m + j];
        for (int64_t j = 0; j < m; ++j) sq[j] += sql[j];
    }
    for (int64_t i = 0; i < n; ++i) res[i] = y[i];
    for (int64_t j = 0; j < m; ++j) weights[j] = 0.0;
    int run = 0;
    for (int s = 0; s < sweeps; ++s) {
        double max_change = 0.0;
        for (int64_t j = 0; j < m; ++j) {
            if (sq[j] == 0.0) continue;
            const double w_old = weights[j];
            double rho = 0.0;
            for (int r = 0; r < p; ++r) { /* regression.cpp:73-78 */
                double loc = 0.0;
                for (int64_t i = off[r]; i < off[r] + ext[r]; ++i) {
                    const double xij = x[i * m + j];
                    loc += xij * (res[i] + w_old * xij);
                }
                rho += loc;
            }
            const double w_new = j == 0 ? rho / sq[0] : dno_soft_threshold(rho, lambda / 2.0) / sq[j];
            if (w_new != w_old) { /* regression.cpp:83-88 */
                const double shift = w_old - w_new;
                for (int64_t i = 0; i < n; ++i) res[i] += shift * x[i * m + j];
                weights[j] = w_new;
            }
            const double ch = fabs(w_new - w_old);
            if (ch > max_change) max_change = ch;
        }
        double ssr = 0.0; /* regression.cpp:92-99 */
        for (int r = 0; r < p; ++r) {
            double loc = 0.0;
            for (int64_t i = off[r]; i < off[r] + ext[r]; ++i) loc += res[i] * res[i];
            ssr += loc;
        }
        double pen = 0.0;
        for (int64_t j = 1; j < m; ++j) pen += fabs(weights[j]);
        trace[s] = ssr + lambda * pen;
        run = s + 1;
        if (max_change < tol) break;
    }
    *sweeps_run = run;
    free(off);
    free(ext);
    free(sq);
    free(sql);
    free(res);
    return 0;
}
