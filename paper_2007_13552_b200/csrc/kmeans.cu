// kmeans.cu -- A8-A12: the fused Lloyd iteration.
//
// Reference: kmeans_fit / assign_local / gather_rows / kmeans_predict
// (cluster.cpp:27-172) on top of cdist_xy (pairwise.cpp:87-100).
//
// Which kernels run a fit (plan<T>, plan_persist; the choice depends only on
// global facts, so every rank takes the same one):
//
//   persistent  (fp32, the cfg1 shape d = 18, k = 8; kmeans_persist.cuh) the
//               whole Lloyd loop in two cooperative launches -- iteration 0
//               sums every row, the delta launch only the rows whose label
//               changed -- with a grid barrier per iteration and, for
//               world > 1, an NVLink exchange of the rank stats inside the
//               kernel.  No relaunch, no host round trip.
//   tc          (k d >= 1024, cfg3; kmeans_tc.cuh) per iteration in one CUDA
//               graph: the tcgen05 3xTF32 scores/labels kernel, the refine
//               kernel (near-ties decided exactly, changed rows summed), the
//               accumulate kernel for full iterations, reduce + update.
//   small / generic  the other shapes: one assign(+accumulate) launch per
//               iteration (fused with the update on one GPU or over NVLink),
//               else assign -> reduce -> NCCL allgather -> update.
//
// Common to all: fp32 scores s_j = |c_j|^2 - 2 x.c_j with a rigorous error
// bound; rows whose top-2 gap falls inside it are re-decided with the
// reference's exact f64 arithmetic (distance_block + assign_local, products
// rounded before adds, strict < so the lowest index wins ties).  Sums are
// int64 fixed point (order-independent: the fit is bit-repeatable), folded
// over ranks in rank order 0..p-1 (transport.hpp:136-148); the update forms
// the f64 master centroids (empty clusters keep theirs, cluster.cpp:125-133),
// the inertia and the displacement (cluster.cpp:139-150).
//
// Inertia is not accumulated per row: with S_j, n_j the new sums/counts and c_j
// the centroids used for the assignment,
//     sum_i |x_i - c_l(i)|^2 = sum_i |x_i|^2 + sum_j (n_j |c_j|^2 - 2 c_j.S_j),
// and sum_i |x_i|^2 is computed once per fit by the validation pass that the
// reference performs anyway (the isfinite scan, cluster.cpp:88-89).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc.cuh"

namespace dndc {

constexpr int KM_THREADS = 256;
constexpr int KM_WARPS = KM_THREADS / 32;
constexpr int KM_TILE = 256;  // rows per tile: one per thread in phase 1
constexpr unsigned FULL = 0xffffffffu;

struct KMeansState {
    // instantiated fit graphs, most recent first (e.g. two alternating input
    // buffers of a pipelined caller); keyed on shape, buffers and slot_gen
    std::vector<std::pair<std::string, cudaGraphExec_t>> graphs;
    void clear_graphs() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.second);
        graphs.clear();
    }
    // dndc_kmeans_assign_timing: event pairs recorded around every assign
    // launch inside the fit graph (external event nodes)
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    double assign_ms = 0.0;
    int assign_launches = 0;
    std::vector<double> per_launch_ms;
};

static void free_events(KMeansState* st) {
    for (cudaEvent_t e : st->ev) cudaEventDestroy(e);
    st->ev.clear();
}

void destroy_kmeans_state(KMeansState* st) {
    if (!st) return;
    free_events(st);
    st->clear_graphs();
    delete st;
}

// Device buffers of the Lloyd state (ctx slots, stable addresses for graphs).
struct KmBuffers {
    double* c64;       // k*m f64 master centroids
    double* cn64;      // k   reference-order |c|^2 of c64
    float* ct;         // k*dpad  -2 * float(c64)
    float* cn32;       // k   float(|float(c)|^2)
    float* bounds;     // [0] max_j |c_j|, [1] max_j cn32_j
    double* stats;     // S = k*m + k local reduced stats
    double* gathered;  // world * S
    double* partials;  // G * S
    double* trace;     // max_iter
    double* disp;      // max_iter
    int* flags;        // [0] done, [1] iterations_run
    double* sx2;       // [0] local sum x^2, [1] non-finite count, [2] global sum x^2
    double* pre;       // validation partials
    float* ctab;       // K*D + K constant-bank layout of the fp32 table
    unsigned long long* refined;
    double* running;   // S running sums/counts of the delta iterations
    unsigned long long* acc64;  // fused tail: fixed-point stats accumulator
    unsigned* counters;  // [0] fused-tail arrival ticket, [1] tile counter
};

static int dpad_of(int m) { return (m + 3) / 4 * 4; }

// Row stride of a staged tile in shared memory.  Rows whose 16-byte chunks are
// whole (m % 4 == 0) are padded so that lane = row reads hit distinct bank
// groups (stride/4 odd); other widths are copied contiguously (m = 18 reads
// conflict-free as 8-byte pairs).
static int srow_of(int m) {
    if (m % 4 != 0) return m;
    return ((m / 4) % 2 == 0) ? m + 4 : m;
}

struct SmemLayout {
    size_t acc, cnt, cts, cns, lbl, total;
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) / 16 * 16; }

__host__ __device__ inline SmemLayout smem_layout(size_t elem, int k, int d, int srow, int dpad,
                                                  int stages) {
    SmemLayout l;
    l.acc = align16(static_cast<size_t>(stages) * KM_TILE * srow * elem);
    l.cnt = align16(l.acc + static_cast<size_t>(k) * d * sizeof(double));
    l.cts = align16(l.cnt + static_cast<size_t>(k) * sizeof(long long));
    const size_t ctab = elem == 4 ? static_cast<size_t>(k) * dpad * sizeof(float) : 0;
    l.cns = align16(l.cts + ctab);
    l.lbl = align16(l.cns + (elem == 4 ? static_cast<size_t>(k) * sizeof(float) : 0));
    l.total = align16(l.lbl + KM_TILE * sizeof(int));
    return l;
}

struct AssignParams {
    const void* x;
    int64_t n;
    int d, k, dpad, srow, stages;
    bool aligned16;
    const float* ct;
    const float* cn32;
    const float* bounds;
    const double* c64;
    const double* cn64;
    double* partials;  // null: predict only
    int32_t* labels;   // optional
    unsigned long long* refined;
    const int* done;
};

// Exact reference decision for one row held in shared memory (cluster.cpp:44-56
// over pairwise.cpp:22-33 and :96-97).
template <typename T>
__device__ int ref_argmin(const T* xr, int d, const double* __restrict__ c64,
                          const double* __restrict__ cn64, int k) {
    double xn = 0.0;
    for (int f = 0; f < d; ++f) {
        const double v = static_cast<double>(xr[f]);
        xn = add_rn(xn, mul_rn(v, v));
    }
    int best = 0;
    double bd = 0.0;
    for (int j = 0; j < k; ++j) {
        const double* c = c64 + static_cast<int64_t>(j) * d;
        double g = 0.0;
        for (int f = 0; f < d; ++f) g = add_rn(g, mul_rn(static_cast<double>(xr[f]), c[f]));
        const double dj = ref_distance(xn, cn64[j], g);
        if (j == 0 || dj < bd) {
            bd = dj;
            best = j;
        }
    }
    return best;
}

// Same decision for a row held in registers (compile-time width).
template <int D>
__device__ __noinline__ int ref_argmin_regs(const float (&xv)[D], const double* __restrict__ c64,
                                            const double* __restrict__ cn64, int k) {
    double xn = 0.0;
#pragma unroll
    for (int f = 0; f < D; ++f) xn = add_rn(xn, mul_rn(static_cast<double>(xv[f]), static_cast<double>(xv[f])));
    int best = 0;
    double bd = 0.0;
    for (int j = 0; j < k; ++j) {
        const double* c = c64 + static_cast<int64_t>(j) * D;
        double g = 0.0;
#pragma unroll
        for (int f = 0; f < D; ++f) g = add_rn(g, mul_rn(static_cast<double>(xv[f]), c[f]));
        const double dj = ref_distance(xn, cn64[j], g);
        if (j == 0 || dj < bd) {
            bd = dj;
            best = j;
        }
    }
    return best;
}

// Exact reference decision restricted to a candidate set (bit j of `cand`):
// every cluster outside it is provably farther (its fp32 score exceeds the
// best by more than the error bound), so the lowest-index minimiser over the
// candidates, visited in ascending order with strict <, is the reference's
// assign_local choice (cluster.cpp:44-56).
template <int D>
__device__ __noinline__ int ref_argmin_cand(const float (&xv)[D], uint64_t cand, const double* __restrict__ c64,
                                            const double* __restrict__ cn64) {
    double xn = 0.0;
#pragma unroll
    for (int f = 0; f < D; ++f) xn = add_rn(xn, mul_rn(static_cast<double>(xv[f]), static_cast<double>(xv[f])));
    int best = -1;
    double bd = 0.0;
    while (cand) {
        const int j = __ffsll(static_cast<long long>(cand)) - 1;
        cand &= cand - 1;
        const double* c = c64 + static_cast<int64_t>(j) * D;
        double g = 0.0;
#pragma unroll
        for (int f = 0; f < D; ++f) g = add_rn(g, mul_rn(static_cast<double>(xv[f]), c[f]));
        const double dj = ref_distance(xn, cn64[j], g);
        if (best < 0 || dj < bd) {
            bd = dj;
            best = j;
        }
    }
    return best;
}

template <typename T>
__device__ __forceinline__ void load_tile(T* dst, const T* __restrict__ x, int64_t n, int d, int srow,
                                          int64_t tile, bool aligned16) {
    const int64_t row0 = tile * KM_TILE;
    const int64_t rows = min(static_cast<int64_t>(KM_TILE), n - row0);
    const T* src = x + row0 * d;
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte chunk
    if (aligned16 && srow == d) {
        const int64_t valid = rows * d * static_cast<int64_t>(sizeof(T));
        const int chunks = KM_TILE * d * static_cast<int>(sizeof(T)) / 16;
        for (int c = threadIdx.x; c < chunks; c += KM_THREADS) {
            const int64_t rem = valid - static_cast<int64_t>(c) * 16;
            const int bytes = rem >= 16 ? 16 : (rem > 0 ? static_cast<int>(rem) : 0);
            cp_async16(dst + c * V, bytes > 0 ? src + c * V : x, bytes);
        }
    } else if (aligned16 && d % V == 0) {
        const int per_row = d / V;
        for (int c = threadIdx.x; c < KM_TILE * per_row; c += KM_THREADS) {
            const int r = c / per_row, q = c % per_row;
            const bool ok = r < rows;
            cp_async16(dst + r * srow + q * V, ok ? src + static_cast<int64_t>(r) * d + q * V : x,
                       ok ? 16 : 0);
        }
    } else {
        for (int e = threadIdx.x; e < KM_TILE * d; e += KM_THREADS) {
            const int r = e / d, f = e % d;
            if (r < rows) {
                if constexpr (sizeof(T) == 4)
                    cp_async4(dst + r * srow + f, src + static_cast<int64_t>(r) * d + f);
                else
                    cp_async8(dst + r * srow + f, src + static_cast<int64_t>(r) * d + f);
            }
            else
                dst[r * srow + f] = T(0);
        }
    }
}

// D > 0: compile-time feature count (row kept in registers); D == 0: runtime.
template <typename T, int D>
__global__ void __launch_bounds__(KM_THREADS) kmeans_assign_kernel(AssignParams p) {
    if (p.done && *p.done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int d = D > 0 ? D : p.d;
    const int k = p.k;
    const int srow = p.srow;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---- carve shared memory (layout shared with assign_smem on the host)
    const SmemLayout lay = smem_layout(sizeof(T), k, d, srow, p.dpad, p.stages);
    T* xs = reinterpret_cast<T*>(smem_raw);
    const size_t stage_elems = static_cast<size_t>(KM_TILE) * srow;
    double* acc = reinterpret_cast<double*>(smem_raw + lay.acc);
    long long* cnt = reinterpret_cast<long long*>(smem_raw + lay.cnt);
    float* cts = reinterpret_cast<float*>(smem_raw + lay.cts);
    float* cns = reinterpret_cast<float*>(smem_raw + lay.cns);
    int* lbl = reinterpret_cast<int*>(smem_raw + lay.lbl);

    const bool accumulate = p.partials != nullptr;
    if (accumulate) {
        for (int e = threadIdx.x; e < k * d; e += KM_THREADS) acc[e] = 0.0;
        for (int j = threadIdx.x; j < k; j += KM_THREADS) cnt[j] = 0;
    }
    if constexpr (sizeof(T) == 4) {
        for (int e = threadIdx.x; e < k * p.dpad; e += KM_THREADS) cts[e] = p.ct[e];
        for (int j = threadIdx.x; j < k; j += KM_THREADS) cns[j] = p.cn32[j];
    }
    const float cmax = sizeof(T) == 4 ? p.bounds[0] : 0.f;
    const float cnmax = sizeof(T) == 4 ? p.bounds[1] : 0.f;
    const float tau_scale = 4.f * static_cast<float>(d + 3) * 0x1.0p-24f;

    const T* __restrict__ x = static_cast<const T*>(p.x);
    const int64_t ntiles = ceil_div(p.n, KM_TILE);
    const int64_t my_tiles =
        blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // prologue: stages-1 tiles in flight
    for (int s = 0; s < p.stages - 1; ++s) {
        if (s < my_tiles)
            load_tile<T>(xs + s * stage_elems, x, p.n, d, srow, blockIdx.x + s * gridDim.x, p.aligned16);
        cp_async_commit();
    }
    unsigned long long refined = 0;

    for (int64_t it = 0; it < my_tiles; ++it) {
        const int64_t tile = blockIdx.x + it * gridDim.x;
        const int stage = p.stages ? static_cast<int>(it % p.stages) : 0;
        // wait until at most stages-2 younger groups are pending -> tile `it` landed
        if (p.stages == 2) cp_async_wait<0>();
        else if (p.stages == 3) cp_async_wait<1>();
        else cp_async_wait<2>();
        __syncthreads();
        if (p.stages > 0) {
            const int64_t nxt = it + p.stages - 1;
            if (nxt < my_tiles)
                load_tile<T>(xs + ((it + p.stages - 1) % p.stages) * stage_elems, x, p.n, d, srow,
                             blockIdx.x + nxt * gridDim.x, p.aligned16);
            cp_async_commit();
        }
        // stages == 0 (rows too wide to stage): read the tile straight from HBM/L2
        const T* xt = p.stages ? xs + stage * stage_elems : x + tile * KM_TILE * d;

        // ---------------- phase 1: lane = row
        const int row = threadIdx.x;
        const int64_t grow = tile * KM_TILE + row;
        int label = -1;
        if (grow < p.n) {
            const T* xr = xt + row * srow;
            if constexpr (sizeof(T) == 4) {
                float b1 = FLT_MAX, b2 = FLT_MAX, xx = 0.f;
                int i1 = 0;
                if constexpr (D > 0) {
                    float xv[D];
                    if constexpr (D % 2 == 0) {
#pragma unroll
                        for (int f = 0; f < D; f += 2) {
                            const float2 v = *reinterpret_cast<const float2*>(xr + f);
                            xv[f] = v.x;
                            xv[f + 1] = v.y;
                        }
                    } else {
#pragma unroll
                        for (int f = 0; f < D; ++f) xv[f] = xr[f];
                    }
#pragma unroll
                    for (int f = 0; f < D; ++f) xx = fmaf(xv[f], xv[f], xx);
                    for (int j = 0; j < k; ++j) {
                        const float* c = cts + j * p.dpad;
                        float s = cns[j];
#pragma unroll
                        for (int f = 0; f < (D & ~3); f += 4) {
                            const float4 cv = *reinterpret_cast<const float4*>(c + f);
                            s = fmaf(xv[f], cv.x, s);
                            s = fmaf(xv[f + 1], cv.y, s);
                            s = fmaf(xv[f + 2], cv.z, s);
                            s = fmaf(xv[f + 3], cv.w, s);
                        }
#pragma unroll
                        for (int f = D & ~3; f < D; ++f) s = fmaf(xv[f], c[f], s);
                        if (s < b1) {
                            b2 = b1;
                            b1 = s;
                            i1 = j;
                        } else if (s < b2) {
                            b2 = s;
                        }
                    }
                } else {
                    for (int f = 0; f < d; ++f) xx = fmaf(xr[f], xr[f], xx);
                    for (int j = 0; j < k; ++j) {
                        const float* c = cts + j * p.dpad;
                        float s = cns[j];
                        for (int f = 0; f < d; ++f) s = fmaf(xr[f], c[f], s);
                        if (s < b1) {
                            b2 = b1;
                            b1 = s;
                            i1 = j;
                        } else if (s < b2) {
                            b2 = s;
                        }
                    }
                }
                label = i1;
                // |s_j - exact_j| <= (d+3) u (|c_j|^2 + 2 |x||c_j|) for both
                // candidates; 2x safety on the sum of the two bounds.
                const float tau = tau_scale * (cnmax + 2.f * sqrtf(xx) * cmax);
                if (k > 1 && !(b2 - b1 > tau)) {
                    label = ref_argmin<T>(xr, d, p.c64, p.cn64, k);
                    ++refined;
                }
            } else {
                label = ref_argmin<T>(xr, d, p.c64, p.cn64, k);
            }
            if (p.labels) p.labels[grow] = label;
        }
        lbl[row] = label;
        __syncthreads();

        // ---------------- phase 2: lane = feature, warp owns clusters
        if (accumulate) {
            for (int j = warp; j < k; j += KM_WARPS) {
                long long cj = 0;
#pragma unroll 1
                for (int c = 0; c < KM_TILE / 32; ++c) {
                    const unsigned mask = __ballot_sync(FULL, lbl[c * 32 + lane] == j);
                    if (mask == 0u) continue;
                    cj += __popc(mask);
                    for (int fb = 0; fb < d; fb += 32) {
                        const int f = fb + lane;
                        if (f < d) {
                            // f64 from the first term: fp32 run sums would put
                            // ~1e-7 relative error into the centroids
                            double part = 0.0;
                            unsigned mm = mask;
                            while (mm) {
                                const int r = __ffs(mm) - 1;
                                mm &= mm - 1;
                                part += static_cast<double>(xt[(c * 32 + r) * srow + f]);
                            }
                            acc[j * d + f] += part;
                        }
                    }
                }
                if (lane == 0) cnt[j] += cj;
            }
        }
    }
    cp_async_wait<0>();
    if (refined) atomicAdd(p.refined, refined);
    if (!accumulate) return;
    __syncthreads();
    const int S = k * d + k;
    double* out = p.partials + static_cast<int64_t>(blockIdx.x) * S;
    for (int e = threadIdx.x; e < k * d; e += KM_THREADS) out[e] = acc[e];
    for (int j = threadIdx.x; j < k; j += KM_THREADS) out[k * d + j] = static_cast<double>(cnt[j]);
}

// ============================================================================
// Specialised assign/accumulate for small compile-time (D, K) -- BASELINE
// config 1 (D = 18, K = 8) and the 32-feature config 5 data.
//
//  * X tiles (256 rows) stream HBM -> smem through a 4-stage ring of 1-D bulk
//    copies (cp.async.bulk + mbarrier complete_tx), issued by one thread.
//  * The centroid table (-2 c_j, |c_j|^2 in fp32) lives in the constant bank,
//    refreshed per iteration by a D2D memcpy node of the graph, so every score
//    FFMA reads its centroid operand from c[][] (no shared-memory traffic).
//  * Phase 1 (lane = row): K*D FFMA, top-2, the fp32 error bound and the f64
//    re-decision of near-ties (same rule as the generic kernel; the bound uses
//    the per-shard max |x_e| * sqrt(D) instead of |x_i|).
//  * Phase 2: a CTA-wide counting sort of the tile by label (ballots, a
//    per-warp prefix over the count table, one row scatter), then warp w sums
//    the sorted positions [32w, 32w+32): runs of one cluster, read as float2 by
//    groups of D/2 lanes, fp32 within the run (<= 32 rows), f64 per warp.
// Deterministic: every sum has a fixed order for a given grid.
// ============================================================================
constexpr int KS_SLOTS = 4;
constexpr int KS_TABLE = 1152;  // floats per slot (K*D + K)
__constant__ float c_km_table[KS_SLOTS * KS_TABLE];

struct UpdArgs {
    int k, d, dpad, world;
    const double* gathered;  // world per-rank stats, folded here in rank order
    int64_t gstride;         // doubles between two ranks' stats in `gathered`
    double* running;         // delta iterations: running sums/counts (or null)
    int accum;               // 1: gathered holds changes, added to running
    double *c64, *cn64;
    float *ct, *cn32, *ctab, *bounds;
    const double* sx2;
    double *trace, *disp;
    int* flags;
    int iter;
    double tol;
    // where the update reads running / c64 / cn64 / sx2 (the fused tail points
    // these at shared-memory copies it prefetched; otherwise the arrays above)
    const double *rd_running, *rd_c64, *rd_cn64, *rd_sx2;
};

__device__ void update_body(const UpdArgs& a, double* upd, double* sh);

// Fused tail of the small kernel (world == 1, or NVLink peer exchange): every
// CTA adds its partial stats into one fixed-point int64 accumulator (integer
// adds are associative: the result does not depend on arrival order); the
// last CTA to arrive converts them back to f64, stores the rank's stats into
// every rank's exchange region, waits for every rank's arrival flag and runs
// the update -- the whole Lloyd iteration in one launch.
struct FuseArgs {
    int on;
    unsigned long long* acc64;  // [S] fixed-point sums, zero between launches
    const double* xabs;   // max |x_e| of the shard (sets the fixed-point scale)
    int64_t n;            // rows of the shard
    unsigned* counters;   // [1] arrival ticket, zero between launches
    double* stats;        // [S] this rank's stats
    void* const* peers;   // [world] exchange regions (world > 1)
    int rank;
    unsigned* tile_ctr;   // reset with the tickets
    UpdArgs upd;
};

struct SmallParams {
    const float* x;
    int64_t n;
    const double* c64;
    const double* cn64;
    const float* bounds;  // [0] max |c_j|, [1] max |c_j|^2
    const double* xabs;   // max |x_e| of the shard
    double* partials;     // null: predict only
    int32_t* labels;
    const int8_t* prev;   // delta mode: last iteration's labels (partials = sum deltas)
    int8_t* lab8;         // this iteration's labels (fit), or null
    unsigned long long* refined;
    const int* done;
    unsigned* tile_ctr;   // delta mode: dynamic tile scheduling (zero at launch)
    FuseArgs fu;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// try_wait with a suspend-time hint (ns): the warp sleeps until the phase
// completes instead of re-polling (the plain poll loop was ~40 issue slots per
// 32 rows of the k-means kernels under ncu, r2).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// The row stream X of the bulk-copy k-means kernels: with DNDC_X_EVICT_FIRST
// its copies carry an L2 evict_first policy (X is re-read only an iteration
// later, after hundreds of MB; labels, stats and tables stay in L2).  Neutral
// for the persistent cfg1 kernel (tools/gpu_var_xev.sh), so off by default;
// the tensor-core path's TMA tiles take it by default (kmeans_tc.cuh).
#ifdef DNDC_X_EVICT_FIRST
#define X_BULK_HINT ".L2::cache_hint"
#define X_BULK_POL , "l"(tc::l2_policy_evict_first())
#define X_BULK_OPS ", %4"
#else
#define X_BULK_HINT ""
#define X_BULK_POL
#define X_BULK_OPS ""
#endif

// One thread: stream `bytes` (any multiple of 4) of global memory into smem,
// completing on `bar`.  The 16-byte-aligned body goes through the bulk-copy
// engine; a <16-byte tail is stored directly before the arrive.
__device__ __forceinline__ void bulk_load(float* dst, const float* src, uint32_t bytes, uint64_t* bar) {
    const uint32_t body = bytes & ~15u;
    for (uint32_t b = body; b < bytes; b += 4) dst[b / 4] = src[b / 4];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(body)
                 : "memory");
    if (body)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes" X_BULK_HINT " [%0], [%1], %2, [%3]" X_BULK_OPS ";" ::"r"(
                smem_u32(dst)),
            "l"(src), "r"(body), "r"(smem_u32(bar)) X_BULK_POL
            : "memory");
}

// Same, plus a second byte segment (the tile's previous labels) on the same barrier.
__device__ __forceinline__ void bulk_load2(float* dst, const float* src, uint32_t bytes, int8_t* dst2,
                                           const int8_t* src2, uint32_t bytes2, uint64_t* bar) {
    const uint32_t body = bytes & ~15u, body2 = bytes2 & ~15u;
    for (uint32_t b = body; b < bytes; b += 4) dst[b / 4] = src[b / 4];
    for (uint32_t b = body2; b < bytes2; ++b) dst2[b] = src2[b];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(body + body2)
                 : "memory");
    if (body)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes" X_BULK_HINT " [%0], [%1], %2, [%3]" X_BULK_OPS ";" ::"r"(
                smem_u32(dst)),
            "l"(src), "r"(body), "r"(smem_u32(bar)) X_BULK_POL
            : "memory");
    if (body2)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(dst2)),
            "l"(src2), "r"(body2), "r"(smem_u32(bar))
            : "memory");
}

// CTA shape of the small kernel: 128 threads (4 warps), each thread deciding
// KS_R rows per tile (KS_R * 128-row tiles): the constant-bank operands, the
// per-tile scan and the per-cluster loops are amortised over more rows while
// the per-tile barriers stay cheap (4 warps).
#ifdef KS_THREADS_OVR
constexpr int KS_THREADS = KS_THREADS_OVR;
#else
constexpr int KS_THREADS = 128;
#endif
constexpr int KS_WARPS = KS_THREADS / 32;
#ifdef KS_R_OVR
constexpr int KS_R = KS_R_OVR;
#else
constexpr int KS_R = 2;
#endif
constexpr int KS_TILE = KS_THREADS * KS_R;
#ifdef KS_STAGES_OVR
constexpr int KS_STAGES = KS_STAGES_OVR;
#else
constexpr int KS_STAGES = 2;
#endif
#ifdef KS_MIN_CTAS_OVR
constexpr int KS_MIN_CTAS = KS_MIN_CTAS_OVR;
#else
constexpr int KS_MIN_CTAS = 4;
#endif
constexpr int KS_VW = KS_WARPS * KS_R;  // 32-row groups per tile
constexpr int KS_SCR = 8;               // changed rows staged per warp and batch (delta mode)
#ifndef KS_FULL_ITERS
#define KS_FULL_ITERS 2  // iterations that accumulate every row (labels still moving a lot)
#endif
#ifndef KS_DONLY_CTAS
#define KS_DONLY_CTAS 4
#endif

#ifdef KS_TAIL_TRACE
__device__ unsigned long long g_tail_trace[16];
__device__ unsigned long long g_cta_trace[2 * 2048];
__device__ unsigned long long g_iter_trace[2 * 64];  // per iteration: CTA 0 start, update done
__device__ __forceinline__ void iter_mark(int it, int i) {
    if (threadIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_iter_trace[2 * it + i] = t;
    }
}
__device__ __forceinline__ void cta_mark(int i) {
    if (threadIdx.x == 0 && blockIdx.x < 2048) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_cta_trace[2 * blockIdx.x + i] = t;
    }
}
__device__ __forceinline__ void tail_mark(int i) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_tail_trace[i] = t;
    }
}
#else
__device__ __forceinline__ void tail_mark(int) {}
__device__ __forceinline__ void cta_mark(int) {}
__device__ __forceinline__ void iter_mark(int, int) {}
#endif

// One CTA-wide arrival ticket; true in every thread of the last CTA to arrive.
__device__ __forceinline__ bool last_arrival(unsigned* ctr, unsigned total, int* s_flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *s_flag = atomicAdd(ctr, 1u) == total - 1u;
    __syncthreads();
    const bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by every thread of every CTA once its partial row is written.
// `work` is >= (3 k d + k + 40) doubles of shared memory no longer in use.
__device__ void fused_tail(const FuseArgs& f, const double* part, int S, int KD, double* work) {
    const int G = gridDim.x;
    int* s_flag = reinterpret_cast<int*>(work);
    unsigned long long* s_epoch = reinterpret_cast<unsigned long long*>(work + 1);
    double* sh = work + 8;
    double* upd = work + 40;
    if (blockIdx.x == 0) tail_mark(0);
    cta_mark(1);
    // sums: f64 partial -> int64 at 2^-(61 - e) with n max|x| < 2^e: exact to
    // ~1e-18 of the largest possible sum, so the total matches an f64
    // accumulation to its own rounding level
    int e2 = 0;
    frexp(static_cast<double>(f.n) * *f.xabs + 1.0, &e2);
    const int shift = 61 - e2;
    // what the update will read, fetched now so only the last CTA's final
    // loads stay on the critical path
    const int k = S - KD;
    double* pre = work + 1536;  // running[S] | c64[KD] | cn64[k] | sx2[4] | stats[S]
    for (int e = threadIdx.x; e < S; e += blockDim.x) {
        if (f.upd.running) pre[e] = f.upd.running[e];
        if (e < KD) pre[S + e] = f.upd.c64[e];
        if (e < k) pre[S + KD + e] = f.upd.cn64[e];
        if (e < 4) pre[S + KD + k + e] = f.upd.sx2[e];
    }
    double* stats_s = pre + S + KD + k + 4;
    __syncthreads();  // `part` complete
    for (int e = threadIdx.x; e < S; e += blockDim.x) {
        const double v = part[e];
        const long long q = e < KD ? llrint(ldexp(v, shift)) : llrint(v);
        if (q != 0) atomicAdd(f.acc64 + e, static_cast<unsigned long long>(q));
    }
    if (!last_arrival(f.counters, G, s_flag)) return;
    tail_mark(1);
    if (threadIdx.x == 0) {
        f.counters[0] = 0u;  // every ticket is in
        if (f.tile_ctr) *f.tile_ctr = 0u;
    }
    const int world = f.upd.world;
    unsigned long long epoch = 0;
    int slot = 0;
    if (world > 1) {
        if (threadIdx.x == 0) {
            unsigned long long* ep = xchg_flags(f.peers[f.rank], world) + world;
            *s_epoch = *ep + 1;
            *ep = *s_epoch;
        }
        __syncthreads();
        epoch = *s_epoch;
        slot = static_cast<int>(epoch & 1);
    }
    for (int e = threadIdx.x; e < S; e += blockDim.x) {
        const long long q = static_cast<long long>(atomicExch(f.acc64 + e, 0ull));  // read + reset
        const double v = e < KD ? ldexp(static_cast<double>(q), -shift) : static_cast<double>(q);
        f.stats[e] = v;
        stats_s[e] = v;
        for (int r = 0; r < world && world > 1; ++r) xchg_recv(f.peers[r], slot, world, f.rank)[e] = v;  // NVLink
    }
    tail_mark(2);
    UpdArgs a = f.upd;
    a.gathered = stats_s;
    a.gstride = S;
    a.rd_running = pre;
    a.rd_c64 = pre + S;
    a.rd_cn64 = pre + S + KD;
    a.rd_sx2 = pre + S + KD + k;
    __syncthreads();  // stats_s complete
    if (world > 1) {
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x < world) {
            st_release_sys(xchg_flags(f.peers[threadIdx.x], world) + f.rank, epoch);
            const unsigned long long* mine = xchg_flags(f.peers[f.rank], world) + threadIdx.x;
            const long long t0 = clock64();
            while (ld_acquire_sys(mine) < epoch) {
                __nanosleep(64);
                if (clock64() - t0 > 40000000000ll) {  // a peer never arrived (~20 s): TimeoutError, no trap
                    atomicExch(f.upd.flags + 3, 1);
                    atomicExch(f.upd.flags, 1);  // every later launch of the fit returns at once
                    break;
                }
            }
        }
        __syncthreads();
        __threadfence();
        a.gathered = xchg_recv(f.peers[f.rank], slot, world, 0);
        a.gstride = XCHG_STATS;
    }
    tail_mark(3);
    update_body(a, upd, sh);
    tail_mark(4);
    iter_mark(f.upd.iter, 1);
}

// fp32 top-2 of R rows held in registers as feature pairs: one FFMA2 per two
// features with the centroid pair broadcast from the constant bank (uniform
// registers), JG clusters x R rows of independent chains at a time.
template <int D, int K, int R>
__device__ __forceinline__ void small_top2(const float2 (&xv)[R][D / 2], const float* CT, float (&b1)[R],
                                           float (&b2)[R], int (&i1)[R]) {
    constexpr int L = D / 2, KD = K * D;
    constexpr int JG = K % 4 == 0 ? 4 : 1;
#pragma unroll
    for (int h = 0; h < R; ++h) {
        b1[h] = FLT_MAX;
        b2[h] = FLT_MAX;
        i1[h] = 0;
    }
#pragma unroll
    for (int j0 = 0; j0 < K; j0 += JG) {
        float2 sp[JG][R];
#pragma unroll
        for (int u = 0; u < JG; ++u)
#pragma unroll
            for (int h = 0; h < R; ++h) sp[u][h] = make_float2(CT[KD + j0 + u], 0.f);
#pragma unroll
        for (int f = 0; f < L; ++f) {
#pragma unroll
            for (int u = 0; u < JG; ++u) {
                const float2 c = make_float2(CT[(j0 + u) * D + 2 * f], CT[(j0 + u) * D + 2 * f + 1]);
#pragma unroll
                for (int h = 0; h < R; ++h) sp[u][h] = ffma2(xv[h][f], c, sp[u][h]);
            }
        }
#pragma unroll
        for (int u = 0; u < JG; ++u)
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const float sc = sp[u][h].x + sp[u][h].y;
                const bool lt = sc < b1[h];
                b2[h] = fminf(b2[h], fmaxf(b1[h], sc));
                b1[h] = fminf(b1[h], sc);
                i1[h] = lt ? j0 + u : i1[h];
            }
    }
}

template <int D, int K, int SLOT, bool DONLY = false>
__global__ void __launch_bounds__(KS_THREADS, DONLY ? KS_DONLY_CTAS : KS_MIN_CTAS) kmeans_small_kernel(SmallParams p) {
    static_assert(D % 2 == 0 && D <= 64 && K <= 32, "small kernel shape");
    constexpr int TILE = KS_TILE, S = KS_STAGES, W = KS_WARPS, R = KS_R, VW = KS_VW;
    constexpr int L = D / 2;                  // lanes per row in phase 2 (float2 each)
    constexpr int G = L <= 32 ? 32 / L : 1;   // rows summed in parallel per warp
    constexpr int KD = K * D;
    constexpr int JW = (K + W - 1) / W;       // clusters owned per warp
    if (p.done && *p.done) return;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* tiles = reinterpret_cast<float*>(smem_raw);                 // S x TILE x D
    int8_t* labs = reinterpret_cast<int8_t*>(tiles + S * TILE * D);    // S x TILE previous labels (delta)
    double* wacc = reinterpret_cast<double*>(labs + S * TILE);         // W x K x D sums of changes (delta)
    float* scr = reinterpret_cast<float*>(wacc + W * KD);              // W x KS_SCR x D changed rows (delta)
    int* scl = reinterpret_cast<int*>(scr + W * KS_SCR * D);           // W x KS_SCR x 2 their new/old labels
    int* cnt = reinterpret_cast<int*>(scl + W * 2 * KS_SCR);           // VW x K
    unsigned* consumed = reinterpret_cast<unsigned*>(cnt + VW * K);    // S (delta mode)
    int* stage_tile = reinterpret_cast<int*>(consumed + S);             // S (dynamic schedule)
    uint64_t* bars = reinterpret_cast<uint64_t*>(cnt + ((VW * K + 2 * S + 1) & ~1));

    const float* CT = c_km_table + SLOT * KS_TABLE;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float tau = 4.f * static_cast<float>(D + 3) * 0x1.0p-24f *
                      (p.bounds[1] + 2.f * sqrtf(static_cast<float>(D)) * static_cast<float>(*p.xabs) * p.bounds[0]);
#ifdef KS_EXP_NOREFINE
    const float tau_used = 0.f;  // timing experiment only
#else
    const float tau_used = tau;
#endif
#ifdef KS_EXP_NOPHASE2
    const bool accumulate = false;  // timing experiment only
#else
    const bool accumulate = DONLY || p.partials != nullptr;
#endif
    const bool delta = DONLY || (accumulate && p.prev != nullptr);
    if (p.fu.on && blockIdx.x == 0) {
        tail_mark(5);
        iter_mark(p.fu.upd.iter, 0);
    }
    if (p.fu.on) cta_mark(0);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (delta)
        for (int e = tid; e < W * KD; e += KS_THREADS) wacc[e] = 0.0;
    if (tid < S) consumed[tid] = 0u;
    __syncthreads();

    const int64_t ntiles = ceil_div(p.n, TILE);
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue = [&](int64_t it) {
        const int64_t tile = blockIdx.x + it * gridDim.x;
        const int64_t rows = min(static_cast<int64_t>(TILE), p.n - tile * TILE);
        if (delta)
            bulk_load2(tiles + (it % S) * TILE * D, p.x + tile * TILE * D, static_cast<uint32_t>(rows * D * 4),
                       labs + (it % S) * TILE, p.prev + tile * TILE, static_cast<uint32_t>(rows), &bars[it % S]);
        else
            bulk_load(tiles + (it % S) * TILE * D, p.x + tile * TILE * D, static_cast<uint32_t>(rows * D * 4),
                      &bars[it % S]);
    };
    // delta mode with a tile counter: tiles handed out dynamically (a CTA that
    // runs ahead takes more), so every CTA finishes within about one tile
    const bool dyn = accumulate && p.tile_ctr != nullptr;
    auto grab = [&](int s) {
        const unsigned t = atomicAdd(p.tile_ctr, 1u);
        if (t < ntiles) {
            const int64_t rows = min(static_cast<int64_t>(TILE), p.n - static_cast<int64_t>(t) * TILE);
            stage_tile[s] = static_cast<int>(t);
            if (delta)
                bulk_load2(tiles + s * TILE * D, p.x + static_cast<int64_t>(t) * TILE * D,
                           static_cast<uint32_t>(rows * D * 4), labs + s * TILE,
                           p.prev + static_cast<int64_t>(t) * TILE, static_cast<uint32_t>(rows), &bars[s]);
            else
                bulk_load(tiles + s * TILE * D, p.x + static_cast<int64_t>(t) * TILE * D,
                          static_cast<uint32_t>(rows * D * 4), &bars[s]);
        } else {
            stage_tile[s] = -1;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
        }
    };
    // full mode refills stage (it-1)%S mid-tile (S-1 tiles ahead); delta mode
    // refills a stage as soon as every warp has its rows in registers (S ahead)
    const int ahead = delta ? S : S - 1;
    if (tid == 0) {
        if (dyn)
            for (int s = 0; s < ahead; ++s) grab(s);
        else
            for (int s = 0; s < ahead && s < my_tiles; ++s) issue(s);
    }

    long long count_acc = 0;  // lane j < K of warp 0: rows of cluster j
    unsigned long long refined = 0;
    const int g = lane / L, q = lane % L;
    double2 wsum[JW];
#pragma unroll
    for (int jj = 0; jj < JW; ++jj) wsum[jj] = make_double2(0.0, 0.0);

    int cnt_delta = 0;  // delta mode, lane j < K: net rows gained by cluster j
    for (int64_t it = 0; dyn || it < my_tiles; ++it) {
        const float* xt = tiles + (it % S) * TILE * D;
        mbar_wait(&bars[it % S], static_cast<uint32_t>((it / S) & 1));
        const int64_t tile_id = dyn ? static_cast<int64_t>(stage_tile[it % S]) : blockIdx.x + it * gridDim.x;
        if (tile_id < 0) break;
        const int64_t row0 = tile_id * TILE;
        if (delta) {
            // ---------------- delta mode: rows to registers, then the stage is
            // handed back at once (the last warp to finish reading refills it),
            // so two tiles per CTA stay in flight while this one is scored
            float2 xv[R][L];
            int prevl[R], label[R];
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const int row = tid + h * KS_THREADS;
#pragma unroll
                for (int f = 0; f < L; ++f) xv[h][f] = *reinterpret_cast<const float2*>(xt + row * D + 2 * f);
                prevl[h] = row0 + row < p.n ? static_cast<int>(labs[(it % S) * TILE + row]) : -1;
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) {
                const unsigned done = atomicAdd(&consumed[it % S], 1u);
                if (done == W - 1) {
                    consumed[it % S] = 0u;
                    if (dyn)
                        grab(static_cast<int>(it % S));
                    else if (it + S < my_tiles)
                        issue(it + S);
                }
            }
            {
                float b1[R], b2[R];
                int i1[R];
#ifdef KS_EXP_NOSCORE
#pragma unroll
                for (int h = 0; h < R; ++h) {  // timing experiment only: stream, no scores
                    float a = 0.f;
#pragma unroll
                    for (int f = 0; f < L; ++f) a += xv[h][f].x + xv[h][f].y;
                    b1[h] = a;
                    b2[h] = a + 1e30f;
                    i1[h] = prevl[h] < 0 ? 0 : prevl[h];
                }
#else
                small_top2<D, K, R>(xv, CT, b1, b2, i1);
#endif
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const int64_t gr = row0 + tid + h * KS_THREADS;
                    label[h] = K;
                    if (gr < p.n) {
                        label[h] = i1[h];
                        if (K > 1 && !(b2[h] - b1[h] > tau_used)) {
                            // the stage may be refilled already: the row from global (L2)
                            label[h] = ref_argmin<float>(p.x + gr * D, D, p.c64, p.cn64, K);
                            ++refined;
                        }
                        if (p.lab8) p.lab8[gr] = static_cast<int8_t>(label[h]);
                    }
                }
            }
            // changed rows: compacted into the warp's scratch, then moved from
            // the old cluster's sums to the new one's, lane = feature, in row
            // order (deterministic)
            float* wscr = scr + warp * KS_SCR * D;
            int* wscl = scl + warp * 2 * KS_SCR;
            double* acc = wacc + warp * KD;
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const bool ch = label[h] < K && label[h] != prevl[h];
                unsigned mask = __ballot_sync(FULL, ch);
                while (mask) {
                    // a batch of at most KS_SCR changed rows (the lowest set bits)
                    unsigned batch = mask;
                    if (__popc(batch) > KS_SCR) {
                        batch = 0u;
                        unsigned rest = mask;
#pragma unroll
                        for (int i = 0; i < KS_SCR; ++i) {
                            batch |= rest & (0u - rest);
                            rest &= rest - 1u;
                        }
                    }
                    mask &= ~batch;
                    if ((batch >> lane) & 1u) {
                        const int pos = __popc(batch & ((1u << lane) - 1u));
#pragma unroll
                        for (int f = 0; f < L; ++f) *reinterpret_cast<float2*>(wscr + pos * D + 2 * f) = xv[h][f];
                        wscl[2 * pos] = label[h];
                        wscl[2 * pos + 1] = prevl[h];
                    }
                    __syncwarp();
                    const int nch = __popc(batch);
                    for (int c = 0; c < nch; ++c) {
                        const int nl = wscl[2 * c], ol = wscl[2 * c + 1];
                        if (lane < K) cnt_delta += (lane == nl) - (lane == ol);
#pragma unroll
                        for (int f = lane; f < D; f += 32) {
                            const double v = static_cast<double>(wscr[c * D + f]);
                            acc[nl * D + f] += v;
                            if (ol >= 0) acc[ol * D + f] -= v;
                        }
                    }
                    __syncwarp();
                }
            }
            continue;
        }

        // ---------------- phase 1: rows tid + h * 128 (h < R), lane = row
        // scores in feature pairs: one FFMA2 per two features, the centroid
        // pair broadcast from uniform registers (constant bank)
        float2 xv[R][L];
        int label[R];
#pragma unroll
        for (int h = 0; h < R; ++h) {
            const int row = tid + h * KS_THREADS;
#pragma unroll
            for (int f = 0; f < L; ++f) xv[h][f] = *reinterpret_cast<const float2*>(xt + row * D + 2 * f);
        }
        {
            float b1[R], b2[R];
            int i1[R];
            small_top2<D, K, R>(xv, CT, b1, b2, i1);
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const int row = tid + h * KS_THREADS;
                label[h] = K;  // rows past the end sort last
                if (row0 + row < p.n) {
                    label[h] = i1[h];
                    if (K > 1 && !(b2[h] - b1[h] > tau_used)) {
                        label[h] = ref_argmin<float>(xt + row * D, D, p.c64, p.cn64, K);
                        ++refined;
                    }
                    if (p.labels) p.labels[row0 + row] = label[h];
                    if (p.lab8) p.lab8[row0 + row] = static_cast<int8_t>(label[h]);
                }
            }
        }
        if (!accumulate) {
            __syncthreads();  // every warp is done with the previous tile's stage
            if (tid == 0 && it + S - 1 < my_tiles) issue(it + S - 1);
            continue;
        }

        // ---------------- phase 2a: counts per 32-row group vw = h * W + warp
        unsigned mine[R];
        int rank[R];
        if (lane < K) {
#pragma unroll
            for (int h = 0; h < R; ++h) cnt[(h * W + warp) * K + lane] = 0;
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < R; ++h) {
            mine[h] = __match_any_sync(FULL, label[h]);
            rank[h] = __popc(mine[h] & ((1u << lane) - 1u));
            if (rank[h] == 0 && label[h] < K) cnt[(h * W + warp) * K + label[h]] = __popc(mine[h]);
        }
        __syncthreads();  // counts visible; every warp is done with the previous tile
        if (tid == 0) {
            if (dyn)
                grab(static_cast<int>((it + S - 1) % S));
            else if (it + S - 1 < my_tiles)
                issue(it + S - 1);
        }

        // lane j: start of cluster j in the sorted tile and the offsets of this
        // warp's groups inside it
        int total = 0, before[R];
#pragma unroll
        for (int h = 0; h < R; ++h) before[h] = 0;
        if (lane < K) {
#pragma unroll
            for (int v = 0; v < VW; ++v) {
                const int c = cnt[v * K + lane];
                total += c;
#pragma unroll
                for (int h = 0; h < R; ++h) before[h] += v < h * W + warp ? c : 0;
            }
        }
        int start = total;  // inclusive scan over lanes 0..K-1
#pragma unroll
        for (int o = 1; o < K; o <<= 1) {
            const int v = __shfl_up_sync(FULL, start, o);
            if (lane >= o) start += v;
        }
        start -= total;
        if (warp == 0 && lane < K) count_acc += total;

        // ---------------- phase 2b: scatter rows into label order, in place:
        // every row of this stage is in registers (barrier above)
        float* sorted = const_cast<float*>(xt);
#pragma unroll
        for (int h = 0; h < R; ++h) {
            const int pos = __shfl_sync(FULL, start + before[h], label[h] < K ? label[h] : 0) + rank[h];
            if (label[h] < K) {
#pragma unroll
                for (int f = 0; f < L; ++f) *reinterpret_cast<float2*>(sorted + pos * D + 2 * f) = xv[h][f];
            }
        }
        __syncthreads();

        // ---------------- phase 2c: warp w sums the sorted runs of clusters w, w+W, ...
#pragma unroll
        for (int jj = 0; jj < JW; ++jj) {
            const int j = warp + jj * W;
            if (j >= K) break;
            const int r0 = __shfl_sync(FULL, start, j);
            const int r1 = r0 + __shfl_sync(FULL, total, j);
            // f64 accumulation straight from the fp32 rows: the run sums carry
            // no fp32 rounding, so the centroids track the reference's to ~1e-16
            // and near-tie flips of its trajectory stay ~1e6x rarer
            double2 part = make_double2(0.0, 0.0), part2 = make_double2(0.0, 0.0);
            if (g < G) {
                const float* src = sorted + 2 * q;
                int r = r0 + g;
#pragma unroll 2
                for (; r + G < r1; r += 2 * G) {  // two independent f64 chains
                    const float2 v = *reinterpret_cast<const float2*>(src + r * D);
                    const float2 u = *reinterpret_cast<const float2*>(src + (r + G) * D);
                    part.x += static_cast<double>(v.x);
                    part.y += static_cast<double>(v.y);
                    part2.x += static_cast<double>(u.x);
                    part2.y += static_cast<double>(u.y);
                }
                if (r < r1) {
                    const float2 v = *reinterpret_cast<const float2*>(src + r * D);
                    part.x += static_cast<double>(v.x);
                    part.y += static_cast<double>(v.y);
                }
                part.x += part2.x;
                part.y += part2.y;
            }
            // tree over the G groups; a source beyond the last group contributes nothing
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                const double vx = __shfl_down_sync(FULL, part.x, o * L);
                const double vy = __shfl_down_sync(FULL, part.y, o * L);
                if (g + o < G) {
                    part.x += vx;
                    part.y += vy;
                }
            }
            // lanes of group 0 own features 2q, 2q+1 of cluster j (f64, registers)
            wsum[jj].x += part.x;
            wsum[jj].y += part.y;
        }
    }
    if (refined) atomicAdd(p.refined, refined);
    if (!accumulate) return;
    const int Sst = KD + K;
    // fused: the CTA's partial row stays in shared memory (past the tail's
    // scratch); otherwise it goes to the partials array for the reduce kernel
    double* out = p.fu.on ? reinterpret_cast<double*>(tiles) + 1024 : p.partials + static_cast<int64_t>(blockIdx.x) * Sst;
    if (p.fu.on) __syncthreads();  // the last tile's rows in `tiles` are consumed
    if (delta) {
        if (lane < K) cnt[warp * K + lane] = cnt_delta;
        __syncthreads();
        for (int e = tid; e < KD; e += KS_THREADS) {
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < W; ++c) v += wacc[c * KD + e];
            out[e] = v;
        }
        if (tid < K) {
            int c = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) c += cnt[w * K + tid];
            out[KD + tid] = static_cast<double>(c);
        }
    } else {
#pragma unroll
        for (int jj = 0; jj < JW; ++jj) {
            const int j = warp + jj * W;
            if (j < K && g == 0 && q < L) *reinterpret_cast<double2*>(out + j * D + 2 * q) = wsum[jj];
        }
        if (warp == 0 && lane < K) out[KD + lane] = static_cast<double>(count_acc);
    }
    if (p.fu.on) fused_tail(p.fu, out, Sst, KD, reinterpret_cast<double*>(tiles));
}

template <int D, int K>
static size_t small_smem() {
    return static_cast<size_t>(KS_STAGES) * KS_TILE * (D * 4 + 1) + static_cast<size_t>(KS_WARPS) * K * D * 8 +
           static_cast<size_t>(KS_WARPS) * KS_SCR * (D * 4 + 8) +
           static_cast<size_t>((KS_VW * K + 2 * KS_STAGES + 1) & ~1) * 4 + KS_STAGES * 8;
}

#include "kmeans_tc.cuh"

// Per-stat sum over the CTA partials: one warp per stat, lanes stride over the
// CTAs, then a fixed xor-butterfly (deterministic for a given grid).
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* __restrict__ partials, int G, int S,
                                                              double* __restrict__ stats, const int* done) {
    if (done && *done) return;
    const int e = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (e >= S) return;
    double v = 0.0;
    for (int g = lane; g < G; g += 32) v += partials[static_cast<int64_t>(g) * S + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) stats[e] = v;
}

// Deterministic block reductions: a fixed xor-butterfly inside each warp, then
// warp 0 combines the per-warp values in a fixed order.  `sh` holds >= 32 doubles.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int nw = (blockDim.x + 31) / 32;
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < nw; ++w) r += sh[w];
    __syncthreads();
    return r;
}
__device__ double block_max(double v, double* sh) {
    v = warp_max(v);
    const int nw = (blockDim.x + 31) / 32;
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
    __syncthreads();
    double r = sh[0];
    for (int w = 1; w < nw; ++w) r = fmax(r, sh[w]);
    __syncthreads();
    return r;
}

// Derived tables of cluster j from its f64 centroid row `c` (smem or global):
// reference-order |c|^2 (pairwise.cpp:13-18), the fp32 score tables, bounds.
__device__ void derive_cluster(int j, int k, int d, int dpad, const double* c, double* cn64, float* ct,
                               float* cn32, float* ctab, double& cnorm, double& cn32v) {
    double n64 = 0.0, n32 = 0.0;
    for (int f = 0; f < d; ++f) {
        const double cf = c[f];
        n64 = add_rn(n64, mul_rn(cf, cf));
        const float c32 = static_cast<float>(cf);
        ct[static_cast<int64_t>(j) * dpad + f] = -2.f * c32;
        if (ctab) ctab[static_cast<int64_t>(j) * d + f] = -2.f * c32;
        n32 += static_cast<double>(c32) * static_cast<double>(c32);
    }
    for (int f = d; f < dpad; ++f) ct[static_cast<int64_t>(j) * dpad + f] = 0.f;
    if (ctab) ctab[static_cast<int64_t>(k) * d + j] = static_cast<float>(n32);
    cn64[j] = n64;
    cn32[j] = static_cast<float>(n32);
    cnorm = sqrt(n32);
    cn32v = static_cast<double>(static_cast<float>(n32));
}

__global__ void derive_tables_kernel(int k, int d, int dpad, const double* c64, double* cn64,
                                     float* ct, float* cn32, float* ctab, float* bounds) {
    __shared__ double sh[256];
    double cmax = 0.0, cnmax = 0.0;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        double cnorm, cnv;
        derive_cluster(j, k, d, dpad, c64 + static_cast<int64_t>(j) * d, cn64, ct, cn32, ctab, cnorm, cnv);
        cmax = fmax(cmax, cnorm);
        cnmax = fmax(cnmax, cnv);
    }
    cmax = block_max(cmax, sh);
    cnmax = block_max(cnmax, sh);
    if (threadIdx.x == 0) {
        bounds[0] = static_cast<float>(cmax) * (1.f + 0x1.0p-20f);
        bounds[1] = static_cast<float>(cnmax) * (1.f + 0x1.0p-20f);
    }
}

// One CTA: rank-order fold, centroid update, inertia, displacement, tables.
// Stage 1 (thread per stat): fold the ranks in order 0..p-1 from the zero
// identity (allreduce(plus_vec), cluster.cpp:123) and form the new centroid
// (cluster.cpp:125-133) into shared memory.  Stage 2 (thread per cluster):
// the reference's sequential per-cluster loops (displacement, norms).
constexpr int UPD_MAX_KD = 8192;

// The update step, executed by one CTA (any blockDim): `upd` is shared memory
// of (3 k d + k) doubles (k d <= UPD_MAX_KD), `sh` 32 doubles.
__device__ void update_body(const UpdArgs& a, double* upd, double* sh) {
    const int k = a.k, d = a.d, dpad = a.dpad, world = a.world, accum = a.accum, iter = a.iter;
    const double* gathered = a.gathered;
    double *running = a.running, *c64 = a.c64, *cn64 = a.cn64, *trace = a.trace, *disp = a.disp;
    float *ct = a.ct, *cn32 = a.cn32, *ctab = a.ctab, *bounds = a.bounds;
    const double* sx2 = a.sx2;
    int* flags = a.flags;
    const double tol = a.tol;
    const int S = k * d + k, KD = k * d;
    const bool staged = KD <= UPD_MAX_KD;
    if (staged) {
        // allreduce(plus_vec) from the zero identity in rank order (cluster.cpp:123).
        // Eight elements per thread per pass, all loads before any store
        // (running may alias rd_running: one at a time, every load waited
        // behind the previous store -- 16 serial L2 round trips per thread)
        constexpr int UB = 8;
        for (int e0 = threadIdx.x; e0 < S; e0 += UB * blockDim.x) {
            double gv[UB], rv[UB], cv[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int e = e0 + u * blockDim.x;
                gv[u] = rv[u] = cv[u] = 0.0;
                if (e < S) {
                    for (int r = 0; r < world; ++r) gv[u] += gathered[static_cast<int64_t>(r) * a.gstride + e];
                    if (running && accum) rv[u] = a.rd_running[e];
                    if (e < KD) cv[u] = a.rd_c64[e];
                }
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int e = e0 + u * blockDim.x;
                if (e >= S) break;
                double v = gv[u];
                // delta iterations: the stats are changes since the last
                // iteration, added to the running per-cluster sums and counts
                if (running) {
                    if (accum) v += rv[u];
                    running[e] = v;
                }
                upd[e < KD ? e : KD + e] = v;
                if (e < KD) upd[KD + e] = cv[u];
            }
        }
        __syncthreads();
        tail_mark(6);
        // element-parallel: new centroid (cluster.cpp:125-133, empty keeps the
        // old one) and its fp32 tables; the order-dependent sums follow per cluster
        double* nxt_s = upd + 2 * KD + k;
        for (int e = threadIdx.x; e < KD; e += blockDim.x) {
            const int j = e / d, f = e % d;
            const double count = upd[2 * KD + j], s = upd[e], old = upd[KD + e];
            const double nxt = count > 0.0 ? s / count : old;
            nxt_s[e] = nxt;
            c64[e] = nxt;
            const float c32 = static_cast<float>(nxt);
            ct[static_cast<int64_t>(j) * dpad + f] = -2.f * c32;
            if (ctab) ctab[e] = -2.f * c32;
        }
        for (int e = threadIdx.x; e < k * (dpad - d); e += blockDim.x)
            ct[static_cast<int64_t>(e / (dpad - d)) * dpad + d + e % (dpad - d)] = 0.f;
        __syncthreads();
        tail_mark(7);
    }
    double inertia_part = 0.0, dmax = 0.0, cmax = 0.0, cnmax = 0.0;
    for (int j = threadIdx.x; j < k && staged; j += blockDim.x) {
        const double count = upd[2 * KD + j], cn_old = a.rd_cn64[j];
        const double* nxt_s = upd + 2 * KD + k;
        double dot = 0.0, dsq = 0.0, n64 = 0.0, n32 = 0.0;
        for (int f = 0; f < d; ++f) {
            const int e = j * d + f;
            const double s = upd[e], old = upd[KD + e], nxt = nxt_s[e];
            dot += old * s;
            const double diff = nxt - old;
            dsq = add_rn(dsq, mul_rn(diff, diff));  // cluster.cpp:142-146 order
            n64 = add_rn(n64, mul_rn(nxt, nxt));    // row_norms order
            const float c32 = static_cast<float>(nxt);
            n32 += static_cast<double>(c32) * static_cast<double>(c32);
        }
        if (ctab) ctab[KD + j] = static_cast<float>(n32);
        cn64[j] = n64;
        cn32[j] = static_cast<float>(n32);
        inertia_part += count * cn_old - 2.0 * dot;  // uses the old |c_j|^2
        dmax = fmax(dmax, __dsqrt_rn(dsq));
        cmax = fmax(cmax, sqrt(n32));
        cnmax = fmax(cnmax, static_cast<double>(static_cast<float>(n32)));
    }
    // large k*d: the same, straight from global memory (no running sums)
    for (int j = threadIdx.x; j < k && !staged; j += blockDim.x) {
        double count = 0.0, dot = 0.0, dsq = 0.0, n64 = 0.0, n32 = 0.0;
        for (int r = 0; r < world; ++r) count += gathered[static_cast<int64_t>(r) * a.gstride + KD + j];
        const double cn_old = cn64[j];
        for (int f = 0; f < d; ++f) {
            const int e = j * d + f;
            double s = 0.0;
            for (int r = 0; r < world; ++r) s += gathered[static_cast<int64_t>(r) * a.gstride + e];
            const double old = c64[e];
            dot += old * s;
            const double nxt = count > 0.0 ? s / count : old;  // cluster.cpp:125-133
            const double diff = nxt - old;
            dsq = add_rn(dsq, mul_rn(diff, diff));              // cluster.cpp:142-146 order
            c64[e] = nxt;
            n64 = add_rn(n64, mul_rn(nxt, nxt));                // row_norms order
            const float c32 = static_cast<float>(nxt);
            ct[static_cast<int64_t>(j) * dpad + f] = -2.f * c32;
            if (ctab) ctab[e] = -2.f * c32;
            n32 += static_cast<double>(c32) * static_cast<double>(c32);
        }
        for (int f = d; f < dpad; ++f) ct[static_cast<int64_t>(j) * dpad + f] = 0.f;
        if (ctab) ctab[KD + j] = static_cast<float>(n32);
        cn64[j] = n64;
        cn32[j] = static_cast<float>(n32);
        inertia_part += count * cn_old - 2.0 * dot;  // uses the old |c_j|^2
        dmax = fmax(dmax, __dsqrt_rn(dsq));
        cmax = fmax(cmax, sqrt(n32));
        cnmax = fmax(cnmax, static_cast<double>(static_cast<float>(n32)));
    }
    tail_mark(8);
    // one combined block reduction (fixed order: xor-butterfly, then warps in order)
    const double sx2_total = threadIdx.x == 0 ? a.rd_sx2[2] : 0.0;
    inertia_part = warp_sum(inertia_part);
    dmax = warp_max(dmax);
    cmax = warp_max(cmax);
    cnmax = warp_max(cnmax);
    const int nw = (blockDim.x + 31) / 32;
    if ((threadIdx.x & 31) == 0) {
        const int w = threadIdx.x / 32;
        sh[4 * w] = inertia_part;
        sh[4 * w + 1] = dmax;
        sh[4 * w + 2] = cmax;
        sh[4 * w + 3] = cnmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double inertia = 0.0;
        for (int w = 0; w < nw; ++w) {
            inertia += sh[4 * w];
            dmax = fmax(dmax, sh[4 * w + 1]);
            cmax = fmax(cmax, sh[4 * w + 2]);
            cnmax = fmax(cnmax, sh[4 * w + 3]);
        }
        trace[iter] = sx2_total + inertia;
        disp[iter] = dmax;
        flags[1] = iter + 1;
        if (dmax < tol) flags[0] = 1;
        bounds[0] = static_cast<float>(cmax) * (1.f + 0x1.0p-20f);
        bounds[1] = static_cast<float>(cnmax) * (1.f + 0x1.0p-20f);
    }
}

#include "kmeans_persist.cuh"

__global__ void __launch_bounds__(256) kmeans_update_kernel(UpdArgs a) {
    if (a.flags[0]) return;
    __shared__ double sh[32];
    extern __shared__ double upd[];  // [KD] folded sums, [KD] old centroids, [k] folded counts, [KD] new
    update_body(a, upd, sh);
}

// The same update spread over CTAs (per-iteration launches, d <= UPD_MC_MAXD):
// CTA b takes clusters b, b + G, ...: the cluster's stats folded over the
// ranks in rank order, running sums, new centroid, fp32 tables (element-
// parallel), then the order-dependent chains (dot, |c_new - c_old|^2, |c|^2 in
// f64 and fp32) by one thread.  Per-cluster inertia / displacement / norm
// maxima go to `red`; the last CTA to finish reduces them exactly like
// update_body (thread t holds clusters t, t + 256, ...; xor-butterfly per warp,
// then the warps in order), so the results are bit-identical to it.  The
// single-CTA kernel took ~27 us per cfg3 iteration (a latency chain: 64-step
// loops over 64 clusters on two warps); this one a few.
constexpr int UPD_MC_MAXD = 1024;  // 3 d doubles of dynamic shared memory: 24 KB at most
__global__ void __launch_bounds__(256) kmeans_update_mc_kernel(UpdArgs a, double* red, unsigned* ticket) {
    if (a.flags[0]) return;
    const int k = a.k, d = a.d, dpad = a.dpad, world = a.world, KD = k * d;
    extern __shared__ double us[];  // [d] sums, [d] old, [d] new
    double* ss = us;
    double* so = us + d;
    double* sn = us + 2 * d;
    __shared__ double scount;
    __shared__ bool last;
    for (int j = blockIdx.x; j < k; j += gridDim.x) {
        // (1) fold, running sums, new centroid, tables: element-parallel
        for (int f = threadIdx.x; f <= d; f += blockDim.x) {
            const int e = f < d ? j * d + f : KD + j;
            double v = 0.0;
            for (int r = 0; r < world; ++r) v += a.gathered[static_cast<int64_t>(r) * a.gstride + e];
            if (a.running) {
                if (a.accum) v += a.rd_running[e];
                a.running[e] = v;
            }
            if (f < d) {
                ss[f] = v;
                so[f] = a.rd_c64[e];
            } else {
                scount = v;
            }
        }
        __syncthreads();
        const double count = scount;
        for (int f = threadIdx.x; f < dpad; f += blockDim.x) {
            if (f < d) {
                const double nxt = count > 0.0 ? ss[f] / count : so[f];  // cluster.cpp:125-133
                sn[f] = nxt;
                a.c64[j * d + f] = nxt;
                const float c32 = static_cast<float>(nxt);
                a.ct[static_cast<int64_t>(j) * dpad + f] = -2.f * c32;
                if (a.ctab) a.ctab[j * d + f] = -2.f * c32;
            } else {
                a.ct[static_cast<int64_t>(j) * dpad + f] = 0.f;
            }
        }
        __syncthreads();
        // (2) the order-dependent sums of update_body, same operations
        if (threadIdx.x == 0) {
            const double cn_old = a.rd_cn64[j];  // (rd_cn64 may alias cn64, written below)
            double dot = 0.0, dsq = 0.0, n64 = 0.0, n32 = 0.0;
            for (int f = 0; f < d; ++f) {
                const double sv = ss[f], old = so[f], nxt = sn[f];
                dot += old * sv;
                const double diff = nxt - old;
                dsq = add_rn(dsq, mul_rn(diff, diff));  // cluster.cpp:142-146 order
                n64 = add_rn(n64, mul_rn(nxt, nxt));    // row_norms order
                const float c32 = static_cast<float>(nxt);
                n32 += static_cast<double>(c32) * static_cast<double>(c32);
            }
            if (a.ctab) a.ctab[KD + j] = static_cast<float>(n32);
            a.cn64[j] = n64;
            a.cn32[j] = static_cast<float>(n32);
            red[j] = count * cn_old - 2.0 * dot;  // uses the old |c_j|^2
            red[k + j] = __dsqrt_rn(dsq);
            red[2 * k + j] = sqrt(n32);
            red[3 * k + j] = static_cast<double>(static_cast<float>(n32));
        }
        __syncthreads();
    }
    // (3) the last CTA: update_body's block reduction over the per-cluster values
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double inertia_part = 0.0, dmax = 0.0, cmax = 0.0, cnmax = 0.0;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        inertia_part += __ldcg(red + j);
        dmax = fmax(dmax, __ldcg(red + k + j));
        cmax = fmax(cmax, __ldcg(red + 2 * k + j));
        cnmax = fmax(cnmax, __ldcg(red + 3 * k + j));
    }
    __shared__ double sh[32];
    const double sx2_total = threadIdx.x == 0 ? a.rd_sx2[2] : 0.0;
    inertia_part = warp_sum(inertia_part);
    dmax = warp_max(dmax);
    cmax = warp_max(cmax);
    cnmax = warp_max(cnmax);
    const int nw = (blockDim.x + 31) / 32;
    if ((threadIdx.x & 31) == 0) {
        const int w = threadIdx.x / 32;
        sh[4 * w] = inertia_part;
        sh[4 * w + 1] = dmax;
        sh[4 * w + 2] = cmax;
        sh[4 * w + 3] = cnmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double inertia = 0.0;
        for (int w = 0; w < nw; ++w) {
            inertia += sh[4 * w];
            dmax = fmax(dmax, sh[4 * w + 1]);
            cmax = fmax(cmax, sh[4 * w + 2]);
            cnmax = fmax(cnmax, sh[4 * w + 3]);
        }
        a.trace[a.iter] = sx2_total + inertia;
        a.disp[a.iter] = dmax;
        a.flags[1] = a.iter + 1;
        if (dmax < a.tol) a.flags[0] = 1;
        a.bounds[0] = static_cast<float>(cmax) * (1.f + 0x1.0p-20f);
        a.bounds[1] = static_cast<float>(cnmax) * (1.f + 0x1.0p-20f);
        *ticket = 0u;  // the next launch starts from zero
    }
}

static size_t update_smem(int k, int d) {
    const size_t kd = static_cast<size_t>(k) * d;
    const size_t bytes = kd <= UPD_MAX_KD ? (3 * kd + k) * sizeof(double) : 0;
    static bool attr = false;
    if (!attr) {
        DNDC_CUDA(cudaFuncSetAttribute(kmeans_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>((3 * UPD_MAX_KD + 1024) * sizeof(double))));
        attr = true;
    }
    return bytes;
}

// Validation pass (cluster.cpp:88-89) fused with sum |x|^2 and max |x|.  fp32
// input streams as float4 (two independent f64 sums; x*x is exact in f64).
template <typename T>
__global__ void __launch_bounds__(256) validate_kernel(const T* __restrict__ x, int64_t count, double* out) {
    __shared__ double sh[256];
    double s = 0.0, s2 = 0.0, bad = 0.0;
    float mxf = 0.f;
    double mx = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t tail0 = 0;
    if constexpr (sizeof(T) == 4) {
        if (reinterpret_cast<uintptr_t>(x) % 16 == 0) {
            const float4* x4 = reinterpret_cast<const float4*>(x);
            const int64_t n4 = count / 4;
            for (int64_t i = t0; i < n4; i += stride) {
                const float4 v = __ldg(x4 + i);
                const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if ((__float_as_uint(a[u]) & 0x7f800000u) == 0x7f800000u) {
                        bad += 1.0;
                    } else {
                        const double d = static_cast<double>(a[u]);
                        if (u & 1) s2 = fma(d, d, s2); else s = fma(d, d, s);
                        mxf = fmaxf(mxf, fabsf(a[u]));
                    }
                }
            }
            tail0 = n4 * 4;
        }
    }
    for (int64_t e = tail0 + t0; e < count; e += stride) {
        const double v = static_cast<double>(x[e]);
        if (!isfinite(v)) {
            bad += 1.0;
        } else {
            s = fma(v, v, s);
            mx = fmax(mx, fabs(v));
        }
    }
    s = block_sum(s + s2, sh);
    bad = block_sum(bad, sh);
    mx = block_max(fmax(mx, static_cast<double>(mxf)), sh);
    if (threadIdx.x == 0) {
        out[3 * blockIdx.x] = s;
        out[3 * blockIdx.x + 1] = bad;
        out[3 * blockIdx.x + 2] = mx;
    }
}

__global__ void __launch_bounds__(256) validate_final_kernel(const double* pre, int G, double* sx2) {
    __shared__ double sh[32];
    double s = 0.0, bad = 0.0, mx = 0.0;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        s += pre[3 * g];
        bad += pre[3 * g + 1];
        mx = fmax(mx, pre[3 * g + 2]);
    }
    s = block_sum(s, sh);
    bad = block_sum(bad, sh);
    mx = block_max(mx, sh);
    if (threadIdx.x == 0) {
        sx2[0] = s;
        sx2[1] = bad;
        sx2[3] = mx;
    }
}

// gather_rows (cluster.cpp:27-42): rows owned by this rank into a zero-filled
// k x m f64 buffer (the allreduce-sum across ranks is then exact).
template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ x, int64_t lo, int64_t hi, int m,
                                   const int64_t* idx, int k, double* c64) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * m; e += gridDim.x * blockDim.x) {
        const int j = e / m, f = e % m;
        const int64_t g = idx[j];
        c64[e] = (g >= lo && g < hi) ? static_cast<double>(x[(g - lo) * m + f]) : 0.0;
    }
}

__global__ void zero_u32_kernel(unsigned* p, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0u;
}

__global__ void kmeans_reset_kernel(int* flags, unsigned long long* refined, unsigned* counters, int ncounters,
                                    unsigned long long* acc64, int S) {
    for (int i = 0; i < ncounters; ++i) counters[i] = 0u;
    for (int i = 0; i < S; ++i) acc64[i] = 0ull;
    flags[0] = flags[2];  // invalid input (validate_fold_kernel): every iteration is skipped
    flags[1] = 0;
    flags[3] = 0;  // peer timeout (fused exchange)
    *refined = 0ull;
}

// Zero state of one persistent fit (kmeans_persist.cuh): the three fixed-point
// accumulators, the arrival counter / release word, flags and the refined count.
__global__ void persist_reset_kernel(int* flags, unsigned long long* refined, unsigned long long* acc, int n_acc,
                                     unsigned* words, int n_words, unsigned* tile_ctr, int n_ctr) {
    for (int i = threadIdx.x; i < n_acc; i += blockDim.x) acc[i] = 0ull;
    for (int i = threadIdx.x; i < n_ctr; i += blockDim.x) tile_ctr[i] = 0u;
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) words[i] = 0u;
    if (threadIdx.x == 0) {
        flags[0] = flags[2];
        flags[1] = 0;
        flags[3] = 0;
        *refined = 0ull;
    }
}

// world x (sum |x|^2, non-finite count) -> sx2[2] = global sum; flags[2] =
// any non-finite value on any rank (cluster.cpp:88-89 raises ValueError)
__global__ void validate_fold_kernel(const double* all, int world, double* sx2, int* flags) {
    if (threadIdx.x != 0) return;
    double sum = 0.0, bad = 0.0;
    for (int r = 0; r < world; ++r) {
        sum += all[2 * r];
        bad += all[2 * r + 1];
    }
    sx2[2] = sum;
    flags[2] = bad > 0.0 ? 1 : 0;
}

// world x (sum |x|^2, non-finite count, the k init rows this rank owns, zeros
// elsewhere) -> sx2[2], flags[2] (as validate_fold_kernel) and the initial
// centroids: the rank-order sum of the rows (one owner each: exact) -- the
// validation allgather and the init allreduce as one collective
__global__ void validate_init_fold_kernel(const double* all, int world, int km, double* sx2, int* flags,
                                          double* c64) {
    const int per = 2 + km;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double sum = 0.0, bad = 0.0;
        for (int r = 0; r < world; ++r) {
            sum += all[static_cast<int64_t>(r) * per];
            bad += all[static_cast<int64_t>(r) * per + 1];
        }
        sx2[2] = sum;
        flags[2] = bad > 0.0 ? 1 : 0;
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < km; e += gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int r = 0; r < world; ++r) v += all[static_cast<int64_t>(r) * per + 2 + e];
        c64[e] = v;
    }
}

// ----------------------------------------------------------------- host
static KmBuffers buffers(dndc_ctx* ctx, int k, int m, int max_iter, int G) {
    KmBuffers b;
    const size_t S = static_cast<size_t>(k) * m + k;
    b.c64 = static_cast<double*>(ctx->slot("km_c64", sizeof(double) * k * m));
    b.cn64 = static_cast<double*>(ctx->slot("km_cn64", sizeof(double) * k));
    b.ct = static_cast<float*>(ctx->slot("km_ct", sizeof(float) * k * dpad_of(m)));
    b.cn32 = static_cast<float*>(ctx->slot("km_cn32", sizeof(float) * k));
    b.bounds = static_cast<float*>(ctx->slot("km_bounds", sizeof(float) * 4));
    b.stats = static_cast<double*>(ctx->slot("km_stats", sizeof(double) * S));
    b.gathered = static_cast<double*>(ctx->slot("km_gathered", sizeof(double) * S * ctx->world));
    b.partials = static_cast<double*>(ctx->slot("km_partials", sizeof(double) * S * std::max(G, 1)));
    b.trace = static_cast<double*>(ctx->slot("km_trace", sizeof(double) * std::max(max_iter, 1)));
    b.disp = static_cast<double*>(ctx->slot("km_disp", sizeof(double) * std::max(max_iter, 1)));
    b.flags = static_cast<int*>(ctx->slot("km_flags", sizeof(int) * 4));
    b.sx2 = static_cast<double*>(ctx->slot("km_sx2", sizeof(double) * 4));
    b.pre = static_cast<double*>(ctx->slot("km_pre", sizeof(double) * 3 * 4096));
    b.ctab = static_cast<float*>(ctx->slot("km_ctab", sizeof(float) * (k * m + k)));
    b.refined = static_cast<unsigned long long*>(ctx->slot("km_refined", sizeof(unsigned long long)));
    b.running = static_cast<double*>(ctx->slot("km_running", sizeof(double) * S));
    b.acc64 = static_cast<unsigned long long*>(ctx->slot("km_acc64", sizeof(unsigned long long) * S));
    b.counters = static_cast<unsigned*>(ctx->slot("km_counters", sizeof(unsigned) * 2));
    return b;
}

template <typename T>
struct AssignLaunch {
    void (*fn)(AssignParams);
    size_t smem;
    int grid;
    int stages;
};

template <typename T, int D>
static void pick(AssignLaunch<T>& L) {
    L.fn = kmeans_assign_kernel<T, D>;
}

template <typename T>
static size_t assign_smem(int k, int d, int stages) {
    return smem_layout(sizeof(T), k, d, srow_of(d), dpad_of(d), stages).total;
}

template <typename T>
static AssignLaunch<T> plan_assign(dndc_ctx* ctx, int k, int d, int64_t n) {
    AssignLaunch<T> L{};
    if constexpr (sizeof(T) == 4) {
        switch (d) {
            case 2: pick<T, 2>(L); break;
            case 3: pick<T, 3>(L); break;
            case 4: pick<T, 4>(L); break;
            case 8: pick<T, 8>(L); break;
            case 16: pick<T, 16>(L); break;
            case 18: pick<T, 18>(L); break;
            case 32: pick<T, 32>(L); break;
            case 64: pick<T, 64>(L); break;
            default: pick<T, 0>(L); break;
        }
    } else {
        pick<T, 0>(L);
    }
    int stages = 4;
    while (stages > 2 && assign_smem<T>(k, d, stages) > 200 * 1024) --stages;
    if (assign_smem<T>(k, d, stages) > 200 * 1024) stages = 0;  // unstaged: rows read from global
    L.stages = stages;
    L.smem = assign_smem<T>(k, d, stages);
    if (L.smem > 227 * 1024)
        throw Error(DNDC_EVALUE, "kmeans: k*m too large for the shared-memory accumulator (k=" +
                                     std::to_string(k) + ", m=" + std::to_string(d) + ")");
    DNDC_CUDA(cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(L.smem)));
    int per_sm = 1;
    DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.fn, KM_THREADS, L.smem));
    per_sm = std::max(per_sm, 1);
    const int64_t tiles = std::max<int64_t>(ceil_div(n, KM_TILE), 1);
    L.grid = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(ctx->num_sms) * per_sm));
    return L;
}

template <typename T>
static AssignParams assign_params(const KmBuffers& b, const T* x, int64_t n, int d, int k,
                                  int stages, bool accumulate, int32_t* labels, bool use_done) {
    AssignParams p{};
    p.x = x;
    p.n = n;
    p.d = d;
    p.k = k;
    p.dpad = dpad_of(d);
    p.srow = stages ? srow_of(d) : d;
    p.stages = stages;
    p.aligned16 = reinterpret_cast<uintptr_t>(x) % 16 == 0;
    p.ct = b.ct;
    p.cn32 = b.cn32;
    p.bounds = b.bounds;
    p.c64 = b.c64;
    p.cn64 = b.cn64;
    p.partials = accumulate ? b.partials : nullptr;
    p.labels = labels;
    p.refined = b.refined;
    p.done = use_done ? b.flags : nullptr;
    return p;
}

// Chooses the assign/accumulate kernel for a shape and launches it.
template <typename T>
struct Assigner {
    bool small = false;
    bool tc = false;
    bool tc_delta = false;  // the tc instantiation supports delta iterations (TcCfg::DELTA_OK)
    void (*tfn)(CUtensorMap, TcParams) = nullptr;
    void (*rfn)(TcRefineParams) = nullptr;  // near-tie refine after each tc launch
    void (*dtfn)(CUtensorMap, TcParams) = nullptr;  // four-warpgroup kernel: delta iterations and predict
    void (*afn)(TcAccumParams) = nullptr;  // full iterations with it: the sums from the final labels
    size_t asmem = 0;
    size_t dtsmem = 0;
    int dtthreads = 0;
    unsigned* rq_ctl = nullptr;
    uint64_t* rq_row = nullptr;
    unsigned long long* rq_cand = nullptr;
    float* rq_x = nullptr;
    long long* racc = nullptr;
    unsigned rq_cap = 0;
    int rgrid = 0, rthreads = 0;
    size_t rsmem = 0;
    CUtensorMap tmap{};
    size_t tsmem = 0;
    int tthreads = 0;
    AssignLaunch<T> gen{};
    void (*sfn)(SmallParams) = nullptr;
    void (*dfn)(SmallParams) = nullptr;  // delta-only instantiation (fewer registers, more CTAs)
    size_t ssmem = 0;
    int sgrid = 0, dgrid = 0, slot = 0;

    // partial rows a launch writes (tc: one per CTA + the refine kernel's)
    int grid() const { return tc ? sgrid + 1 : small ? sgrid : gen.grid; }
    // the grid of a launch (delta iterations run the delta-only kernel)
    int grid_for(bool delta) const { return (small && delta && dfn) ? dgrid : grid(); }
    int max_grid() const { return std::max(grid(), small ? dgrid : 0); }

    void launch(const KmBuffers& b, const T* x, int64_t n, int d, int k, bool accumulate, int32_t* labels,
                bool use_done, cudaStream_t st, const int8_t* prev = nullptr, int8_t* lab8 = nullptr,
                const FuseArgs* fu = nullptr, unsigned* tile_ctr = nullptr) const {
        if (tc) {
            TcParams tp{};
            tp.n = n;
            tp.c64 = b.c64;
            tp.cn64 = b.cn64;
            tp.ctab = b.ctab;
            tp.bounds = b.bounds;
            tp.partials = accumulate ? b.partials : nullptr;
            tp.labels = labels;
            tp.refined = b.refined;
            tp.done = use_done ? b.flags : nullptr;
            tp.prev = tc_delta ? prev : nullptr;
            tp.lab8 = tc_delta ? lab8 : nullptr;
            tp.xabs = b.sx2 + 3;
            tp.rq_ctl = rq_cap ? rq_ctl : nullptr;  // none: inline refine, the refine kernel finds no entries
            tp.rq_row = rq_row;
            tp.rq_cand = rq_cand;
            tp.rq_x = rq_x;
            tp.rq_cap = rq_cap;
            tp.x = reinterpret_cast<const float*>(x);
            // launches that accumulate no row themselves (delta, predict) take the
            // four-warpgroup kernel; full accumulation needs the sort of the old one
            const bool four = dtfn && (tp.prev != nullptr || !accumulate);
            // full iterations with the labels buffer: labels by the TMEM kernel,
            // then the sums of every row by kmeans_tc_accum_kernel
            const bool split_full = dtfn && afn && accumulate && tp.prev == nullptr && tp.lab8 != nullptr;
            if (split_full) {
                TcParams lp = tp;
                lp.partials = nullptr;
                dtfn<<<sgrid, dtthreads, dtsmem, st>>>(tmap, lp);
            } else if (four) {
                dtfn<<<sgrid, dtthreads, dtsmem, st>>>(tmap, tp);
            } else {
                tfn<<<sgrid, tthreads, tsmem, st>>>(tmap, tp);
            }
            TcRefineParams rp{};
            rp.n = n;
            rp.c64 = b.c64;
            rp.cn64 = b.cn64;
            rp.bounds = b.bounds;
            rp.xabs = b.sx2 + 3;
            rp.ctl = rq_ctl;
            rp.qrow = rq_row;
            rp.qcand = rq_cand;
            rp.qx = (four || split_full) ? nullptr : rq_x;  // the TMEM kernel queues no rows: read X
            rp.x = reinterpret_cast<const float*>(x);
            rp.cap = rq_cap;
            rp.labels = labels;
            rp.lab8 = tp.lab8;
            rp.racc = racc;
            rp.partial = accumulate && !split_full
                             ? b.partials + static_cast<int64_t>(sgrid) * (static_cast<int64_t>(k) * d + k)
                             : nullptr;
            rp.refined = b.refined;
            rp.done = tp.done;
            rfn<<<rgrid, rthreads, rsmem, st>>>(rp);
            if (split_full) {
                TcAccumParams ap{};
                ap.x = reinterpret_cast<const float*>(x);
                ap.n = n;
                ap.lab8 = tp.lab8;
                ap.xabs = b.sx2 + 3;
                ap.partials = b.partials;
                ap.done = tp.done;
                afn<<<sgrid, 512, asmem, st>>>(ap);
            }
        } else if (small) {
            DNDC_CUDA(cudaMemcpyToSymbolAsync(c_km_table, b.ctab, sizeof(float) * (k * d + k),
                                              sizeof(float) * KS_TABLE * slot, cudaMemcpyDeviceToDevice, st));
            SmallParams sp{};
            sp.x = reinterpret_cast<const float*>(x);
            sp.n = n;
            sp.c64 = b.c64;
            sp.cn64 = b.cn64;
            sp.bounds = b.bounds;
            sp.xabs = b.sx2 + 3;
            sp.partials = accumulate ? b.partials : nullptr;
            sp.labels = labels;
            sp.prev = prev;
            sp.lab8 = lab8;
            if (fu) sp.fu = *fu;
            sp.tile_ctr = tile_ctr;
            sp.refined = b.refined;
            sp.done = use_done ? b.flags : nullptr;
            if (prev && dfn)
                dfn<<<dgrid, KS_THREADS, ssmem, st>>>(sp);
            else
                sfn<<<sgrid, KS_THREADS, ssmem, st>>>(sp);
        } else {
            const AssignParams ap = assign_params<T>(b, x, n, d, k, gen.stages, accumulate, labels, use_done);
            gen.fn<<<gen.grid, KM_THREADS, gen.smem, st>>>(ap);
        }
    }
};

template <int D, int K>
static bool pick_small(void (*&fn)(SmallParams), void (*&dfn)(SmallParams), size_t& smem, int slot) {
    switch (slot) {
        case 0: fn = kmeans_small_kernel<D, K, 0>; dfn = kmeans_small_kernel<D, K, 0, true>; break;
        case 1: fn = kmeans_small_kernel<D, K, 1>; dfn = kmeans_small_kernel<D, K, 1, true>; break;
        case 2: fn = kmeans_small_kernel<D, K, 2>; dfn = kmeans_small_kernel<D, K, 2, true>; break;
        default: fn = kmeans_small_kernel<D, K, 3>; dfn = kmeans_small_kernel<D, K, 3, true>; break;
    }
    smem = small_smem<D, K>();
    return true;
}

template <int D, int K, int P>
static void pick_tc(Assigner<float>& A) {
    const char* w = std::getenv("DNDC_TC_WGS");
    if (w && w[0] == '1') {
        A.tfn = kmeans_tc_kernel<D, K, P, 1>;
        A.tsmem = TcCfg<D, K, P, 1>::SMEM;
        A.tthreads = TcCfg<D, K, P, 1>::THREADS;
        A.tc_delta = TcCfg<D, K, P, 1>::DELTA_OK;
    } else {
        A.tfn = kmeans_tc_kernel<D, K, P, 2>;
        A.tsmem = TcCfg<D, K, P, 2>::SMEM;
        A.tthreads = TcCfg<D, K, P, 2>::THREADS;
        A.tc_delta = TcCfg<D, K, P, 2>::DELTA_OK;
    }
    if (std::getenv("DNDC_TC_NO_DELTA")) A.tc_delta = false;
    A.rfn = kmeans_tc_refine_kernel<D, K>;
    A.rthreads = tc_refine_threads<D, K>();
    A.rsmem = TcRefineSmem<D, K>::BYTES;
    DNDC_CUDA(cudaFuncSetAttribute(A.rfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(A.rsmem)));
    if constexpr (P == 1 && D % 4 == 0) {
        if (!std::getenv("DNDC_TC_NO_FOUR") && A.tc_delta) {
            A.dtfn = kmeans_tcd_kernel<D, K>;
            A.dtsmem = TcdCfg<D, K>::SMEM;
            A.dtthreads = TcdCfg<D, K>::THREADS;
            if (!std::getenv("DNDC_TC_OLD_FULL")) {
                A.afn = kmeans_tc_accum_kernel<D, K>;
                A.asmem = TcAccumCfg<D, K>::SMEM;
                DNDC_CUDA(cudaFuncSetAttribute(A.afn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(A.asmem)));
            }
        }
    }
}

// DNDC_KMEANS_KERNEL=tc|small|generic overrides the automatic choice (tests, A/B timing).
static const char* kernel_override() {
    const char* v = std::getenv("DNDC_KMEANS_KERNEL");
    return v ? v : "";
}

template <typename T>
static Assigner<T> plan(dndc_ctx* ctx, int k, int d, int64_t n, const T* x) {
    Assigner<T> A;
    const std::string force = kernel_override();
    if constexpr (sizeof(T) == 4) {
        int P = 0;
        // tensor cores where the K*D FMAs dominate (measured: cfg3 k=64, d=64 runs
        // 2x the FFMA kernel); for k=8 the CUDA-core kernel is faster (its epilogue
        // is cheaper than the split + TMEM readback), so tc there only on request
        const bool want_tc = force == "tc" || (force.empty() && k * d >= 1024);
        if (want_tc && reinterpret_cast<uintptr_t>(x) % 16 == 0 && n > 0) {
            if (d == 18 && k == 8 && n % 2 == 0) { pick_tc<18, 8, 2>(A); P = 2; }
            else if (d == 32 && k == 8 && n % 2 == 0) { pick_tc<32, 8, 2>(A); P = 2; }
            else if (d == 64 && k == 64) { pick_tc<64, 64, 1>(A); P = 1; }
        }
        if (P > 0) {
            A.tc = true;
            A.tmap = make_tmap_2d_f32(x, static_cast<uint64_t>(n / P), static_cast<uint64_t>(P * d),
                                      static_cast<uint64_t>(P * d * 4), 32, 128, true);
            DNDC_CUDA(cudaFuncSetAttribute(A.tfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(A.tsmem)));
            if (A.dtfn)
                DNDC_CUDA(cudaFuncSetAttribute(A.dtfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(A.dtsmem)));
            int per_sm = 1;
            DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, A.tfn, A.tthreads, A.tsmem));
            per_sm = std::max(1, std::min(per_sm, 2));
            const int64_t tiles = std::max<int64_t>(ceil_div(n / P, 128), 1);
            A.sgrid = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(ctx->num_sms) * per_sm));
            // near-tie queue (DNDC_TC_QUEUE=0: refine inside the tc kernel) and
            // the refine kernel's accumulator; zeroed here, then the refine
            // kernel leaves them zero after every launch
            A.rq_cap = std::getenv("DNDC_TC_QUEUE") && std::getenv("DNDC_TC_QUEUE")[0] == '0'
                           ? 0u
                           : static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(n / 4, 4096), 1 << 22));
            A.rq_ctl = static_cast<unsigned*>(ctx->slot("km_rq_ctl", sizeof(unsigned) * 4));
            A.rq_row = static_cast<uint64_t*>(ctx->slot("km_rq_row", sizeof(uint64_t) * std::max(A.rq_cap, 1u)));
            A.rq_x = static_cast<float*>(ctx->slot("km_rq_x", sizeof(float) * d * std::max(A.rq_cap, 1u)));
            A.rq_cand = static_cast<unsigned long long*>(
                ctx->slot("km_rq_cand", sizeof(unsigned long long) * std::max(A.rq_cap, 1u)));
            A.racc = static_cast<long long*>(ctx->slot("km_racc", sizeof(long long) * (k * d + k)));
            DNDC_CUDA(cudaMemsetAsync(A.rq_ctl, 0, sizeof(unsigned) * 4, ctx->stream));
            DNDC_CUDA(cudaMemsetAsync(A.racc, 0, sizeof(long long) * (k * d + k), ctx->stream));
            int rper_sm = 1;
            DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rper_sm, A.rfn, A.rthreads, A.rsmem));
            A.rgrid = ctx->num_sms * std::max(rper_sm, 1);
            return A;
        }
    }
    if constexpr (sizeof(T) == 4) {
        if (force == "generic") {
            A.gen = plan_assign<T>(ctx, k, d, n);
            return A;
        }
        const int slot = ctx->km_slot % KS_SLOTS;
        bool ok = false;
        if (d == 18 && k == 8) ok = pick_small<18, 8>(A.sfn, A.dfn, A.ssmem, slot);
        else if (d == 32 && k == 8) ok = pick_small<32, 8>(A.sfn, A.dfn, A.ssmem, slot);
        if (ok) {
            A.small = true;
            A.slot = slot;
            DNDC_CUDA(cudaFuncSetAttribute(A.sfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(A.ssmem)));
            int per_sm = 1;
            DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, A.sfn, KS_THREADS, A.ssmem));
            per_sm = std::max(per_sm, 1);
            const int64_t tiles = std::max<int64_t>(ceil_div(n, KS_TILE), 1);
            A.sgrid = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(ctx->num_sms) * per_sm));
            DNDC_CUDA(cudaFuncSetAttribute(A.dfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(A.ssmem)));
            int dper_sm = 1;
            DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&dper_sm, A.dfn, KS_THREADS, A.ssmem));
            dper_sm = std::max(dper_sm, 1);
            A.dgrid = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(ctx->num_sms) * dper_sm));
            return A;
        }
    }
    A.gen = plan_assign<T>(ctx, k, d, n);
    return A;
}


static void validate_k(int64_t n, int k, const char* who) {
    if (k < 1) value_error(std::string(who) + ": k must be positive, got " + std::to_string(k));
    if (static_cast<int64_t>(k) > n)
        value_error(std::string(who) + ": k=" + std::to_string(k) + " exceeds the " + std::to_string(n) +
                    " available samples");
}

std::vector<int64_t> init_indices(int64_t n, int k, uint64_t seed) {
    // cluster.cpp:60-75 without the O(n) pool: only swapped positions differ
    // from the identity.
    if (k < 1 || static_cast<int64_t>(k) > n)
        value_error("kmeans_init_indices: k=" + std::to_string(k) + " out of range for n=" +
                    std::to_string(n));
    std::map<int64_t, int64_t> pool;
    auto get = [&](int64_t i) {
        auto it = pool.find(i);
        return it == pool.end() ? i : it->second;
    };
    for (int j = 0; j < k; ++j) {
        const uint64_t draw = splitmix64(seed ^ splitmix64(0x6b8b4567u + static_cast<uint64_t>(j)));
        const int64_t pick = j + static_cast<int64_t>(draw % static_cast<uint64_t>(n - j));
        const int64_t a = get(j), b = get(pick);
        pool[j] = b;
        pool[pick] = a;
    }
    std::vector<int64_t> out(k);
    for (int j = 0; j < k; ++j) out[j] = get(j);
    return out;
}

template <typename T>
static void init_centroids(dndc_ctx* ctx, const KmBuffers& b, const T* x_local, int64_t lo,
                           int64_t n_local, int m, int k, uint64_t seed, int64_t n_global, bool sync = true) {
    const auto idx = init_indices(n_global, k, seed);
    int64_t* didx = static_cast<int64_t*>(ctx->slot("km_idx", sizeof(int64_t) * k));
    int64_t* hidx = static_cast<int64_t*>(ctx->host_staging(sizeof(int64_t) * k));
    std::memcpy(hidx, idx.data(), sizeof(int64_t) * k);
    DNDC_CUDA(cudaMemcpyAsync(didx, hidx, sizeof(int64_t) * k, cudaMemcpyHostToDevice, ctx->stream));
    gather_rows_kernel<T><<<std::max(1, std::min(1024, (k * m + 255) / 256)), 256, 0, ctx->stream>>>(
        x_local, lo, lo + n_local, m, didx, k, b.c64);
    DNDC_LAUNCHED(ctx);
    allreduce_sum_f64(ctx, b.c64, static_cast<size_t>(k) * m, ctx->stream);
    // the pinned staging buffer is reused by later calls: finish the copy first
    // (kmeans_fit orders its next use on the stream instead)
    if (sync) DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// validation pass: sum x^2, non-finite count and max |x| of the shard -> b.sx2[0, 1, 3]
template <typename T>
static void scan_input(dndc_ctx* ctx, const KmBuffers& b, const T* x, int64_t count, cudaStream_t s) {
    // enough CTAs for ~32 KB in flight per SM, each thread >= 8 float4
    const int G = static_cast<int>(std::min<int64_t>(std::max<int64_t>(ceil_div(count, 256 * 32), 1),
                                                     static_cast<int64_t>(ctx->num_sms) * 8));
    validate_kernel<T><<<G, 256, 0, s>>>(x, count, b.pre);
    DNDC_LAUNCHED(ctx);
    validate_final_kernel<<<1, 256, 0, s>>>(b.pre, G, b.sx2);
    DNDC_LAUNCHED(ctx);
}

static void derive_tables(dndc_ctx* ctx, const KmBuffers& b, int k, int m) {
    derive_tables_kernel<<<1, 256, 0, ctx->stream>>>(k, m, dpad_of(m), b.c64, b.cn64, b.ct, b.cn32,
                                                     b.ctab, b.bounds);
    DNDC_LAUNCHED(ctx);
}

static UpdArgs upd_args(const KmBuffers& b, int k, int m, int world, const double* gathered, double* running,
                        bool delta, int it, double tol) {
    UpdArgs a{};
    a.k = k;
    a.d = m;
    a.dpad = dpad_of(m);
    a.world = world;
    a.gathered = gathered;
    a.gstride = static_cast<int64_t>(k) * m + k;
    a.running = running;
    a.accum = delta ? 1 : 0;
    a.c64 = b.c64;
    a.cn64 = b.cn64;
    a.ct = b.ct;
    a.cn32 = b.cn32;
    a.ctab = b.ctab;
    a.bounds = b.bounds;
    a.sx2 = b.sx2;
    a.trace = b.trace;
    a.disp = b.disp;
    a.flags = b.flags;
    a.iter = it;
    a.tol = tol;
    a.rd_running = running;
    a.rd_c64 = b.c64;
    a.rd_cn64 = b.cn64;
    a.rd_sx2 = b.sx2;
    return a;
}

// ---- the persistent fit (kmeans_persist.cuh): the full iterations in one
// cooperative launch (R = 2 rows per thread: counting sort of the tile), the
// delta iterations in a second, leaner one (R rows per thread, no sort)
struct PersistLaunch {
    void (*fn)(PersistParams) = nullptr;
    int grid = 0, static_tiles = 0;
    int wg = 1;  // warpgroups (virtual CTAs) per CTA
    size_t smem = 0;
    const char* name = "";
};
struct PersistPlan {
    PersistLaunch full, delta;
};

// Grid = CTAs that fit per SM x SMs (capped by the tile count), all
// co-resident (cooperative launch: the kernel's grid barrier needs it).
template <int D, int K, int R, int NST, int MINB, int MODE, bool TCS = false, int WG = 1>
static bool try_persist(dndc_ctx* ctx, int64_t n, PersistLaunch& P, const char* name) {
    using namespace persist;
    void (*fn)(PersistParams) = kmeans_persist_kernel<D, K, R, NST, MINB, MODE, TCS, WG>;
    const int64_t ntiles = std::max<int64_t>(ceil_div(n, THREADS * R), 1);
    const size_t smem = static_cast<size_t>(persist_layout<D, K, R, NST, TCS>().total) * WG;
    if (smem > 227 * 1024) return false;
    DNDC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, THREADS * WG, smem));
    if (occ < 1) return false;
    const int per_sm = WG == 1 ? std::min(occ, MINB) : 1;
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(ntiles, static_cast<int64_t>(WG)),
                                                        static_cast<int64_t>(per_sm) * ctx->num_sms));
    if (std::getenv("DNDC_PERSIST_VERBOSE"))
        std::fprintf(stderr, "[dndc] %s: smem %zu B, %d CTAs/SM, grid %d x %d warpgroups\n", name, smem, occ, grid,
                     WG);
    // static share: ~70% of the tiles (DNDC_PERSIST_STATIC=percent overrides)
    const char* e = std::getenv("DNDC_PERSIST_STATIC");
    const int pct = e ? std::max(0, std::min(100, std::atoi(e))) : 70;
    P.fn = fn;
    P.grid = grid;
    P.wg = WG;
    P.static_tiles = static_cast<int>(ntiles * pct / 100 / (static_cast<int64_t>(grid) * WG));
    P.smem = smem;
    P.name = name;
    return true;
}

// Iterations that sum every row before the delta iterations take over
// (DNDC_FULL_ITERS overrides; at least 1: a delta needs previous labels).
// Persistent fit: one (the delta launch takes over at iteration 1: 1.1% faster
// than two full iterations at cfg1, profiles/r02_env_sweep.txt).
static int persist_full_iters() {
    const char* e = std::getenv("DNDC_FULL_ITERS");
    return e ? std::max(1, std::atoi(e)) : 1;
}

// DNDC_PERSIST=0 disables the persistent fit; DNDC_PERSIST_DELTA=r4|r4s3
// picks the delta kernel's (rows per thread, stages) instantiation (A/B timing).
static bool plan_persist(dndc_ctx* ctx, int k, int m, int64_t n_local, PersistPlan& P) {
    const char* e = std::getenv("DNDC_PERSIST");
    if (e && std::string(e) == "0") return false;
    if (m == 18 && k == 8) {
        using namespace persist;
        // DNDC_PERSIST_TC=1: scores on the tensor core (persist_top2_tc, four
        // warpgroups per CTA).  Measured slower (~150 us per
        // delta iteration against ~88: 18 MMAs of N = 16 per 256-row tile, each
        // tile's MMAs waited for), so not the default.
        const char* t = std::getenv("DNDC_PERSIST_TC");
        if (t && std::string(t) == "1") {
            if (!try_persist<18, 8, 2, 2, 4, FULL_ONLY, true, 4>(ctx, n_local, P.full,
                                                                 "kmeans_persist_kernel<18,8,R2,S2,full,tc,wg4>"))
                return false;
            return try_persist<18, 8, 2, 2, 4, DELTA_ONLY, true, 4>(ctx, n_local, P.delta,
                                                                    "kmeans_persist_kernel<18,8,R2,S2,delta,tc,wg4>");
        }
        if (!try_persist<18, 8, 2, 2, 4, FULL_ONLY>(ctx, n_local, P.full, "kmeans_persist_kernel<18,8,R2,S2,full>"))
            return false;
        const char* d = std::getenv("DNDC_PERSIST_DELTA");
        const std::string v = d ? d : "";
        if (v == "r4s3") return try_persist<18, 8, 4, 3, 2, DELTA_ONLY>(ctx, n_local, P.delta, "kmeans_persist_kernel<18,8,R4,S3,delta>");
        if (v == "r4") return try_persist<18, 8, 4, 2, 3, DELTA_ONLY>(ctx, n_local, P.delta, "kmeans_persist_kernel<18,8,R4,S2,delta>");
        if (v == "r1s3") return try_persist<18, 8, 1, 3, 4, DELTA_ONLY>(ctx, n_local, P.delta, "kmeans_persist_kernel<18,8,R1,S3,delta>");
        if (v == "r1s4") return try_persist<18, 8, 1, 4, 4, DELTA_ONLY>(ctx, n_local, P.delta, "kmeans_persist_kernel<18,8,R1,S4,delta>");
        if (v == "r2s3") return try_persist<18, 8, 2, 3, 3, DELTA_ONLY>(ctx, n_local, P.delta, "kmeans_persist_kernel<18,8,R2,S3,delta>");
        return try_persist<18, 8, 2, 2, 4, DELTA_ONLY>(ctx, n_local, P.delta, "kmeans_persist_kernel<18,8,R2,S2,delta>");
    }
    return false;
}

template <typename T>
static void kmeans_fit(dndc_ctx* ctx, const T* x_local, int64_t n_local, int64_t n_global, int64_t m64,
                       int k, int max_iter, double tol, uint64_t seed, const double* init_host,
                       double* cent_host, double* trace_host, int* iters_host) {
    validate_k(n_global, k, "kmeans_fit");
    if (max_iter < 1) value_error("kmeans_fit: max_iter must be positive, got " + std::to_string(max_iter));
    std::vector<int64_t> off, ext;
    chunk_map(n_global, ctx->world, off, ext);
    if (n_local != ext[ctx->rank])
        value_error("kmeans_fit: local shard has " + std::to_string(n_local) + " rows, chunk_map gives " +
                    std::to_string(ext[ctx->rank]));
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    // A shard that is not 16-byte aligned is copied to an aligned scratch
    // buffer first (the bulk-copy / TMA kernels need the alignment), so that on
    // every rank the kernel plan below follows from global facts only -- (k, m),
    // the chunk_map extents, the environment -- and needs no cross-rank
    // agreement in the common case.
    if (ctx->world > 1 && n_local > 0 && reinterpret_cast<uintptr_t>(x_local) % 16 != 0) {
        T* xa = static_cast<T*>(ctx->slot("km_xalign", sizeof(T) * static_cast<size_t>(n_local) * m));
        DNDC_CUDA(cudaMemcpyAsync(xa, x_local, sizeof(T) * static_cast<size_t>(n_local) * m,
                                  cudaMemcpyDeviceToDevice, s));
        x_local = xa;
    }
    Assigner<T> A = plan<T>(ctx, k, m, n_local, x_local);
    // the kernel choice fixes the stats protocol (fused NVLink exchange,
    // delta vs full sums): every rank must take the same one
    PersistPlan PP;
    bool persist = sizeof(T) == 4 && A.small && (ctx->world == 1 || ctx->p2p) && n_local > 0 &&
                   plan_persist(ctx, k, m, n_local, PP);
    // The plan differs between ranks only when some rank's shard is empty, or
    // under a kernel override (forced tc packs row pairs: shard parity).  Every
    // rank evaluates this rule from the same global facts, so all of them take
    // the host-synchronised agreement below or none does (skipping it saves
    // ~40 us per fit at N = 4: tools/gpu_plan_ab.sh).  DNDC_PLAN_AGREE=1 forces it.
    bool agree = std::getenv("DNDC_PLAN_AGREE") != nullptr || !std::string(kernel_override()).empty();
    for (int r = 0; r < ctx->world; ++r) agree = agree || ext[r] == 0;
    if (ctx->world > 1 && agree) {
        const int code = (persist ? 1 : 0) | (A.small ? 2 : 0) | (A.tc ? 4 : 0) | (A.tc && A.tc_delta ? 8 : 0);
        int* dcode = static_cast<int*>(ctx->slot("km_plan", sizeof(int) * (ctx->world + 1)));
        DNDC_CUDA(cudaMemcpyAsync(dcode + ctx->world, &code, sizeof(int), cudaMemcpyHostToDevice, s));
        xport_allgather(ctx, dcode + ctx->world, dcode, sizeof(int), s);
        std::vector<int> all(ctx->world);
        DNDC_CUDA(cudaMemcpyAsync(all.data(), dcode, sizeof(int) * ctx->world, cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaStreamSynchronize(s));
        for (int r = 1; r < ctx->world; ++r)
            if (all[r] != all[0]) {  // disagreement (e.g. an empty shard): the generic full-sum path everywhere
                A = Assigner<T>{};
                A.gen = plan_assign<T>(ctx, k, m, n_local);
                persist = false;
                break;
            }
    }
    const KmBuffers b = buffers(ctx, k, m, max_iter, A.max_grid());
    const int S = k * m + k;

    // ---- validation + sum |x|^2 (one pass), agreed by every rank, all on the
    // device: a non-finite value anywhere sets flags[2] (and the iterations
    // skip); the host raises after the single synchronisation at the end
    scan_input<T>(ctx, b, x_local, n_local * m, s);
    const bool fused_init = ctx->world > 1 && !init_host && !ctx->group;
    if (fused_init) {
        // one collective for the validation stats and the initial centroids
        // (the k seeded rows, each owned by one rank: cluster.cpp:60-81)
        const int km = k * m;
        double* pre = static_cast<double*>(ctx->slot("km_pre_init", sizeof(double) * (2 + km)));
        double* pre_all = static_cast<double*>(ctx->slot("km_pre_all", sizeof(double) * (2 + km) * ctx->world));
        const auto idx = init_indices(n_global, k, seed);
        int64_t* didx = static_cast<int64_t*>(ctx->slot("km_idx", sizeof(int64_t) * k));
        int64_t* hidx = static_cast<int64_t*>(ctx->host_staging(sizeof(int64_t) * k));
        std::memcpy(hidx, idx.data(), sizeof(int64_t) * k);
        DNDC_CUDA(cudaMemcpyAsync(didx, hidx, sizeof(int64_t) * k, cudaMemcpyHostToDevice, s));
        DNDC_CUDA(cudaMemcpyAsync(pre, b.sx2, sizeof(double) * 2, cudaMemcpyDeviceToDevice, s));
        gather_rows_kernel<T><<<std::max(1, std::min(1024, (km + 255) / 256)), 256, 0, s>>>(
            x_local, off[ctx->rank], off[ctx->rank] + n_local, m, didx, k, pre + 2);
        DNDC_LAUNCHED(ctx);
        allgather_f64(ctx, pre, pre_all, static_cast<size_t>(2 + km), s);
        validate_init_fold_kernel<<<std::max(1, std::min(64, (km + 255) / 256)), 256, 0, s>>>(
            pre_all, ctx->world, km, b.sx2, b.flags, b.c64);
        DNDC_LAUNCHED(ctx);
    } else {
        allgather_f64(ctx, b.sx2, b.gathered, 2, s);  // gathered: scratch, world x 2
        validate_fold_kernel<<<1, 32, 0, s>>>(b.gathered, ctx->world, b.sx2, b.flags);
        DNDC_LAUNCHED(ctx);
    }

    // ---- initial centroids (no host round trip: the pinned staging buffer is
    // next written by the results copy, which is ordered after this upload)
    if (fused_init) {
        // (above)
    } else if (init_host) {
        double* h = static_cast<double*>(ctx->host_staging(sizeof(double) * k * m));
        std::memcpy(h, init_host, sizeof(double) * k * m);
        DNDC_CUDA(cudaMemcpyAsync(b.c64, h, sizeof(double) * k * m, cudaMemcpyHostToDevice, s));
    } else {
        init_centroids<T>(ctx, b, x_local, off[ctx->rank], n_local, m, k, seed, n_global, false);
    }
    derive_tables(ctx, b, k, m);

    // ---- the Lloyd loop, one graph per (shape, buffers, max_iter, tol)
    // small kernel: every iteration records int8 labels; the first ones
    // accumulate full sums, later ones only the rows whose label changed
    const bool use_delta = A.small || (A.tc && A.tc_delta);
    // (+64: kmeans_tc_accum_kernel bulk-copies labels in 16-byte multiples)
    int8_t* lab8 = use_delta ? static_cast<int8_t*>(ctx->slot("km_lab8", std::max<int64_t>(n_local, 1) + 64)) : nullptr;
    if (!ctx->km) ctx->km = new KMeansState();
    KMeansState* km = ctx->km;
    if (km->timing && km->ev.size() < 2 * static_cast<size_t>(max_iter)) {
        free_events(km);
        km->ev.resize(2 * static_cast<size_t>(max_iter));
        for (auto& e : km->ev) DNDC_CUDA(cudaEventCreate(&e));
        km->clear_graphs();
    }
    // one launch per iteration (fused tail) on one GPU or with the NVLink
    // peer exchange; otherwise assign -> reduce -> NCCL allgather -> update
    const bool fuse = A.small && (ctx->world == 1 || ctx->p2p) && !std::getenv("DNDC_NO_FUSE");
    // (persist: the whole loop in cooperative launches, planned above)
    const int ncounters = 2;
    unsigned* tile_ctr = b.counters + 1;
    // (slots are allocated here, outside the capture: cudaMalloc is not capturable)
    unsigned long long* acc3 =
        persist ? static_cast<unsigned long long*>(ctx->slot("km_pacc", sizeof(unsigned long long) * 3 * S)) : nullptr;
    // per launch: [0] root arrival, [1..32] group arrivals, [33] go -> 40 words x 2 launches
    unsigned* words = persist ? static_cast<unsigned*>(ctx->slot("km_pwords", sizeof(unsigned) * 80)) : nullptr;
    double* gst = persist ? static_cast<double*>(ctx->slot("km_pgstats", sizeof(double) * 2 * S)) : nullptr;
    unsigned* tctr = persist ? static_cast<unsigned*>(ctx->slot("km_ptiles", sizeof(unsigned) * max_iter)) : nullptr;
    int8_t* plab = persist ? static_cast<int8_t*>(ctx->slot("km_plab", static_cast<size_t>(n_local))) : nullptr;
    // multi-CTA update (per-iteration launches): per-cluster results + ticket
    double* upd_red = static_cast<double*>(ctx->slot("km_upd_red", sizeof(double) * 4 * k));
    unsigned* upd_ticket = static_cast<unsigned*>(ctx->slot("km_upd_ticket", sizeof(unsigned)));
    DNDC_CUDA(cudaMemsetAsync(upd_ticket, 0, sizeof(unsigned), s));
    unsigned long long* pmarks = nullptr;
    if (persist && std::getenv("DNDC_PERSIST_TRACE")) {
        const int tg = std::max(PP.full.grid * PP.full.wg, PP.delta.grid * PP.delta.wg);  // virtual CTAs
        ctx->persist_trace_len = static_cast<int64_t>(max_iter) * (2 * tg + 2);
        ctx->persist_trace_grid = tg;
        pmarks = static_cast<unsigned long long*>(
            ctx->slot("km_pmarks", sizeof(unsigned long long) * ctx->persist_trace_len));
    }
    auto record_persist = [&](cudaStream_t st) {
        persist_reset_kernel<<<1, 256, 0, st>>>(b.flags, b.refined, acc3, 3 * S, words, 80, tctr, max_iter);
        const int F = std::max(1, std::min(persist_full_iters(), max_iter));
        PersistParams pp{};
        pp.x = reinterpret_cast<const float*>(x_local);
        pp.n = n_local;
        pp.max_iter = max_iter;
        pp.full_iters = F;
        pp.tol = tol;
        pp.c64_init = b.c64;
        pp.c64_out = b.c64;
        pp.run_io = b.running;
        pp.trace = b.trace;
        pp.disp = b.disp;
        pp.flags = b.flags;
        pp.sx2 = b.sx2;
        pp.acc = acc3;
        pp.gstats = gst;
        pp.refined = b.refined;
        pp.world = ctx->world;
        pp.rank = ctx->rank;
        pp.peers = ctx->world > 1 ? ctx->peer_bases_dev : nullptr;
        pp.labels = plab;
        pp.tile_ctr = tctr;
        pp.trace_marks = pmarks;
        pp.trace_grid = ctx->persist_trace_grid;
        if (km->timing) DNDC_CUDA(cudaEventRecordWithFlags(km->ev[0], st, cudaEventRecordExternal));
        auto launch = [&](const PersistLaunch& L, int it0, int it1, unsigned* arrive, unsigned* go) {
            PersistParams q = pp;
            q.it_begin = it0;
            q.it_end = it1;
            q.arrive = arrive;
            q.go = go;
            q.static_tiles = L.static_tiles;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(L.grid);
            cfg.blockDim = dim3(persist::THREADS * L.wg);
            cfg.dynamicSmemBytes = L.smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
            attr[0].val.cooperative = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            DNDC_CUDA(cudaLaunchKernelEx(&cfg, L.fn, q));
        };
        launch(PP.full, 0, F, words, words + 33);
        if (F < max_iter) launch(PP.delta, F, max_iter, words + 40, words + 73);
        if (km->timing) DNDC_CUDA(cudaEventRecordWithFlags(km->ev[1], st, cudaEventRecordExternal));
    };
    // tc full iterations with the labels buffer launch one kernel more (the sums pass)
    const unsigned long long split_full_iters =
        (A.tc && A.afn && lab8) ? static_cast<unsigned long long>(std::min(KS_FULL_ITERS, max_iter)) : 0ull;
    auto record = [&](cudaStream_t st) {
        if (persist) {
            record_persist(st);
            return;
        }
        kmeans_reset_kernel<<<1, 1, 0, st>>>(b.flags, b.refined, b.counters, ncounters, b.acc64, S);
        for (int it = 0; it < max_iter; ++it) {
            // iterations 0 and 1 accumulate every row (after the first update most
            // labels still move); from iteration 2 on only the rows that changed
            const bool delta = use_delta && it > KS_FULL_ITERS - 1;
            FuseArgs fa{};
            if (fuse) {
                fa.on = 1;
                fa.acc64 = b.acc64;
                fa.xabs = b.sx2 + 3;
                fa.n = n_local;
                fa.counters = b.counters;
                fa.stats = b.stats;
                fa.peers = ctx->world > 1 ? ctx->peer_bases_dev : nullptr;
                fa.rank = ctx->rank;
                fa.tile_ctr = tile_ctr;
                fa.upd = upd_args(b, k, m, ctx->world, nullptr, b.running, delta, it, tol);
            }
            if (km->timing) DNDC_CUDA(cudaEventRecordWithFlags(km->ev[2 * it], st, cudaEventRecordExternal));
            if (A.small && !fuse) zero_u32_kernel<<<1, 32, 0, st>>>(tile_ctr, 1);
            // static tile assignment (no tile counter): every CTA's f64 partial
            // covers the same rows in every run, so the fit is bit-repeatable
            // (the dynamic counter made it depend on arrival order)
            A.launch(b, x_local, n_local, m, k, true, nullptr, true, st, delta ? lab8 : nullptr, lab8,
                     fuse ? &fa : nullptr, nullptr);
            if (km->timing) DNDC_CUDA(cudaEventRecordWithFlags(km->ev[2 * it + 1], st, cudaEventRecordExternal));
            if (fuse) continue;
            reduce_partials_kernel<<<(S + 7) / 8, 256, 0, st>>>(b.partials, A.grid_for(delta), S, b.stats, b.flags);
            if (ctx->world > 1) allgather_f64(ctx, b.stats, b.gathered, S, st);
            const UpdArgs ua = upd_args(b, k, m, ctx->world, ctx->world > 1 ? b.gathered : b.stats,
                                        use_delta ? b.running : nullptr, delta, it, tol);
            if (m <= UPD_MC_MAXD && !std::getenv("DNDC_UPDATE_1CTA")) {
                const int ug = std::min(k, ctx->num_sms);
                kmeans_update_mc_kernel<<<ug, 256, sizeof(double) * 3 * m, st>>>(ua, upd_red, upd_ticket);
            } else {
                kmeans_update_kernel<<<1, 256, update_smem(k, m), st>>>(ua);
            }
        }
    };
    if (ctx->group) {
        // ranks sharing GPUs: the stats exchange is host-staged, not capturable
        record(s);  // (allgather_f64 counts itself here)
        ctx->launches += 1 + ((A.small || A.tc) ? 4ull : 3ull) * max_iter + split_full_iters;
    }
    cudaStream_t gs = ctx->own_stream;
    char keybuf[256];
    std::snprintf(keybuf, sizeof(keybuf), "%p/%lld/%d/%d/%d/%.17g/%p/%d/%d/%d/%d/%llu", (const void*)x_local,
                  (long long)n_local, m, k, max_iter, tol, (void*)s, A.grid(), ctx->world, km->timing ? 1 : 0,
                  (fuse ? 1 : 0) + (persist ? 2 : 0), static_cast<unsigned long long>(ctx->slot_gen));
    const std::string key = std::string(sizeof(T) == 4 ? "f32/" : "f64/") + keybuf;
    cudaGraphExec_t exec = nullptr;
    for (size_t i = 0; i < km->graphs.size() && !ctx->group; ++i)
        if (km->graphs[i].first == key) {
            exec = km->graphs[i].second;
            std::rotate(km->graphs.begin(), km->graphs.begin() + i, km->graphs.begin() + i + 1);
            break;
        }
    if (!exec && !ctx->group) {
        const uint64_t before = ctx->counters.allgathers;
        cudaGraph_t graph;
        // capture on the context's own (non-legacy) stream: the legacy default
        // stream that torch hands us cannot be captured
        DNDC_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        try {
            record(gs);
        } catch (...) {
            cudaStreamEndCapture(gs, &graph);
            throw;
        }
        DNDC_CUDA(cudaStreamEndCapture(gs, &graph));
        ctx->counters.allgathers = before;  // counted per replay below
        DNDC_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        DNDC_CUDA(cudaGraphDestroy(graph));
        km->graphs.insert(km->graphs.begin(), {key, exec});
        while (km->graphs.size() > 4) {
            cudaGraphExecDestroy(km->graphs.back().second);
            km->graphs.pop_back();
        }
    }
    if (!ctx->group) {
    DNDC_CUDA(cudaEventRecord(ctx->ev_a, s));
    DNDC_CUDA(cudaStreamWaitEvent(gs, ctx->ev_a, 0));
    DNDC_CUDA(cudaGraphLaunch(exec, gs));
    DNDC_CUDA(cudaEventRecord(ctx->ev_b, gs));
    DNDC_CUDA(cudaStreamWaitEvent(s, ctx->ev_b, 0));
    // reset + per iteration: assign (fused) | [tile reset,] assign, reduce, update
    // (persistent: reset + the one cooperative launch)
    ctx->launches += persist ? (max_iter > persist_full_iters() ? 3ull : 2ull)
                             : 1 + (fuse ? 1ull : (A.small || A.tc) ? 4ull : 3ull) * max_iter + split_full_iters;
    if (ctx->world > 1) ctx->counters.allgathers += max_iter;
    }
    ctx->last_kernel = persist ? (max_iter > persist_full_iters() ? PP.delta.name : PP.full.name) : "";

    // ---- results
    const size_t hb = sizeof(double) * (k * m + max_iter) + 64;
    unsigned char* h = static_cast<unsigned char*>(ctx->host_staging(hb));
    DNDC_CUDA(cudaMemcpyAsync(h, b.c64, sizeof(double) * k * m, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaMemcpyAsync(h + sizeof(double) * k * m, b.trace, sizeof(double) * max_iter,
                              cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaMemcpyAsync(h + sizeof(double) * (k * m + max_iter), b.flags, sizeof(int) * 4,
                              cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaMemcpyAsync(h + sizeof(double) * (k * m + max_iter) + 16, b.refined,
                              sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    const int* flags = reinterpret_cast<const int*>(h + sizeof(double) * (k * m + max_iter));
    if (flags[2]) value_error("kmeans_fit: input contains non-finite values");
    if (flags[3])
        throw Error(DNDC_ETIMEOUT, "kmeans_fit: a peer rank did not arrive at the per-iteration stats exchange "
                                   "within the deadlock timeout (transport.cpp:76-93)");
    std::memcpy(cent_host, h, sizeof(double) * k * m);
    const int iters = flags[1];
    std::memcpy(trace_host, h + sizeof(double) * k * m, sizeof(double) * max_iter);
    *iters_host = iters;
    if (km->timing && persist) {
        float t = 0.f;
        DNDC_CUDA(cudaEventElapsedTime(&t, km->ev[0], km->ev[1]));
        km->per_launch_ms.assign(1, t);
        km->assign_ms = t;
        km->assign_launches = 1;
    } else if (km->timing) {
        // iterations past convergence return at once; only the ones that ran count
        double tot = 0.0;
        km->per_launch_ms.assign(iters, 0.0);
        for (int it = 0; it < iters; ++it) {
            float t = 0.f;
            DNDC_CUDA(cudaEventElapsedTime(&t, km->ev[2 * it], km->ev[2 * it + 1]));
            tot += t;
            km->per_launch_ms[it] = t;
        }
        km->assign_ms = tot;
        km->assign_launches = iters;
    }
    ctx->last_refined = static_cast<int64_t>(
        *reinterpret_cast<const unsigned long long*>(h + sizeof(double) * (k * m + max_iter) + 16));
}

template <typename T>
static void kmeans_predict(dndc_ctx* ctx, const T* x, int64_t n, int64_t m64, const double* cent_host,
                           int k, int32_t* labels) {
    if (k < 1) value_error("kmeans_predict: k must be positive");
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    const Assigner<T> A = plan<T>(ctx, k, m, n, x);
    const KmBuffers b = buffers(ctx, k, m, 1, A.grid());
    double* h = static_cast<double*>(ctx->host_staging(sizeof(double) * k * m));
    std::memcpy(h, cent_host, sizeof(double) * k * m);
    DNDC_CUDA(cudaMemcpyAsync(b.c64, h, sizeof(double) * k * m, cudaMemcpyHostToDevice, s));
    DNDC_CUDA(cudaMemsetAsync(b.refined, 0, sizeof(unsigned long long), s));
    derive_tables(ctx, b, k, m);
    if (n > 0) {
        if (A.small || A.tc) scan_input<T>(ctx, b, x, n * m, s);
        A.launch(b, x, n, m, k, false, labels, false, s);
        DNDC_LAUNCHED(ctx);
        if (A.tc) ctx->launches++;  // + the near-tie refine kernel
    }
    unsigned long long* hr = reinterpret_cast<unsigned long long*>(h);
    DNDC_CUDA(cudaMemcpyAsync(hr, b.refined, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    ctx->last_refined = static_cast<int64_t>(*hr);
}

// One assignment/accumulation pass against given centroids: local stats and
// local inertia (sum |x|^2 + sum_j n_j |c_j|^2 - 2 c_j . S_j, the fit's form).
template <typename T>
static void kmeans_step(dndc_ctx* ctx, const T* x, int64_t n, int64_t m64, const double* cent_host, int k,
                        double* stats_host, int32_t* labels) {
    if (k < 1) value_error("kmeans_step: k must be positive");
    if (n < 0 || m64 < 1) value_error("kmeans_step: bad extents");
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    const Assigner<T> A = plan<T>(ctx, k, m, n, x);
    const KmBuffers b = buffers(ctx, k, m, 1, A.grid());
    const int S = k * m + k;
    double* h = static_cast<double*>(ctx->host_staging(sizeof(double) * std::max(k * m, S + 4)));
    std::memcpy(h, cent_host, sizeof(double) * k * m);
    DNDC_CUDA(cudaMemcpyAsync(b.c64, h, sizeof(double) * k * m, cudaMemcpyHostToDevice, s));
    DNDC_CUDA(cudaMemsetAsync(b.refined, 0, sizeof(unsigned long long), s));
    DNDC_CUDA(cudaMemsetAsync(b.stats, 0, sizeof(double) * S, s));
    DNDC_CUDA(cudaMemsetAsync(b.sx2, 0, sizeof(double) * 4, s));
    derive_tables(ctx, b, k, m);
    if (n > 0) {
        scan_input<T>(ctx, b, x, n * m, s);
        A.launch(b, x, n, m, k, true, labels, false, s);
        DNDC_LAUNCHED(ctx);
        if (A.tc) ctx->launches++;  // + the near-tie refine kernel
        reduce_partials_kernel<<<(S + 7) / 8, 256, 0, s>>>(b.partials, A.grid(), S, b.stats, nullptr);
        DNDC_LAUNCHED(ctx);
    }
    DNDC_CUDA(cudaMemcpyAsync(h, b.stats, sizeof(double) * S, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaMemcpyAsync(h + S, b.sx2, sizeof(double), cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    double inertia = h[S];
    for (int j = 0; j < k; ++j) {
        double cn = 0.0, dot = 0.0;
        for (int f = 0; f < m; ++f) {
            const double c = cent_host[static_cast<int64_t>(j) * m + f];
            cn += c * c;
            dot += c * h[j * m + f];
        }
        inertia += h[k * m + j] * cn - 2.0 * dot;
    }
    std::memcpy(stats_host, h, sizeof(double) * S);
    stats_host[S] = inertia;
}

template <typename T>
static void init_centroids_api(dndc_ctx* ctx, const T* x_local, int64_t n_local, int64_t n_global,
                               int64_t m, int k, uint64_t seed, double* out_host) {
    validate_k(n_global, k, "kmeans_init_centroids");
    std::vector<int64_t> off, ext;
    chunk_map(n_global, ctx->world, off, ext);
    if (n_local != ext[ctx->rank]) value_error("kmeans_init_centroids: shard does not match chunk_map");
    const KmBuffers b = buffers(ctx, k, static_cast<int>(m), 1, 1);
    init_centroids<T>(ctx, b, x_local, off[ctx->rank], n_local, static_cast<int>(m), k, seed, n_global);
    double* h = static_cast<double*>(ctx->host_staging(sizeof(double) * k * m));
    DNDC_CUDA(cudaMemcpyAsync(h, b.c64, sizeof(double) * k * m, cudaMemcpyDeviceToHost, ctx->stream));
    DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(out_host, h, sizeof(double) * k * m);
}

// Times the dominant kernel (assign + accumulate) alone: `reps` back-to-back
// launches bracketed by CUDA events on the context's stream, against the
// centroid tables of the last fit (or the first k rows when there was none).
static void time_assign(dndc_ctx* ctx, const float* x, int64_t n, int64_t m64, int k, int reps, double* ms,
                        double* bytes) {
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    const Assigner<float> A = plan<float>(ctx, k, m, n, x);
    const bool fresh = ctx->slots.find("km_c64") == ctx->slots.end();
    const KmBuffers b = buffers(ctx, k, m, 1, A.grid());
    if (fresh) {
        std::vector<int64_t> idx(k);
        for (int j = 0; j < k; ++j) idx[j] = j;
        int64_t* didx = static_cast<int64_t*>(ctx->slot("km_idx", sizeof(int64_t) * k));
        DNDC_CUDA(cudaMemcpy(didx, idx.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice));
        gather_rows_kernel<float><<<1, 256, 0, s>>>(x, 0, n, m, didx, k, b.c64);
        derive_tables(ctx, b, k, m);
    }
    scan_input<float>(ctx, b, x, n * m, s);
    cudaEvent_t e0, e1;
    DNDC_CUDA(cudaEventCreate(&e0));
    DNDC_CUDA(cudaEventCreate(&e1));
    A.launch(b, x, n, m, k, true, nullptr, false, s);  // warm
    DNDC_CUDA(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) A.launch(b, x, n, m, k, true, nullptr, false, s);
    DNDC_CUDA(cudaEventRecord(e1, s));
    DNDC_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    DNDC_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ctx->launches += reps + 1;
    *ms = static_cast<double>(t) / reps;
    *bytes = static_cast<double>(n) * m * sizeof(float);
}

}  // namespace dndc

using dndc::guard;

extern "C" {

int dndc_kmeans_init_indices(int64_t n, int k, uint64_t seed, int64_t* out_host) {
    return guard([&] {
        const auto v = dndc::init_indices(n, k, seed);
        std::memcpy(out_host, v.data(), v.size() * sizeof(int64_t));
    });
}

int dndc_kmeans_init_centroids_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local,
                                   int64_t n_global, int64_t m, int k, uint64_t seed,
                                   double* centroids_host) {
    return guard([&] {
        dndc::init_centroids_api<float>(ctx, x_local, n_local, n_global, m, k, seed, centroids_host);
    });
}

int dndc_kmeans_fit_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, int64_t n_global,
                        int64_t m, int k, int max_iter, double tol, uint64_t seed,
                        const double* init_centroids_host, double* centroids_host,
                        double* inertia_trace_host, int* iterations_run) {
    return guard([&] {
        dndc::kmeans_fit<float>(ctx, x_local, n_local, n_global, m, k, max_iter, tol, seed,
                                init_centroids_host, centroids_host, inertia_trace_host, iterations_run);
    });
}

int dndc_kmeans_fit_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, int64_t n_global,
                        int64_t m, int k, int max_iter, double tol, uint64_t seed,
                        const double* init_centroids_host, double* centroids_host,
                        double* inertia_trace_host, int* iterations_run) {
    return guard([&] {
        dndc::kmeans_fit<double>(ctx, x_local, n_local, n_global, m, k, max_iter, tol, seed,
                                 init_centroids_host, centroids_host, inertia_trace_host, iterations_run);
    });
}

int dndc_kmeans_predict_f32(dndc_ctx* ctx, const float* x, int64_t n, int64_t m,
                            const double* centroids_host, int k, int32_t* labels) {
    return guard([&] { dndc::kmeans_predict<float>(ctx, x, n, m, centroids_host, k, labels); });
}

int dndc_kmeans_predict_f64(dndc_ctx* ctx, const double* x, int64_t n, int64_t m,
                            const double* centroids_host, int k, int32_t* labels) {
    return guard([&] { dndc::kmeans_predict<double>(ctx, x, n, m, centroids_host, k, labels); });
}

int dndc_kmeans_step_f32(dndc_ctx* ctx, const float* x, int64_t n, int64_t m, const double* centroids_host,
                         int k, double* stats_host, int32_t* labels) {
    return guard([&] { dndc::kmeans_step<float>(ctx, x, n, m, centroids_host, k, stats_host, labels); });
}

int dndc_kmeans_step_f64(dndc_ctx* ctx, const double* x, int64_t n, int64_t m, const double* centroids_host,
                         int k, double* stats_host, int32_t* labels) {
    return guard([&] { dndc::kmeans_step<double>(ctx, x, n, m, centroids_host, k, stats_host, labels); });
}

int dndc_kmeans_time_assign_f32(dndc_ctx* ctx, const float* x, int64_t n, int64_t m, int k, int reps,
                                double* ms_per_launch, double* algorithmic_bytes) {
    return guard([&] { dndc::time_assign(ctx, x, n, m, k, reps, ms_per_launch, algorithmic_bytes); });
}

#ifdef KS_TAIL_TRACE
int dndc_internal_tail_trace(unsigned long long* out16) {
    return guard([&] { DNDC_CUDA(cudaMemcpyFromSymbol(out16, dndc::g_tail_trace, 16 * sizeof(unsigned long long))); });
}
int dndc_internal_iter_trace(unsigned long long* out128) {
    return guard([&] { DNDC_CUDA(cudaMemcpyFromSymbol(out128, dndc::g_iter_trace, 128 * sizeof(unsigned long long))); });
}
int dndc_internal_cta_trace(unsigned long long* out4096) {
    return guard([&] { DNDC_CUDA(cudaMemcpyFromSymbol(out4096, dndc::g_cta_trace, 4096 * sizeof(unsigned long long))); });
}
#endif

#ifdef TCD_TRACE
extern "C" int dndc_internal_tcd_trace(unsigned long long* out512) {
    return guard([&] { DNDC_CUDA(cudaMemcpyFromSymbol(out512, dndc::g_tcd_trace, 512 * sizeof(unsigned long long))); });
}
#endif

int dndc_kmeans_assign_timing(dndc_ctx* ctx, int enable) {
    return guard([&] {
        if (!ctx->km) ctx->km = new dndc::KMeansState();
        if (ctx->km->timing != (enable != 0)) ctx->km->clear_graphs();  // re-record the graphs
        ctx->km->timing = enable != 0;
    });
}

int dndc_internal_assign_times(const dndc_ctx* ctx, double* out, int cap) {
    const int n = ctx->km ? static_cast<int>(ctx->km->per_launch_ms.size()) : 0;
    for (int i = 0; i < n && i < cap; ++i) out[i] = ctx->km->per_launch_ms[i];
    return n;
}

int dndc_kmeans_last_assign_ms(const dndc_ctx* ctx, double* total_ms, int* launches) {
    *total_ms = ctx->km ? ctx->km->assign_ms : 0.0;
    *launches = ctx->km ? ctx->km->assign_launches : 0;
    return DNDC_OK;
}

int dndc_kmeans_last_refined(const dndc_ctx* ctx, int64_t* rows_refined) {
    *rows_refined = ctx->last_refined;
    return DNDC_OK;
}

const char* dndc_kmeans_last_kernel(const dndc_ctx* ctx) { return ctx ? ctx->last_kernel : ""; }

// Diagnostics (tools/persist_trace.py): the %globaltimer marks of the last
// persistent fit run with DNDC_PERSIST_TRACE set; returns the count copied.
int64_t dndc_kmeans_persist_trace(dndc_ctx* ctx, unsigned long long* out_host, int64_t cap, int* grid) {
    auto it = ctx->slots.find("km_pmarks");
    if (it == ctx->slots.end() || ctx->persist_trace_len == 0) return 0;
    const int64_t n = std::min(cap, ctx->persist_trace_len);
    if (cudaMemcpy(out_host, it->second.first, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    *grid = ctx->persist_trace_grid;
    return n;
}

}  // extern "C"
