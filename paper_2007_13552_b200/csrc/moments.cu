// moments.cu -- A13/A14: per-column count/mean/M2 along the split axis 0.
//
// Reference: welford_update, local_moments_axis, combine, axis_statistic,
// mean_axis / var_axis / stddev_axis (moments.cpp:10-140).
//
// One pass over the shard.  Thread (column c, row-lane r) walks rows r,
// r + R, ... of its CTA's row range in chunks of KC rows: inside a chunk it
// keeps f64 sums of (x - K) and (x - K)^2 around the chunk's first value K
// (exact differences for fp32 input, no per-element division), converts the
// chunk to (count, mean, M2) and merges it into its running state with the
// reference's combine formula (Chan et al., moments.cpp:69-89).  States are
// then merged in a fixed order: row-lanes inside the CTA, CTAs in a second
// kernel, ranks on the host in rank order 0..p-1 from the identity -- the
// reference's allreduce(combine) fold (moments.cpp:45-47, transport.hpp:140-146).
#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.cuh"

namespace dndc {

constexpr int MO_THREADS = 256;
constexpr int MO_KC = 32;  // rows per shifted-sum chunk

struct Moment {
    double n, mean, m2;
};

// combine(a, b) of moments.cpp:69-89 for one slot (identity = n == 0).
__host__ __device__ inline Moment combine1(Moment a, Moment b) {
    if (a.n == 0.0) return b;
    if (b.n == 0.0) return a;
    Moment o;
    o.n = a.n + b.n;
    const double delta = b.mean - a.mean;
    o.mean = a.mean + delta * b.n / o.n;
    o.m2 = a.m2 + b.m2 + delta * delta * a.n * b.n / o.n;
    return o;
}

template <typename T>
__global__ void __launch_bounds__(MO_THREADS)
    moments_partial_kernel(const T* __restrict__ x, int64_t n, int m, int cols, int lanes,
                           int64_t rows_per_cta, double* __restrict__ partials) {
    // partials: [gridDim.x][3][m] as (n, mean, m2) per column
    __shared__ Moment sh[MO_THREADS];
    const int c_local = threadIdx.x % cols;
    const int rl = threadIdx.x / cols;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_cta;
    const int64_t r1 = min(n, r0 + rows_per_cta);
    for (int cb = 0; cb < m; cb += cols) {
        const int c = cb + c_local;
        Moment run{0.0, 0.0, 0.0};
        const bool active = rl < lanes && c < m;
        if (active) {
            int64_t i = r0 + rl;
            while (i < r1) {
                const double K = static_cast<double>(x[i * m + c]);
                double s1 = 0.0, s2 = 0.0;
                const int64_t left = (r1 - i + lanes - 1) / lanes;  // rows this thread still owns
                int cnt;
                if (left >= MO_KC) {
                    // full chunk: batches of 8 independent loads in flight per thread
#pragma unroll
                    for (int b = 0; b < MO_KC; b += 8) {
                        T v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) v[u] = x[(i + static_cast<int64_t>(b + u) * lanes) * m + c];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const double d = static_cast<double>(v[u]) - K;
                            s1 += d;
                            s2 = fma(d, d, s2);
                        }
                    }
                    cnt = MO_KC;
                } else {
                    cnt = static_cast<int>(left);
                    for (int u = 0; u < cnt; ++u) {
                        const double d = static_cast<double>(x[(i + static_cast<int64_t>(u) * lanes) * m + c]) - K;
                        s1 += d;
                        s2 = fma(d, d, s2);
                    }
                }
                i += static_cast<int64_t>(cnt) * lanes;
                const double nc = static_cast<double>(cnt);
                Moment ch;
                ch.n = nc;
                ch.mean = K + s1 / nc;
                ch.m2 = fmax(s2 - s1 * s1 / nc, 0.0);
                run = combine1(run, ch);
            }
        }
        sh[threadIdx.x] = run;
        __syncthreads();
        if (rl == 0 && c < m) {
            Moment acc = sh[c_local];
            for (int l = 1; l < lanes; ++l) acc = combine1(acc, sh[l * cols + c_local]);
            double* out = partials + static_cast<int64_t>(blockIdx.x) * 3 * m;
            out[c] = acc.n;
            out[m + c] = acc.mean;
            out[2 * m + c] = acc.m2;
        }
        __syncthreads();
    }
}

// fp32, 16-byte aligned: the shard is read as groups of rg = 4/gcd(m, 4)
// rows (rg*m floats, a whole number of float4s), each thread owning one
// float4 slot of a group -- 4 fixed (row-in-group, column) positions -- so a
// warp streams contiguous bytes with 8 groups of loads in flight per thread
// whatever m is (m = 18: 2-row groups of 9 float4s).  The same shifted-chunk
// sums and Chan merges per slot as above; a column's rg slots per row lane are
// merged in (lane, row-in-group) order.  n here counts groups; the n % rg
// leftover rows are folded in by moments_final_kernel.
#ifndef MO_V4_MIN_CTAS
#define MO_V4_MIN_CTAS 2
#endif
__global__ void __launch_bounds__(MO_THREADS, MO_V4_MIN_CTAS)
    moments_partial_v4_kernel(const float4* __restrict__ x4, int64_t n, int m, int rg, int lanes,
                              int64_t rows_per_cta, double* __restrict__ partials) {
    __shared__ Moment sh[MO_THREADS][4];
    const int m4 = rg * m / 4;
    const int c4 = threadIdx.x % m4, rl = threadIdx.x / m4;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_cta;
    const int64_t r1 = min(n, r0 + rows_per_cta);
    Moment run[4] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    if (rl < lanes) {
        int64_t i = r0 + rl;
        while (i < r1) {
            const float4 k4 = __ldg(x4 + i * m4 + c4);
            const double K[4] = {k4.x, k4.y, k4.z, k4.w};
            double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
            const int64_t left = (r1 - i + lanes - 1) / lanes;
            int cnt;
            if (left >= MO_KC) {
#pragma unroll
                for (int b = 0; b < MO_KC; b += 8) {
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldg(x4 + (i + static_cast<int64_t>(b + u) * lanes) * m4 + c4);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double d[4] = {static_cast<double>(v[u].x) - K[0], static_cast<double>(v[u].y) - K[1],
                                             static_cast<double>(v[u].z) - K[2], static_cast<double>(v[u].w) - K[3]};
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            s1[c] += d[c];
                            s2[c] = fma(d[c], d[c], s2[c]);
                        }
                    }
                }
                cnt = MO_KC;
            } else {
                cnt = static_cast<int>(left);
                for (int u = 0; u < cnt; ++u) {
                    const float4 v = __ldg(x4 + (i + static_cast<int64_t>(u) * lanes) * m4 + c4);
                    const double d[4] = {static_cast<double>(v.x) - K[0], static_cast<double>(v.y) - K[1],
                                         static_cast<double>(v.z) - K[2], static_cast<double>(v.w) - K[3]};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        s1[c] += d[c];
                        s2[c] = fma(d[c], d[c], s2[c]);
                    }
                }
            }
            i += static_cast<int64_t>(cnt) * lanes;
            const double nc = static_cast<double>(cnt);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                Moment ch;
                ch.n = nc;
                ch.mean = K[c] + s1[c] / nc;
                ch.m2 = fmax(s2[c] - s1[c] * s1[c] / nc, 0.0);
                run[c] = combine1(run[c], ch);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) sh[threadIdx.x][c] = run[c];
    __syncthreads();
    // column col sits at group offsets r*m + col, r < rg
    for (int col = threadIdx.x; col < m; col += MO_THREADS) {
        Moment acc{0.0, 0.0, 0.0};
        for (int l = 0; l < lanes; ++l)
            for (int r = 0; r < rg; ++r) {
                const int e = r * m + col;
                acc = combine1(acc, sh[l * m4 + e / 4][e % 4]);
            }
        double* out = partials + static_cast<int64_t>(blockIdx.x) * 3 * m;
        out[col] = acc.n;
        out[m + col] = acc.mean;
        out[2 * m + col] = acc.m2;
    }
}

// one CTA per column: the CTA partials merged in a fixed tree (thread t folds
// partials t, t+256, ... in order, then a pairwise tree over the threads),
// then the tail_rows rows at `tail` (rows the grouped kernel did not cover)
// one Welford step each
__global__ void __launch_bounds__(MO_THREADS)
    moments_final_kernel(const double* __restrict__ partials, int G, int m, const float* __restrict__ tail,
                         int tail_rows, double* __restrict__ out) {
    __shared__ Moment sh[MO_THREADS];
    const int c = blockIdx.x;
    Moment acc{0.0, 0.0, 0.0};
    for (int g = threadIdx.x; g < G; g += MO_THREADS) {
        const double* p = partials + static_cast<int64_t>(g) * 3 * m;
        acc = combine1(acc, Moment{p[c], p[m + c], p[2 * m + c]});
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int h = MO_THREADS / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) sh[threadIdx.x] = combine1(sh[threadIdx.x], sh[threadIdx.x + h]);
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    acc = sh[0];
    for (int t = 0; t < tail_rows; ++t)
        acc = combine1(acc, Moment{1.0, static_cast<double>(tail[static_cast<int64_t>(t) * m + c]), 0.0});
    out[c] = acc.n;
    out[m + c] = acc.mean;
    out[2 * m + c] = acc.m2;
}

template <typename T>
static void moments_axis0(dndc_ctx* ctx, const T* x, int64_t n_local, int64_t m64, int64_t* count_host,
                          double* mean_host, double* m2_host) {
    if (m64 < 0 || n_local < 0) value_error("moments: negative extent");
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    const size_t rec = 3 * static_cast<size_t>(std::max(m, 1));
    double* local = static_cast<double*>(ctx->slot("mo_local", sizeof(double) * rec));
    double* all = static_cast<double*>(ctx->slot("mo_all", sizeof(double) * rec * ctx->world));
    const int rg = m > 0 ? 4 / std::gcd(m, 4) : 1;  // rows per float4-aligned group
    const int64_t n_groups = n_local / rg;
    const bool v4 = sizeof(T) == 4 && m > 0 && rg * m / 4 <= MO_THREADS && n_groups > 0 &&
                    reinterpret_cast<uintptr_t>(x) % 16 == 0;
    if (v4) {
        const int m4 = rg * m / 4, lanes = MO_THREADS / m4;
        const int64_t min_groups = static_cast<int64_t>(lanes) * MO_KC * 4;
        // one full wave: resident CTAs per SM x SMs (a partial second wave
        // costs up to 2x at 5M x 18), fewer when the shard is small
        static int occ = 0;
        if (!occ) DNDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, moments_partial_v4_kernel, MO_THREADS, 0));
        const int64_t G = std::max<int64_t>(
            1, std::min<int64_t>(static_cast<int64_t>(ctx->num_sms) * std::max(occ, 1), ceil_div(n_groups, min_groups)));
        const int64_t groups_per_cta = ceil_div(n_groups, G);
        double* partials = static_cast<double*>(ctx->slot("mo_partials", sizeof(double) * rec * G));
        moments_partial_v4_kernel<<<static_cast<unsigned>(G), MO_THREADS, 0, s>>>(
            reinterpret_cast<const float4*>(x), n_groups, m, rg, lanes, groups_per_cta, partials);
        DNDC_LAUNCHED(ctx);
        const int tail_rows = static_cast<int>(n_local - n_groups * rg);
        const float* tail = reinterpret_cast<const float*>(x) + n_groups * rg * static_cast<int64_t>(m);
        moments_final_kernel<<<m, MO_THREADS, 0, s>>>(partials, static_cast<int>(G), m, tail, tail_rows,
                                                             local);
        DNDC_LAUNCHED(ctx);
    } else if (n_local > 0 && m > 0) {
        const int cols = std::min(m, MO_THREADS);
        const int lanes = MO_THREADS / cols;
        // enough CTAs to fill the GPU, each with at least a few chunks per lane
        const int64_t min_rows = static_cast<int64_t>(lanes) * MO_KC * 4;
        const int64_t G = std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 8, ceil_div(n_local, min_rows)));
        const int64_t rows_per_cta = ceil_div(n_local, G);
        double* partials = static_cast<double*>(ctx->slot("mo_partials", sizeof(double) * rec * G));
        moments_partial_kernel<T><<<static_cast<unsigned>(G), MO_THREADS, 0, s>>>(x, n_local, m, cols, lanes,
                                                                                rows_per_cta, partials);
        DNDC_LAUNCHED(ctx);
        moments_final_kernel<<<m, MO_THREADS, 0, s>>>(partials, static_cast<int>(G), m, nullptr, 0, local);
        DNDC_LAUNCHED(ctx);
    } else {
        DNDC_CUDA(cudaMemsetAsync(local, 0, sizeof(double) * rec, s));
    }
    allgather_f64(ctx, local, all, rec, s);
    double* h = static_cast<double*>(ctx->host_staging(sizeof(double) * rec * ctx->world));
    DNDC_CUDA(cudaMemcpyAsync(h, all, sizeof(double) * rec * ctx->world, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    // rank-order fold from the identity (moments.cpp:45-47), on every rank
    int64_t count = 0;
    std::vector<Moment> acc(std::max(m, 0), Moment{0.0, 0.0, 0.0});
    for (int r = 0; r < ctx->world; ++r) {
        const double* p = h + rec * r;
        const int64_t rc = m > 0 ? static_cast<int64_t>(p[0]) : 0;
        if (rc == 0) continue;  // combine(a, identity) == a exactly
        for (int c = 0; c < m; ++c) acc[c] = combine1(acc[c], Moment{p[c], p[m + c], p[2 * m + c]});
        count += rc;
    }
    *count_host = m > 0 ? count : 0;
    for (int c = 0; c < m; ++c) {
        mean_host[c] = acc[c].mean;
        m2_host[c] = acc[c].m2;
    }
}

}  // namespace dndc

extern "C" {

int dndc_moments_axis0_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, int64_t m,
                           int64_t* count_host, double* mean_host, double* m2_host) {
    return dndc::guard(
        [&] { dndc::moments_axis0<float>(ctx, x_local, n_local, m, count_host, mean_host, m2_host); });
}

int dndc_moments_axis0_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, int64_t m,
                           int64_t* count_host, double* mean_host, double* m2_host) {
    return dndc::guard(
        [&] { dndc::moments_axis0<double>(ctx, x_local, n_local, m, count_host, mean_host, m2_host); });
}

}  // extern "C"
