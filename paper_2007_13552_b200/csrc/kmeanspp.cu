// kmeanspp.cu -- A16: k-means++ (D^2) seeding for BASELINE config 5.
//
// NOT in the reference (SPEC.md:413 defers it); the definition is this repo's
// and is restated bit for bit by the test oracle (oracle/dnd_oracle.c):
//   - first pick: kmeans_init_indices(n, 1, seed)[0]  (cluster.cpp:60-75);
//   - D2[i] = min over picks of sum_f ((double)x - (double)c)^2, sequential
//     over f with the product rounded before the add;
//   - per rank shard, blocks of 2048 rows: lane l sums rows l, l+32, ...
//     sequentially, then a xor-butterfly over the 32 lanes -> S_b; groups of
//     1024 blocks the same way -> T_g; W = sequential sum over the global group
//     list (rank-major);
//   - draw j: u = uniform01(seed ^ KPP_SALT, j) (common.hpp:24-27), target
//     u*W, descend groups -> blocks -> rows with running sequential sums.
// Every step is one fused pass (update D2 against the newest pick + block sums)
// plus tiny group/select kernels; across ranks only the group sums (allgather)
// and the picked row (exact zero-filled allreduce) travel.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "tc.cuh"

namespace dndc {

constexpr int KPP_BLOCK = 2048;
constexpr int KPP_GROUP = 1024;
constexpr uint64_t KPP_SALT = 0x5851f42d4c957f2dULL;

template <typename T>
__device__ __forceinline__ double kpp_dist2(const T* __restrict__ xr, const T* c, int m) {
    double acc = 0.0;
    for (int f = 0; f < m; ++f) {
        const double dd = sub_rn(static_cast<double>(xr[f]), static_cast<double>(c[f]));
        acc = add_rn(acc, mul_rn(dd, dd));
    }
    return acc;
}

__device__ __forceinline__ double warp_butterfly(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// D2 of one row against the newest pick: sequential over features in f64,
// product rounded before the add (the oracle's order).  M > 0: compile-time
// width (all loads issued up front, float4 when aligned); M == 0: runtime.
// f64 input: the same chain on the doubles as they are.
template <int M, typename T>
__device__ __forceinline__ double kpp_row(const T* __restrict__ xr, const T* c, int m) {
    if constexpr (M > 0 && std::is_same_v<T, float>) {
        float v[M];
        if constexpr (M % 4 == 0) {
#pragma unroll
            for (int f = 0; f < M; f += 4) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(xr + f));
                v[f] = q.x;
                v[f + 1] = q.y;
                v[f + 2] = q.z;
                v[f + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int f = 0; f < M; ++f) v[f] = __ldg(xr + f);
        }
        double acc = 0.0;
#pragma unroll
        for (int f = 0; f < M; ++f) {
            const double dd = sub_rn(static_cast<double>(v[f]), static_cast<double>(c[f]));
            acc = add_rn(acc, mul_rn(dd, dd));
        }
        return acc;
    } else {
        return kpp_dist2(xr, c, m);
    }
}

// One warp per 2048-row block of the local shard; lane l owns rows l, l+32, ...
// (the summation order of the definition), two rows in flight per lane.
template <int M, typename T>
__global__ void kpp_update_kernel(const T* __restrict__ x, int64_t n, int m,
                                  const T* __restrict__ crow, double* __restrict__ d2, int first,
                                  double* __restrict__ S, int64_t nblocks) {
    extern __shared__ __align__(16) unsigned char kpp_sh[];
    T* c_sh = reinterpret_cast<T*>(kpp_sh);
    for (int f = threadIdx.x; f < m; f += blockDim.x) c_sh[f] = crow[f];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (b >= nblocks) return;
    const int64_t lo = b * KPP_BLOCK;
    const int64_t hi = min(n, lo + KPP_BLOCK);
    double acc = 0.0;
    for (int64_t i = lo + lane; i < hi; i += 64) {
        const int64_t i2 = i + 32;
        const double da = kpp_row<M, T>(x + i * m, c_sh, m);
        const double db = i2 < hi ? kpp_row<M, T>(x + i2 * m, c_sh, m) : 0.0;
        double va = da, vb = db;
        if (!first) {
            va = da < d2[i] ? da : d2[i];
            if (i2 < hi) vb = db < d2[i2] ? db : d2[i2];
        }
        d2[i] = va;
        acc = add_rn(acc, va);
        if (i2 < hi) {
            d2[i2] = vb;
            acc = add_rn(acc, vb);
        }
    }
    acc = warp_butterfly(acc);
    if (lane == 0) S[b] = acc;
}

// The same pass for 32-feature fp32 rows with the rows staged by TMA: the
// per-lane float4 loads of kpp_update_kernel (lane = row, 128-byte rows) cost
// 32 L1 wavefronts per warp instruction and bounded it near 4.2 TB/s.  Here
// each warp streams its blocks in 64-row chunks (2-D TMA box {32, 64},
// SWIZZLE_128B: chunk q of row r sits at q ^ (r & 7), so the lanes' 16-byte
// shared-memory reads are conflict-free) through a KPP_NS-stage ring of its
// own; lane l still takes rows l, l + 32 of every chunk, i.e. rows l, l + 32,
// l + 64, ... of the block in order -- the same D2 values and the same sums.
constexpr int KPP_WPB = 8, KPP_NS = 3, KPP_CH = 64;
constexpr int KPP_CHUNK_BYTES = KPP_CH * 128;
constexpr int KPP_TMA_SMEM = KPP_WPB * KPP_NS * KPP_CHUNK_BYTES + KPP_WPB * KPP_NS * 8 + 32 * 4 + 1024;

__global__ void __launch_bounds__(32 * KPP_WPB, 1)
    kpp_update_tma_kernel(const __grid_constant__ CUtensorMap map, int64_t n, const float* __restrict__ crow,
                          double* __restrict__ d2, int first, double* __restrict__ S, int64_t nblocks) {
    extern __shared__ unsigned char kpp_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(kpp_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = base + warp * KPP_NS * KPP_CHUNK_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + KPP_WPB * KPP_NS * KPP_CHUNK_BYTES) + warp * KPP_NS;
    float* c_sh = reinterpret_cast<float*>(base + KPP_WPB * KPP_NS * KPP_CHUNK_BYTES + KPP_WPB * KPP_NS * 8);
    if (threadIdx.x < 32) c_sh[threadIdx.x] = crow[threadIdx.x];
    if (lane == 0) {
        for (int st = 0; st < KPP_NS; ++st) tc::mbar_init(&bars[st], 1);
        tc::mbar_fence_init();
    }
    __syncthreads();
    float c[32];
#pragma unroll
    for (int f = 0; f < 32; ++f) c[f] = c_sh[f];

    const int64_t gw = static_cast<int64_t>(blockIdx.x) * KPP_WPB + warp, tw = static_cast<int64_t>(gridDim.x) * KPP_WPB;
    constexpr int CPB = KPP_BLOCK / KPP_CH;  // chunks per full block
    // sequence index q of this warp -> (block, chunk); valid while inside the shard
    auto item = [&](int64_t q, int64_t& b, int& ch) -> bool {
        b = gw + (q / CPB) * tw;
        ch = static_cast<int>(q % CPB);
        return b < nblocks && b * KPP_BLOCK + static_cast<int64_t>(ch) * KPP_CH < n;
    };
    auto issue = [&](int64_t q) {
        int64_t b;
        int ch;
        if (!item(q, b, ch)) return;
        const int st = static_cast<int>(q % KPP_NS);
        tc::fence_async_smem();
        tc::mbar_expect_tx(&bars[st], KPP_CHUNK_BYTES);
        tc::tma_load_2d(ring + st * KPP_CHUNK_BYTES, &map, &bars[st], 0,
                        static_cast<int>(b * KPP_BLOCK + static_cast<int64_t>(ch) * KPP_CH));
    };
    if (lane == 0)
        for (int64_t q = 0; q < KPP_NS; ++q) issue(q);
    double acc = 0.0;
    for (int64_t q = 0;; ++q) {
        int64_t b;
        int ch;
        if (!item(q, b, ch)) break;
        const int st = static_cast<int>(q % KPP_NS);
        tc::mbar_wait(&bars[st], static_cast<uint32_t>((q / KPP_NS) & 1));
        const unsigned char* buf = ring + st * KPP_CHUNK_BYTES;
        const int64_t lo = b * KPP_BLOCK, hi = min(n, lo + KPP_BLOCK);
        const int64_t r0 = lo + static_cast<int64_t>(ch) * KPP_CH;
        double va[2];
        bool ok[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            const int64_t i = r0 + r;
            ok[h] = i < hi;
            float v[32];
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) {
                const float4 t = *reinterpret_cast<const float4*>(buf + r * 128 + ((qq ^ (r & 7)) << 4));
                v[4 * qq] = t.x;
                v[4 * qq + 1] = t.y;
                v[4 * qq + 2] = t.z;
                v[4 * qq + 3] = t.w;
            }
            double dd2 = 0.0;
#pragma unroll
            for (int f = 0; f < 32; ++f) {
                const double dd = sub_rn(static_cast<double>(v[f]), static_cast<double>(c[f]));
                dd2 = add_rn(dd2, mul_rn(dd, dd));
            }
            va[h] = dd2;
        }
        __syncwarp();
        if (lane == 0) issue(q + KPP_NS);  // the stage is read: refill it
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t i = r0 + lane + 32 * h;
            if (ok[h]) {
                double v = va[h];
                if (!first) {
                    const double old = d2[i];
                    v = v < old ? v : old;
                }
                d2[i] = v;
                acc = add_rn(acc, v);
            }
        }
        // last chunk of the block: its sum
        if (ch == CPB - 1 || r0 + KPP_CH >= hi) {
            const double t = warp_butterfly(acc);
            if (lane == 0) S[b] = t;
            acc = 0.0;
        }
    }
}

// One warp per group of 1024 blocks.
__global__ void kpp_group_kernel(const double* __restrict__ S, int64_t nblocks, double* __restrict__ T,
                                 int64_t ngroups) {
    const int lane = threadIdx.x & 31;
    const int64_t g = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (g >= ngroups) return;
    const int64_t b0 = g * KPP_GROUP, b1 = min(nblocks, b0 + KPP_GROUP);
    double acc = 0.0;
    for (int64_t b = b0 + lane; b < b1; b += 32) acc = add_rn(acc, S[b]);
    acc = warp_butterfly(acc);
    if (lane == 0) T[g] = acc;
}

// sel: [0] owner rank, [1] local group, [2] residual target t1, [3] fallback
// global row (or -1)
__global__ void kpp_select_group_kernel(const double* __restrict__ Tall, int world, int64_t gmax,
                                        const int64_t* __restrict__ gcount, double u, int64_t n_global,
                                        double* __restrict__ sel) {
    if (threadIdx.x != 0) return;
    double W = 0.0;
    for (int r = 0; r < world; ++r)
        for (int64_t g = 0; g < gcount[r]; ++g) W = add_rn(W, Tall[r * gmax + g]);
    if (!(W > 0.0)) {
        int64_t pick = static_cast<int64_t>(u * static_cast<double>(n_global));
        if (pick >= n_global) pick = n_global - 1;
        sel[0] = -1.0;
        sel[3] = static_cast<double>(pick);
        return;
    }
    const double target = mul_rn(u, W);
    double P = 0.0, Plast = 0.0;
    int rs = -1, rlast = -1;
    int64_t gs = -1, glast = -1;
    for (int r = 0; r < world && rs < 0; ++r)
        for (int64_t g = 0; g < gcount[r]; ++g) {
            const double t = Tall[r * gmax + g];
            if (t > 0.0) {
                rlast = r;
                glast = g;
                Plast = P;
            }
            if (add_rn(P, t) > target) {
                rs = r;
                gs = g;
                break;
            }
            P = add_rn(P, t);
        }
    if (rs < 0) {
        rs = rlast;
        gs = glast;
        P = Plast;
    }
    sel[0] = static_cast<double>(rs);
    sel[1] = static_cast<double>(gs);
    sel[2] = sub_rn(target, P);
    sel[3] = -1.0;
}

// Owner rank: blocks of the chosen group, then rows of the chosen block.
// out: [0] global row index, [1..m] the row (zeros on non-owners).
template <typename T>
__global__ void kpp_select_row_kernel(const double* __restrict__ sel, int rank, const double* __restrict__ S,
                                      int64_t nblocks, const double* __restrict__ d2, int64_t n,
                                      int64_t row_off, const T* __restrict__ x, int m,
                                      double* __restrict__ out) {
    __shared__ int64_t pick_sh;
    if (threadIdx.x == 0) {
        int64_t pick = -1;
        if (sel[0] < 0.0) {
            const int64_t g = static_cast<int64_t>(sel[3]);
            if (g >= row_off && g < row_off + n) pick = g - row_off;
        } else if (static_cast<int>(sel[0]) == rank) {
            const int64_t g = static_cast<int64_t>(sel[1]);
            const double t1 = sel[2];
            const int64_t b0 = g * KPP_GROUP, b1 = min(nblocks, b0 + KPP_GROUP);
            double Q = 0.0, Qlast = 0.0;
            int64_t b = -1, blast = -1;
            for (int64_t bb = b0; bb < b1; ++bb) {
                if (S[bb] > 0.0) {
                    blast = bb;
                    Qlast = Q;
                }
                if (add_rn(Q, S[bb]) > t1) {
                    b = bb;
                    break;
                }
                Q = add_rn(Q, S[bb]);
            }
            if (b < 0) {
                b = blast;
                Q = Qlast;
            }
            const double t2 = sub_rn(t1, Q);
            double R = 0.0;
            int64_t row = -1, rl = -1;
            const int64_t r1 = min(n, (b + 1) * KPP_BLOCK);
            for (int64_t i = b * KPP_BLOCK; i < r1; ++i) {
                const double v = d2[i];
                if (v > 0.0) rl = i;
                if (add_rn(R, v) > t2) {
                    row = i;
                    break;
                }
                R = add_rn(R, v);
            }
            pick = row >= 0 ? row : rl;
        }
        pick_sh = pick;
        out[0] = pick >= 0 ? static_cast<double>(row_off + pick) : 0.0;
    }
    __syncthreads();
    const int64_t pick = pick_sh;
    for (int f = threadIdx.x; f < m; f += blockDim.x)
        out[1 + f] = pick >= 0 ? static_cast<double>(x[pick * m + f]) : 0.0;
}

template <typename T>
__global__ void kpp_unpack_kernel(const double* __restrict__ in, int m, T* __restrict__ crow,
                                  int64_t* __restrict__ idx_out, int j) {
    for (int f = threadIdx.x; f < m; f += blockDim.x) crow[f] = static_cast<T>(in[1 + f]);
    if (threadIdx.x == 0) idx_out[j] = static_cast<int64_t>(in[0]);
}

template <typename T>
__global__ void kpp_first_row_kernel(const T* __restrict__ x, int64_t lo, int64_t hi, int m,
                                     int64_t g, double* __restrict__ out) {
    for (int f = threadIdx.x; f < m; f += blockDim.x)
        out[1 + f] = (g >= lo && g < hi) ? static_cast<double>(x[(g - lo) * m + f]) : 0.0;
    if (threadIdx.x == 0) out[0] = (g >= lo && g < hi) ? static_cast<double>(g) : 0.0;
}

template <typename E>
static void kmeanspp(dndc_ctx* ctx, const E* x, int64_t n_local, int64_t n_global, int64_t m64, int k,
                     uint64_t seed, int64_t* idx_host) {
    if (k < 1 || static_cast<int64_t>(k) > n_global)
        value_error("kmeanspp: k=" + std::to_string(k) + " out of range for n=" + std::to_string(n_global));
    std::vector<int64_t> off, ext;
    chunk_map(n_global, ctx->world, off, ext);
    if (n_local != ext[ctx->rank]) value_error("kmeanspp: shard does not match chunk_map");
    const int m = static_cast<int>(m64);
    cudaStream_t s = ctx->stream;
    const int p = ctx->world;
    std::vector<int64_t> gcount(p);
    int64_t gmax = 1;
    for (int r = 0; r < p; ++r) {
        gcount[r] = ceil_div(ceil_div(ext[r], KPP_BLOCK), KPP_GROUP);
        gmax = std::max(gmax, gcount[r]);
    }
    const int64_t nblocks = ceil_div(n_local, KPP_BLOCK);
    const int64_t ngroups = gcount[ctx->rank];
    double* d2 = static_cast<double*>(ctx->slot("kpp_d2", sizeof(double) * std::max<int64_t>(n_local, 1)));
    double* S = static_cast<double*>(ctx->slot("kpp_S", sizeof(double) * std::max<int64_t>(nblocks, 1)));
    double* T = static_cast<double*>(ctx->slot("kpp_T", sizeof(double) * gmax));
    double* Tall = static_cast<double*>(ctx->slot("kpp_Tall", sizeof(double) * gmax * p));
    int64_t* gc = static_cast<int64_t*>(ctx->slot("kpp_gc", sizeof(int64_t) * p));
    double* sel = static_cast<double*>(ctx->slot("kpp_sel", sizeof(double) * 4));
    double* pk = static_cast<double*>(ctx->slot("kpp_pick", sizeof(double) * (m + 1)));
    E* crow = static_cast<E*>(ctx->slot("kpp_crow", sizeof(double) * std::max(m, 1)));
    int64_t* didx = static_cast<int64_t*>(ctx->slot("kpp_idx", sizeof(int64_t) * k));

    int64_t* hgc = static_cast<int64_t*>(ctx->host_staging(sizeof(int64_t) * p));
    std::memcpy(hgc, gcount.data(), sizeof(int64_t) * p);
    DNDC_CUDA(cudaMemcpyAsync(gc, hgc, sizeof(int64_t) * p, cudaMemcpyHostToDevice, s));
    DNDC_CUDA(cudaMemsetAsync(T, 0, sizeof(double) * gmax, s));

    // first pick: kmeans_init_indices(n, 1, seed)[0]
    int64_t first = 0;
    {
        const uint64_t draw = splitmix64(seed ^ splitmix64(0x6b8b4567u));
        first = static_cast<int64_t>(draw % static_cast<uint64_t>(n_global));
    }
    kpp_first_row_kernel<E><<<1, 128, 0, s>>>(x, off[ctx->rank], off[ctx->rank] + n_local, m, first, pk);
    DNDC_LAUNCHED(ctx);
    allreduce_sum_f64(ctx, pk, m + 1, s);
    kpp_unpack_kernel<E><<<1, 128, 0, s>>>(pk, m, crow, didx, 0);
    DNDC_LAUNCHED(ctx);
    DNDC_CUDA(cudaStreamSynchronize(s));  // hgc staging reuse below

    const int wpb = 8;
    // fp32 rows of 32 features, 16-byte aligned: the TMA-staged pass
    const bool tma = std::is_same_v<E, float> && m == 32 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                     n_local > 0 && !std::getenv("DNDC_KPP_NO_TMA");
    CUtensorMap kmap{};
    int tgrid = 0;
    if (tma) {
        kmap = make_tmap_2d_f32(x, static_cast<uint64_t>(n_local), 32, 128, 32, KPP_CH, true);
        DNDC_CUDA(cudaFuncSetAttribute(kpp_update_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       KPP_TMA_SMEM));
        tgrid = static_cast<int>(std::min<int64_t>(ceil_div(nblocks, static_cast<int64_t>(KPP_WPB)), ctx->num_sms));
    }
    for (int j = 1; j < k; ++j) {
        if (nblocks > 0) {
            const unsigned g = static_cast<unsigned>(ceil_div(nblocks, wpb));
            const size_t sm = sizeof(E) * m;
            const bool a16 = reinterpret_cast<uintptr_t>(x) % 16 == 0;
            if (tma) {
                kpp_update_tma_kernel<<<tgrid, 32 * KPP_WPB, KPP_TMA_SMEM, s>>>(
                    kmap, n_local, reinterpret_cast<const float*>(crow), d2, j == 1, S, nblocks);
            } else if constexpr (std::is_same_v<E, float>) {
                if (m == 32 && a16) kpp_update_kernel<32, E><<<g, 32 * wpb, sm, s>>>(x, n_local, m, crow, d2, j == 1, S, nblocks);
                else if (m == 64 && a16) kpp_update_kernel<64, E><<<g, 32 * wpb, sm, s>>>(x, n_local, m, crow, d2, j == 1, S, nblocks);
                else if (m == 16 && a16) kpp_update_kernel<16, E><<<g, 32 * wpb, sm, s>>>(x, n_local, m, crow, d2, j == 1, S, nblocks);
                else if (m == 18) kpp_update_kernel<18, E><<<g, 32 * wpb, sm, s>>>(x, n_local, m, crow, d2, j == 1, S, nblocks);
                else kpp_update_kernel<0, E><<<g, 32 * wpb, sm, s>>>(x, n_local, m, crow, d2, j == 1, S, nblocks);
            } else {
                kpp_update_kernel<0, E><<<g, 32 * wpb, sm, s>>>(x, n_local, m, crow, d2, j == 1, S, nblocks);
            }
            DNDC_LAUNCHED(ctx);
            kpp_group_kernel<<<static_cast<unsigned>(ceil_div(ngroups, wpb)), 32 * wpb, 0, s>>>(S, nblocks, T,
                                                                                               ngroups);
            DNDC_LAUNCHED(ctx);
        }
        allgather_f64(ctx, T, Tall, gmax, s);
        const double u = uniform01(seed ^ KPP_SALT, static_cast<uint64_t>(j));
        kpp_select_group_kernel<<<1, 32, 0, s>>>(Tall, p, gmax, gc, u, n_global, sel);
        DNDC_LAUNCHED(ctx);
        kpp_select_row_kernel<E><<<1, 128, 0, s>>>(sel, ctx->rank, S, nblocks, d2, n_local, off[ctx->rank], x, m,
                                                   pk);
        DNDC_LAUNCHED(ctx);
        allreduce_sum_f64(ctx, pk, m + 1, s);
        kpp_unpack_kernel<E><<<1, 128, 0, s>>>(pk, m, crow, didx, j);
        DNDC_LAUNCHED(ctx);
    }
    int64_t* h = static_cast<int64_t*>(ctx->host_staging(sizeof(int64_t) * k));
    DNDC_CUDA(cudaMemcpyAsync(h, didx, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(idx_host, h, sizeof(int64_t) * k);
}

}  // namespace dndc

extern "C" int dndc_kmeanspp_indices_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local,
                                         int64_t n_global, int64_t m, int k, uint64_t seed,
                                         int64_t* indices_host) {
    return dndc::guard([&] { dndc::kmeanspp<float>(ctx, x_local, n_local, n_global, m, k, seed, indices_host); });
}

extern "C" int dndc_kmeanspp_indices_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local,
                                         int64_t n_global, int64_t m, int k, uint64_t seed,
                                         int64_t* indices_host) {
    return dndc::guard([&] { dndc::kmeanspp<double>(ctx, x_local, n_local, n_global, m, k, seed, indices_host); });
}
