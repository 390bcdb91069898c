// kmeans_tc.cuh -- tcgen05 assign/accumulate kernel (included by kmeans.cu
// inside namespace dndc; needs ref_argmin_cand, FULL and ceil_div from there).
//
// The K*D score FMAs per row run on the 5th-gen tensor cores:
//   * X is streamed by TMA 2-D tile loads as P rows per MMA row ("packed
//     rows": X viewed as [n/P x P*D]; D = 18 rows pair up into 36 columns with
//     a 144-byte pitch), box {32 columns, 128 packed rows} with SWIZZLE_128B:
//     each K-block of 32 columns is one [128 rows x 128 B] swizzle-atom stack
//     (the K-major SW128 layout of cdist_tc.cu), so a tile is ceil(KC/32)
//     boxes of 128-byte row segments (the earlier 4-column SWIZZLE_NONE boxes
//     cost 16 TMA requests of 16 B per row and bounded the kernel at ~0.6 TB/s).
//     2-3 stage ring, one producer thread.
//   * scores[packed row][h*K + j] = x_h . (-2 c_j) with a block-diagonal
//     centroid operand (N = P*K), 3xTF32: the tensor core truncates fp32
//     inputs to tf32 (pinned by tests/test_gpu_tc.py), so hi = the raw TMA
//     tile and the epilogue only writes lo = x - trunc(x);
//     hi.Bhi + hi.Blo + lo.Bhi accumulate in TMEM (fp32).
//   * Two epilogue warpgroups take alternating tiles (thread = packed row =
//     TMEM lane), so one warpgroup's CUDA-core work overlaps the other's MMA.
//     Per tile: split, score readback (tcgen05.ld), top-2 against a rigorous
//     per-row error bound, exact f64 re-decision over the candidate clusters
//     only, then the counting sort by label into the (now free) lo buffer and
//     warp-per-cluster f64 run sums -- as kmeans_small_kernel.
//   * tf32 MN-major operands are not supported (zeros; tests/test_gpu_tc.py),
//     so the one-hot accumulation stays on the CUDA cores.

struct TcParams {
    int64_t n;            // rows (a multiple of P)
    const double* c64;
    const double* cn64;
    const float* ctab;    // [K*D] -2 c (fp32), [K] |c|^2 (fp32)
    const float* bounds;  // [0] max |c_j|, [1] max |c_j|^2
    double* partials;     // null: predict only
    int32_t* labels;
    unsigned long long* refined;
    const int* done;
    const int8_t* prev;   // delta iterations: last iteration's labels (null: full accumulation)
    int8_t* lab8;         // this iteration's labels (fit only; null in predict)
    const double* xabs;   // max |x| of the shard: the int64 fixed-point scale of the sums
    // near-tie queue (null: refine inline): rows whose fp32 top-2 gap is inside
    // the error bound go to kmeans_tc_refine_kernel with their candidate mask
    unsigned* rq_ctl;             // [0] entries, [1] refine-kernel ticket
    uint64_t* rq_row;             // row | (uint8)(decided label + 1) << 48 | (uint8)last label << 56
    unsigned long long* rq_cand;  // candidate clusters
    float* rq_x;                  // the row itself (D floats; null: the refine kernel reads X)
    unsigned rq_cap;
    const float* x;               // X (kmeans_tcd_kernel's queue-overflow fallback)
};

// an unused queue slot
constexpr uint64_t TC_QHOLE = ~0ull;

// label of a row handed to the refine kernel (not written, not accumulated here)
template <int K>
constexpr int tc_deferred() { return K + 1; }

// The exact decision for one near-tie row, by one warp (result warp-uniform):
// `row` (D floats, shared memory) against the candidate clusters `cm`.
// (1) fast filter: f64 distances with the lanes over the features (any
// summation order).  Its error and the reference's are both <= (D+2)*2^-53*S,
// S = |x|^2 + max|c|^2 + 2|x|max|c|, so a winner whose margin over the
// runner-up (and over the clamp at 0) exceeds 2^-40*S is the reference's
// choice, sqrt rounding included.  (2) otherwise the reference's own operation
// order (cluster.cpp:44-56 via ref_distance), lanes over the candidates, with
// its lowest-index tie rule.
template <int D, int K>
__device__ __forceinline__ int tc_refine_warp(const float* row, uint64_t cm, const double* __restrict__ c64,
                                              const double* __restrict__ cn64, float cnmax, float cmax,
                                              unsigned long long* fallback_ctr) {
    const int lane = threadIdx.x & 31;
    constexpr int FL = (D + 31) / 32;
    double xf[FL];
    double xn = 0.0;
#pragma unroll
    for (int u = 0; u < FL; ++u) {
        const int f = lane + 32 * u;
        xf[u] = f < D ? static_cast<double>(row[f]) : 0.0;
        xn = fma(xf[u], xf[u], xn);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xn += __shfl_xor_sync(FULL, xn, o);
    double d1 = DBL_MAX, d2 = DBL_MAX;
    int best = K;
    for (uint64_t rest = cm; rest;) {
        int js[4];
        double gp[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            js[q] = rest ? __ffsll(static_cast<long long>(rest)) - 1 : -1;
            rest &= rest - 1;
            gp[q] = 0.0;
            const double* cq = c64 + static_cast<int64_t>(js[q] < 0 ? 0 : js[q]) * D;
#pragma unroll
            for (int u = 0; u < FL; ++u) {
                const int f = lane + 32 * u;
                if (f < D) gp[q] = fma(xf[u], __ldg(cq + f), gp[q]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int q = 0; q < 4; ++q) gp[q] += __shfl_xor_sync(FULL, gp[q], o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (js[q] < 0) continue;
            const double dq = xn + cn64[js[q]] - 2.0 * gp[q];
            if (dq < d1) {
                d2 = d1;
                d1 = dq;
                best = js[q];
            } else if (dq < d2) {
                d2 = dq;
            }
        }
    }
    const double margin =
        0x1.0p-40 * (xn + static_cast<double>(cnmax) + 2.0 * sqrt(xn) * static_cast<double>(cmax));
    const bool decided = d1 > margin && d2 - d1 > margin;
    if (decided) return best;
    if (fallback_ctr && lane == 0) atomicAdd(fallback_ctr, 1ull);
    double bd = 0.0;
    best = K;
    for (uint64_t rest = cm; rest;) {  // rounds of up to 32 candidates, ascending j
        uint64_t mm = rest;
        for (int i = 0; i < lane && mm; ++i) mm &= mm - 1;
        const int j = mm ? __ffsll(static_cast<long long>(mm)) - 1 : -1;
        for (int i = 0; i < 32 && rest; ++i) rest &= rest - 1;
        const double* c = c64 + static_cast<int64_t>(j < 0 ? 0 : j) * D;
        double xs = 0.0, g = 0.0;
        // batches of 16 features: the centroid loads are issued ahead of the
        // two serial f64 chains (one L1 round trip per batch, not per step)
        constexpr int FB = D % 16 == 0 ? 16 : D % 8 == 0 ? 8 : 2;
#pragma unroll
        for (int f0 = 0; f0 < D; f0 += FB) {
            double2 cb[FB / 2];
#pragma unroll
            for (int u = 0; u < FB / 2; ++u) cb[u] = __ldg(reinterpret_cast<const double2*>(c + f0) + u);
#pragma unroll
            for (int u = 0; u < FB; ++u) {
                const double xv = static_cast<double>(row[f0 + u]);
                xs = add_rn(xs, mul_rn(xv, xv));
                g = add_rn(g, mul_rn(xv, u % 2 ? cb[u / 2].y : cb[u / 2].x));
            }
        }
        double dj = j < 0 ? 0.0 : ref_distance(xs, cn64[j], g);
        int jj = j < 0 ? K : j;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(FULL, dj, o);
            const int oj = __shfl_xor_sync(FULL, jj, o);
            if (oj < K && (jj == K || od < dj || (od == dj && oj < jj))) {
                dj = od;
                jj = oj;
            }
        }
        if (jj < K && (best == K || dj < bd)) {  // later rounds hold larger j: strict <
            bd = dj;
            best = jj;
        }
    }
    return best;
}

__host__ __device__ constexpr int tc_pow2_cols(int c) {
    return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int D, int K, int P, int WG_ = 2>
struct TcCfg {
    static constexpr int KC = ((P * D + 7) / 8) * 8;  // MMA K (tf32 steps of 8)
    static constexpr int NCH = KC / 4;                // 16-byte column chunks
    static constexpr int NKB = (KC + 31) / 32;        // 128-byte K-blocks (TMA boxes) per tile
    static constexpr int NS = P * K;                  // MMA N: score slots
    static constexpr int PR = 128;                    // packed rows per tile (MMA M)
    static constexpr int TROWS = PR * P;              // data rows per tile
    static constexpr int S = 3;                       // TMA stages
    static constexpr int WGS = WG_;                   // epilogue warpgroups
    static constexpr int EPI = 128 * WGS;
    static constexpr int THREADS = EPI + 32;          // + the producer / MMA warp
    static constexpr int TILE_BYTES = NKB * PR * 128;
    static constexpr int SORT_BYTES = TROWS * D * 4;
    static constexpr int WORK_BYTES = TILE_BYTES > SORT_BYTES ? TILE_BYTES : SORT_BYTES;  // lo, then sorted rows
    static constexpr int B_BYTES = NCH * NS * 16;
    static constexpr int VW = 4 * P;                  // 32-row groups per tile
    static constexpr int TMEM_COLS = tc_pow2_cols(WGS * NS);
    static constexpr int OFF_TILE = 0;
    static constexpr int OFF_WORK = OFF_TILE + S * TILE_BYTES;
    static constexpr int OFF_BHI = OFF_WORK + WGS * WORK_BYTES;
    static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
    static constexpr int OFF_CN = OFF_BLO + B_BYTES;
    static constexpr int OFF_CNT = OFF_CN + ((K * 4 + 15) / 16) * 16;  // u16 tile counts per warpgroup
    static constexpr int OFF_BAR = OFF_CNT + WGS * ((VW * K * 2 + 15) / 16) * 16;
    static constexpr int NBARS = 2 * S + 3 * WGS;
    static constexpr int OFF_TMEM = OFF_BAR + NBARS * 8;
    static constexpr int SMEM = OFF_TMEM + 16;
    static_assert(NS % 16 == 0 && NS <= 256, "MMA N (P*K) must be a multiple of 16, <= 256");
    static_assert(D % 2 == 0 && D <= 64 && K <= 64, "tc kernel shape");
    static_assert(OFF_TMEM + 16 <= 232448, "shared memory");
    static_assert(TILE_BYTES % 1024 == 0 && WORK_BYTES % 1024 == 0, "SW128 tiles need 1024-byte alignment");
    // delta iterations: each warp moves its own changed rows (int8 labels)
    static constexpr bool DELTA_OK = P == 1 && K <= 127;
};

template <int D, int K, int P, int WG_>
__global__ void __launch_bounds__(TcCfg<D, K, P, WG_>::THREADS, 1)
    kmeans_tc_kernel(const __grid_constant__ CUtensorMap map, TcParams p) {
    using C = TcCfg<D, K, P, WG_>;
    constexpr int NCH = C::NCH, NS = C::NS, PR = C::PR, S = C::S, KD = K * D, VW = C::VW, WGS = C::WGS;
    constexpr int L = D / 2;                // phase-2 lanes per row (float2 each)
    constexpr int G = 32 / L;               // rows summed in parallel per warp
    constexpr int JW = (K + 3) / 4;         // clusters owned per epilogue warp
    constexpr int KL = (K + 31) / 32;       // clusters per lane in the scans
#ifndef KT_NU
#define KT_NU 4
#endif
    constexpr int NU = KT_NU;               // cluster runs summed together per warp
    if (p.done && *p.done) return;

    extern __shared__ __align__(1024) unsigned char smem[];
    if (tc::smem_u32(smem) & 1023u) __trap();  // SW128 atoms: the dynamic window must start 1024-aligned
    float* tiles = reinterpret_cast<float*>(smem + C::OFF_TILE);
    float* bhi = reinterpret_cast<float*>(smem + C::OFF_BHI);
    float* blo = reinterpret_cast<float*>(smem + C::OFF_BLO);
    float* cn = reinterpret_cast<float*>(smem + C::OFF_CN);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* full = bars;              // [S] TMA landed
    uint64_t* empty = bars + S;         // [S] stage free
    uint64_t* loready = bars + 2 * S;   // [WGS] lo split written
    uint64_t* dfull = loready + WGS;    // [WGS] scores ready
    uint64_t* dempty = dfull + WGS;     // [WGS] scores read
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool accumulate = p.partials != nullptr;
    constexpr int CTRL = C::EPI / 32;  // control warp index

    if (warp == CTRL) {
        tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            for (int w = 0; w < WGS; ++w) {
                tc::mbar_init(&loready[w], 1);
                tc::mbar_init(&dfull[w], 1);
                tc::mbar_init(&dempty[w], 128);
            }
            tc::mbar_fence_init();
            tc::tma_prefetch_desc(&map);
        }
    } else {
        // block-diagonal centroid operand, split into tf32 hi / lo, K-major chunks
        for (int e = tid; e < NS * C::KC; e += C::EPI) {
            const int n = e / C::KC, c = e % C::KC;
            const int h = n / K, j = n % K;
            const int f = c - h * D;
            const float v = (f >= 0 && f < D) ? p.ctab[j * D + f] : 0.f;
            const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            const int off = (c / 4) * (NS * 4) + n * 4 + (c % 4);
            bhi[off] = hi;
            blo[off] = v - hi;
        }
        for (int j = tid; j < K; j += C::EPI) cn[j] = p.ctab[KD + j];
        tc::fence_async_smem();
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int64_t npacked = p.n / P;
    const int64_t ntiles = ceil_div(npacked, PR);
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == CTRL) {
        // ------------------------------------------------ TMA + MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(128, NS, 0, 0);
            int64_t issued = 0;
            for (int64_t it = 0; it < my_tiles; ++it) {
                while (issued < my_tiles && issued < it + S) {
                    const int st = static_cast<int>(issued % S);
                    if (issued >= S) tc::mbar_wait(&empty[st], static_cast<uint32_t>((issued / S - 1) & 1));
                    const int prow = static_cast<int>((blockIdx.x + issued * gridDim.x) * PR);
                    tc::mbar_expect_tx(&full[st], C::TILE_BYTES);
                    float* dst = tiles + st * (C::TILE_BYTES / 4);
#pragma unroll
    #ifndef DNDC_TC_NO_EVICT_FIRST  // X tiles leave L2 first (cfg3 shard: 0.532 -> 0.518 ms per iteration)
                for (int kb = 0; kb < C::NKB; ++kb)
                    tc::tma_load_2d_hint(dst + kb * PR * 32, &map, &full[st], kb * 32, prow, tc::l2_policy_evict_first());
#else
                for (int kb = 0; kb < C::NKB; ++kb) tc::tma_load_2d(dst + kb * PR * 32, &map, &full[st], kb * 32, prow);
#endif
                    ++issued;
                }
                const int st = static_cast<int>(it % S), w = static_cast<int>(it % WGS);
                const int64_t use = it / WGS;  // this warpgroup's use index
                // the two MMAs on the raw tile (hi.Bhi + hi.Blo) go out as soon as
                // the tile has landed and the accumulator is free; only lo.Bhi
                // waits for the warpgroup's split, so the warpgroup then waits for
                // one third of the MMAs instead of all of them
                if (use >= 1) tc::mbar_wait(&dempty[w], static_cast<uint32_t>((use - 1) & 1));
                tc::mbar_wait(&full[st], static_cast<uint32_t>((it / S) & 1));
                tc::tc_fence_after();
                const uint32_t a0 = tc::smem_u32(tiles + st * (C::TILE_BYTES / 4));
                const uint32_t l0 = tc::smem_u32(smem + C::OFF_WORK + w * C::WORK_BYTES);
                const uint32_t bh0 = tc::smem_u32(bhi), bl0 = tc::smem_u32(blo);
                const uint32_t dt = tmem + w * NS;
#pragma unroll
                for (int ks = 0; ks < C::KC / 8; ++ks) {
                    const uint32_t ko = (ks / 4) * PR * 128 + (ks % 4) * 32;  // K-block, then bytes inside the atom
                    const uint64_t ahi = tc::smem_desc(a0 + ko, 16, 1024, 2);
                    const uint64_t bh = tc::smem_desc(bh0 + ks * 2 * NS * 16, NS * 16, 128);
                    const uint64_t bl = tc::smem_desc(bl0 + ks * 2 * NS * 16, NS * 16, 128);
                    tc::mma_tf32(dt, ahi, bh, idesc, ks > 0);
#ifndef KT_EXP_ONEMMA
                    tc::mma_tf32(dt, ahi, bl, idesc, 1);
#endif
                }
                tc::mbar_wait(&loready[w], static_cast<uint32_t>(use & 1));
                tc::tc_fence_after();
#ifndef KT_EXP_ONEMMA
#pragma unroll
                for (int ks = 0; ks < C::KC / 8; ++ks) {
                    const uint32_t ko = (ks / 4) * PR * 128 + (ks % 4) * 32;
                    const uint64_t alo = tc::smem_desc(l0 + ko, 16, 1024, 2);
                    const uint64_t bh = tc::smem_desc(bh0 + ks * 2 * NS * 16, NS * 16, 128);
                    tc::mma_tf32(dt, alo, bh, idesc, 1);
                }
#endif
                tc::mma_commit(&dfull[w]);
                // the stage is free once its MMAs retire (the split already read
                // it): released here rather than after the epilogue's readback
                // and near-tie work, so TMA runs ahead of a slow tile
                tc::mma_commit(&empty[st]);
            }
        }
    } else {
        // ------------------------------------------------ epilogue warpgroups
        const int wg = warp / 4, wq = warp % 4, t = tid % 128;  // t = packed row = TMEM lane
        float* work = reinterpret_cast<float*>(smem + C::OFF_WORK + wg * C::WORK_BYTES);
        unsigned short* cnt = reinterpret_cast<unsigned short*>(smem + C::OFF_CNT + wg * ((VW * K * 2 + 15) / 16) * 16);
        const uint32_t bar_id = 1 + wg;
        const float cmax = p.bounds[0], cnmax = p.bounds[1];
        constexpr float ERR = 4.f * (static_cast<float>(3 * C::KC) * 0x1.0p-24f + 3.f * 0x1.0p-20f);
        unsigned long long refined = 0;
        // this warp's reserved run of queue slots (warp-uniform): slots are taken
        // from the global counter QCHUNK at a time, so the ~1 us atomic round
        // trip is paid once per run instead of once per tile; a run's unused
        // slots are marked as holes (TC_QHOLE) for the refine kernel
        constexpr unsigned QCHUNK = 64;
        unsigned qbase = 0, qleft = 0;
        auto qholes = [&]() {
            for (unsigned i = lane; i < qleft; i += 32)
                if (qbase + i < p.rq_cap) p.rq_row[qbase + i] = TC_QHOLE;
        };
        const int g = lane / L, q = lane % L;
        // cluster sums: int64 fixed point at 2^-(61-e), n max|x| < 2^e, in the
        // CTA's own partial row (global, L2-resident; converted to f64 in place
        // at the end), shared by the warpgroups.  Integer adds commute, and
        // global reductions are fire-and-forget RED at L2 -- shared memory has
        // no native 64-bit add (a CAS loop that stalled the warp).
        long long* acc = accumulate ? reinterpret_cast<long long*>(p.partials + static_cast<int64_t>(blockIdx.x) * (KD + K))
                                    : nullptr;
        if (accumulate)
            for (int e = tid; e < KD + K; e += C::EPI) acc[e] = 0ll;
        __threadfence();
        int e2 = 0;
        frexp(static_cast<double>(p.n) * (p.xabs ? *p.xabs : 1.0) + 1.0, &e2);
        const int shift = 61 - e2;
        const float qscale = ldexpf(1.f, shift);
        tc::named_sync(15, C::EPI);  // zeroed before any warpgroup adds

        for (int64_t it = wg; it < my_tiles; it += WGS) {
            const int st = static_cast<int>(it % S);
            const int64_t use = it / WGS;
            const int64_t prow0 = (blockIdx.x + it * gridDim.x) * PR;
            const float* xt = tiles + st * (C::TILE_BYTES / 4);
            // last iteration's labels, loaded now: the global round trip overlaps
            // the split and the MMAs instead of holding up the accumulator release
            int oldl[P];
#pragma unroll
            for (int h = 0; h < P; ++h) {
                const int64_t row = (prow0 + t) * P + h;
                oldl[h] = (p.prev && row < p.n) ? static_cast<int>(p.prev[row]) : -1;
            }
            tc::mbar_wait(&full[st], static_cast<uint32_t>((it / S) & 1));

            // split: lo = x - trunc_tf32(x); the raw row stays in registers; the
            // row's |x|^2 (error bound) in four independent fp32 chains
            float4 xr[NCH];
            float4 xq = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                // 16-byte chunk c of row t: K-block c/8, chunk (c%8) ^ (t%8) of the row's 128-byte line
                const int off = (c / 8) * PR * 32 + t * 32 + (((c % 8) ^ (t & 7)) * 4);
                const float4 v = *reinterpret_cast<const float4*>(xt + off);
                xr[c] = v;
                float4 l;
                l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                *reinterpret_cast<float4*>(work + off) = l;
                xq.x = fmaf(v.x, v.x, xq.x);
                xq.y = fmaf(v.y, v.y, xq.y);
                xq.z = fmaf(v.z, v.z, xq.z);
                xq.w = fmaf(v.w, v.w, xq.w);
            }
            tc::fence_async_smem();
            tc::named_sync(bar_id, 128);
            if (t == 0) tc::mbar_arrive(&loready[wg]);

            auto xval = [&](int c) {
                const float4 v4 = xr[c / 4];
                return (c % 4 == 0) ? v4.x : (c % 4 == 1) ? v4.y : (c % 4 == 2) ? v4.z : v4.w;
            };
            // hands the rows of this warp with `want` to the refine kernel's
            // queue (row, last label, the decided label or none, candidates, the
            // row itself); false for the lanes whose row did not fit
            auto enqueue = [&](int h, bool want, uint64_t cm, int newl) -> bool {
                const unsigned fm = __ballot_sync(FULL, want);
                if (!p.rq_ctl || !fm) return false;
                const unsigned cnt = static_cast<unsigned>(__popc(fm));
                if (cnt > qleft) {
                    qholes();
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(p.rq_ctl, QCHUNK);
                    qbase = __shfl_sync(FULL, base, 0);
                    qleft = QCHUNK;
                }
                const unsigned pos = qbase + static_cast<unsigned>(__popc(fm & ((1u << lane) - 1u)));
                qbase += cnt;
                qleft -= cnt;
                if (!want || pos >= p.rq_cap) return false;
                p.rq_row[pos] = static_cast<uint64_t>((prow0 + t) * P + h) |
                                (static_cast<uint64_t>(static_cast<uint8_t>(oldl[h])) << 56) |
                                (static_cast<uint64_t>(static_cast<uint8_t>(newl + 1)) << 48);
                p.rq_cand[pos] = cm;
                float* qx = p.rq_x + static_cast<int64_t>(pos) * D;
                if constexpr (P == 1 && D % 4 == 0) {
#pragma unroll
                    for (int c = 0; c < D / 4; ++c) reinterpret_cast<float4*>(qx)[c] = xr[c];
                } else {
#pragma unroll
                    for (int f = 0; f < D; f += 2)
                        *reinterpret_cast<float2*>(qx + f) = make_float2(xval(h * D + f), xval(h * D + f + 1));
                }
                return true;
            };
            // per-row |x|^2 for the error bound (fp32; only scales the bound)
            float xx[P];
#pragma unroll
            for (int h = 0; h < P; ++h) {
                if (P == 1) {
                    xx[h] = (xq.x + xq.y) + (xq.z + xq.w);
                } else {
                    xx[h] = 0.f;
#pragma unroll
                    for (int f = 0; f < D; ++f) xx[h] = fmaf(xval(h * D + f), xval(h * D + f), xx[h]);
                }
#ifdef KT_EXP_NOXX
                xx[h] = 16.f;
#endif
            }

            // scores: running top-2 over 16-column TMEM chunks
            tc::mbar_wait(&dfull[wg], static_cast<uint32_t>(use & 1));
            tc::tc_fence_after();
            const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16) + wg * NS;
            // two interleaved top-2 chains per row (even / odd score columns),
            // merged below: halves the serial min chain.  Which of two equal fp32
            // scores wins does not matter: a zero gap is always a flagged near-tie.
            float b1x[2][P], b2x[2][P];
            int i1x[2][P];
#pragma unroll
            for (int h = 0; h < P; ++h) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    b1x[e][h] = FLT_MAX;
                    b2x[e][h] = FLT_MAX;
                    i1x[e][h] = 0;
                }
            }
            // (32-column loads where NS allows: one TMEM round trip per 32 scores)
            constexpr int QC = NS % 32 == 0 ? 32 : 16;
#pragma unroll
#ifdef KT_EXP_NOSCORE
            for (int q16 = 0; q16 < 1; ++q16) {
#else
            for (int q16 = 0; q16 < NS / QC; ++q16) {
#endif
                float v[QC];
                if constexpr (QC == 32) tc::tmem_ld32(trow + q16 * QC, v);
                else tc::tmem_ld16(trow + q16 * QC, v);
#pragma unroll
                for (int i = 0; i < QC; ++i) {
                    const int slot = q16 * QC + i, h = slot / K, j = slot % K;
                    const float s = cn[j] + v[i];
                    float& c1 = b1x[i & 1][h];
                    const bool lt = s < c1;
                    b2x[i & 1][h] = fminf(b2x[i & 1][h], fmaxf(c1, s));
                    c1 = fminf(c1, s);
                    i1x[i & 1][h] = lt ? j : i1x[i & 1][h];
                }
            }
            float b1[P], b2[P];
            int i1[P];
#pragma unroll
            for (int h = 0; h < P; ++h) {
                const bool second = b1x[1][h] < b1x[0][h];
                b1[h] = fminf(b1x[0][h], b1x[1][h]);
                b2[h] = fminf(fmaxf(b1x[0][h], b1x[1][h]), fminf(b2x[0][h], b2x[1][h]));
                i1[h] = second ? i1x[1][h] : i1x[0][h];
            }
            int label[P];
            bool flag[P];
            float tau[P];
            bool any_flag = false;
#pragma unroll
            for (int h = 0; h < P; ++h) {
                const int64_t row = (prow0 + t) * P + h;
                label[h] = row < p.n ? i1[h] : K;  // rows past the end sort last
                tau[h] = ERR * (cnmax + 2.f * sqrtf(xx[h]) * cmax);
                flag[h] = row < p.n && K > 1 && !(b2[h] - b1[h] > tau[h]);
                any_flag |= flag[h];
            }
            // near-ties: candidate clusters (score within tau of the best) from a
            // second, warp-uniform TMEM pass (tcgen05.ld is .sync.aligned), then
            // the exact f64 decision over the candidates only
#ifdef KT_EXP_NOREFINE
            any_flag = false;
#endif
            if (__any_sync(FULL, any_flag)) {
                uint64_t cand[P];
#pragma unroll
                for (int h = 0; h < P; ++h) cand[h] = 0;
#pragma unroll
                for (int q16 = 0; q16 < NS / QC; ++q16) {
                    float v[QC];
                    if constexpr (QC == 32) tc::tmem_ld32(trow + q16 * QC, v);
                    else tc::tmem_ld16(trow + q16 * QC, v);
#pragma unroll
                    for (int i = 0; i < QC; ++i) {
                        const int slot = q16 * QC + i, h = slot / K, j = slot % K;
                        if (cn[j] + v[i] <= b1[h] + tau[h]) cand[h] |= 1ull << j;
                    }
                }
                // near-tie rows go to the refine kernel (one warp per row over a
                // balanced queue) instead of stalling this warp -- and with it
                // the warpgroup's next MMA -- for the f64 decision; only a
                // queue overflow refines here
#pragma unroll
                for (int h = 0; h < P; ++h) {
                    if (enqueue(h, flag[h], cand[h], -1)) label[h] = tc_deferred<K>();
                    unsigned fm = __ballot_sync(FULL, flag[h] && label[h] != tc_deferred<K>());
                    // warp-cooperative exact decision, one flagged row at a time
                    // (the row parked in this warp's rows of the lo buffer: free,
                    // the tile's MMAs completed)
                    while (fm) {
                        const int src = __ffs(fm) - 1;
                        fm &= fm - 1;
                        const uint64_t cm = __shfl_sync(FULL, cand[h], src);
                        float* scr = work + wq * 32 * 32;
                        if (lane == src) {
#pragma unroll
                            for (int f = 0; f < D; ++f) scr[f] = xval(h * D + f);
                        }
                        __syncwarp();
                        const int best = tc_refine_warp<D, K>(scr, cm, p.c64, p.cn64, cnmax, cmax, nullptr);
                        __syncwarp();
                        if (lane == src) {
                            label[h] = best;
                            ++refined;
                        }
                    }
                }
            }
            // every score has been read: the accumulator goes back to the MMA
            // issuer before the label stores and the accumulation
            tc::tc_fence_before();
            tc::mbar_arrive(&dempty[wg]);
            if (p.labels) {
#pragma unroll
                for (int h = 0; h < P; ++h) {
                    const int64_t row = (prow0 + t) * P + h;
                    if (row < p.n && label[h] < K) p.labels[row] = label[h];
                }
            }
#pragma unroll
            for (int h = 0; h < P; ++h) {
                const int64_t row = (prow0 + t) * P + h;
                if (row < p.n && label[h] < K && p.lab8) p.lab8[row] = static_cast<int8_t>(label[h]);
            }
            if (!accumulate) continue;

            if (C::DELTA_OK && p.prev) {
                // ---------------- delta iteration: only rows whose label changed,
                // +x into the new cluster and -x out of the old one (the update
                // adds these to the running sums).  They go to the refine
                // kernel's queue like the near-ties (it accumulates them off this
                // warpgroup's MMA critical path); a full queue falls back to the
                // warp itself: the changed row parked in the warp's own rows of
                // `work` (free: the tile's MMAs completed), lanes over features
                float* wrow = work + wq * 32 * 32;  // this warp's first row slot (K-block 0)
#pragma unroll
                for (int h = 0; h < P; ++h) {
                    bool ch = label[h] < K && label[h] != oldl[h];
                    if (enqueue(h, ch, 0ull, label[h])) ch = false;
                    unsigned fm = __ballot_sync(FULL, ch);
                    while (fm) {
                        const int src = __ffs(fm) - 1;
                        fm &= fm - 1;
                        if (lane == src) {
#pragma unroll
                            for (int f = 0; f < D; ++f) wrow[(f / 32) * PR * 32 + f % 32] = xval(h * D + f);
                        }
                        __syncwarp();
                        const int jn = __shfl_sync(FULL, label[h], src), jo = __shfl_sync(FULL, oldl[h], src);
                        for (int f = lane; f < D; f += 32) {
                            const long long qv = __float2ll_rn(wrow[(f / 32) * PR * 32 + f % 32] * qscale);
                            atomicAdd(reinterpret_cast<unsigned long long*>(acc + jn * D + f), static_cast<unsigned long long>(qv));
                            if (jo >= 0)
                                atomicAdd(reinterpret_cast<unsigned long long*>(acc + jo * D + f), static_cast<unsigned long long>(-qv));
                        }
                        if (lane == 0) {
                            atomicAdd(reinterpret_cast<unsigned long long*>(acc + KD + jn), 1ull);
                            if (jo >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc + KD + jo), ~0ull);
                        }
                        __syncwarp();
                    }
                }
                continue;
            }

            // ---------------- counting sort of the tile by label (groups vw = h*4 + wq)
            unsigned mine[P];
            int rank[P];
            for (int e = lane; e < P * K; e += 32) cnt[((e / K) * 4 + wq) * K + (e % K)] = 0;
            __syncwarp();
#pragma unroll
            for (int h = 0; h < P; ++h) {
                mine[h] = __match_any_sync(FULL, label[h]);
                rank[h] = __popc(mine[h] & ((1u << lane) - 1u));
                if (rank[h] == 0 && label[h] < K) cnt[(h * 4 + wq) * K + label[h]] = static_cast<unsigned short>(__popc(mine[h]));
            }
            tc::named_sync(bar_id, 128);
            int total[KL], before[KL][P], start[KL];
#pragma unroll
            for (int u = 0; u < KL; ++u) {
                const int j = lane + 32 * u;
                total[u] = 0;
#pragma unroll
                for (int h = 0; h < P; ++h) before[u][h] = 0;
                if (j < K) {
#pragma unroll
                    for (int v = 0; v < VW; ++v) {
                        const int c = cnt[v * K + j];
                        total[u] += c;
#pragma unroll
                        for (int h = 0; h < P; ++h) before[u][h] += v < h * 4 + wq ? c : 0;
                    }
                }
            }
            {
                int carry = 0;
#pragma unroll
                for (int u = 0; u < KL; ++u) {
                    int incl = total[u];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int v = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += v;
                    }
                    start[u] = carry + incl - total[u];
                    carry += __shfl_sync(FULL, incl, 31);
                    if (wq == 0 && lane + 32 * u < K && total[u])
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + KD + lane + 32 * u),
                                  static_cast<unsigned long long>(total[u]));
                }
            }
            // scatter rows into label order (features from registers) -- the lo
            // buffer is free once the scores are in (its MMAs completed)
#pragma unroll
            for (int h = 0; h < P; ++h) {
                const int lb = label[h] < K ? label[h] : 0;
                int base = 0;
#pragma unroll
                for (int u = 0; u < KL; ++u) {
                    const int v = __shfl_sync(FULL, start[u] + before[u][h], lb % 32);
                    if (lb / 32 == u) base = v;
                }
                const int pos = base + rank[h];
                if (label[h] < K) {
#pragma unroll
                    for (int f = 0; f < D; f += 2)
                        *reinterpret_cast<float2*>(work + pos * D + f) = make_float2(xval(h * D + f), xval(h * D + f + 1));
                }
            }
            tc::named_sync(bar_id, 128);

            // warp wq sums the sorted runs of clusters wq, wq+4, ... (f64 from the
            // fp32 rows), NU clusters at a time so their load/add chains overlap;
            // each run is still summed in row order (bit-identical), and empty runs
            // skip the shared-memory update (adding +0.0 would be a no-op)
#pragma unroll
            for (int jj = 0; jj < JW; jj += NU) {
                int js[NU], rs[NU], re[NU];
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    js[u] = wq + (jj + u) * 4;
                    const int jc = js[u] < K ? js[u] : 0;
                    rs[u] = __shfl_sync(FULL, start[jc / 32], jc % 32);
                    re[u] = js[u] < K && jj + u < JW ? rs[u] + __shfl_sync(FULL, total[jc / 32], jc % 32) : rs[u];
                }
                double2 part[NU];
#pragma unroll
                for (int u = 0; u < NU; ++u) part[u] = make_double2(0.0, 0.0);
                if (g < G) {
                    int nmax = 0;
#pragma unroll
                    for (int u = 0; u < NU; ++u) nmax = max(nmax, re[u] - rs[u]);
#pragma unroll 2
                    for (int i = g; i < nmax; i += G) {
#pragma unroll
                        for (int u = 0; u < NU; ++u) {
                            if (i < re[u] - rs[u]) {
                                const float2 v = *reinterpret_cast<const float2*>(work + (rs[u] + i) * D + 2 * q);
                                part[u].x += static_cast<double>(v.x);
                                part[u].y += static_cast<double>(v.y);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    if (re[u] == rs[u]) continue;  // warp-uniform
#pragma unroll
                    for (int o = 1; o < G; o <<= 1) {
                        const double vx = __shfl_down_sync(FULL, part[u].x, o * L);
                        const double vy = __shfl_down_sync(FULL, part[u].y, o * L);
                        if (g + o < G) {
                            part[u].x += vx;
                            part[u].y += vy;
                        }
                    }
                    if (g == 0 && q < L) {  // the tile's run sum, once rounded to fixed point
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + js[u] * D + 2 * q),
                                  static_cast<unsigned long long>(llrint(ldexp(part[u].x, shift))));
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + js[u] * D + 2 * q + 1),
                                  static_cast<unsigned long long>(llrint(ldexp(part[u].y, shift))));
                    }
                }
            }
            // the next tile's split rewrites `work` (lo): all warps must be done reading it
            tc::named_sync(bar_id, 128);
        }
        if (refined) atomicAdd(p.refined, refined);
        qholes();
        if (accumulate) {
            // every warpgroup is past its last tile: the CTA's fixed-point sums
            // and counts -> its f64 partial row, in place (summed over CTAs in
            // CTA order)
            __threadfence();
            tc::named_sync(15, C::EPI);
            double* out = p.partials + static_cast<int64_t>(blockIdx.x) * (KD + K);
            for (int e = tid; e < KD + K; e += C::EPI) {
                const long long v = __ldcg(acc + e);
                out[e] = e < KD ? ldexp(static_cast<double>(v), -shift) : static_cast<double>(v);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == CTRL) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ---------------------------------------------------------------- near-tie refine
// Runs after kmeans_tc_kernel in the same stream: one warp per queued row (the
// rows whose fp32 top-2 gap fell inside the error bound, ~2% at cfg3), the
// exact decision of tc_refine_warp, then what the tc kernel skipped for the
// row: labels / lab8, and its accumulation -- every row in a full iteration,
// +x / -x when the label changed in a delta iteration -- as int64 fixed point
// (the tc kernel's scale; integer adds commute, so the result does not depend
// on which warp took which row).  The last CTA turns the sums into partial row
// `partial` (after the tc kernel's per-CTA rows) and resets the queue and the
// accumulator for the next launch.
struct TcRefineParams {
    int64_t n;
    const double* c64;
    const double* cn64;
    const float* bounds;
    const double* xabs;
    unsigned* ctl;                 // [0] queue entries, [1] ticket
    const uint64_t* qrow;          // row | (uint8)(decided label + 1) << 48 | (uint8)last label << 56
    const unsigned long long* qcand;
    const float* qx;               // rows in the queue, or null: read from x
    const float* x;
    unsigned cap;
    int32_t* labels;
    int8_t* lab8;
    long long* racc;               // K*D sums, K counts (zero between launches)
    double* partial;               // null: predict (no accumulation)
    unsigned long long* refined;
    const int* done;
};

#ifndef DNDC_REFINE_THREADS
#define DNDC_REFINE_THREADS 512
#endif
#ifndef DNDC_REFINE_CH
#define DNDC_REFINE_CH 1024
#endif
template <int D, int K>
__host__ __device__ constexpr int tc_refine_threads() { return DNDC_REFINE_THREADS; }

// shared memory of kmeans_tc_refine_kernel (dynamic): transposed f64
// centroids, |c|^2, the int64 sums, and one queue chunk's bookkeeping
template <int D, int K>
struct TcRefineSmem {
    static constexpr int CH = DNDC_REFINE_CH, NW = tc_refine_threads<D, K>() / 32;
    static constexpr int OFF_CT = 0;                                  // double [D][K]
    static constexpr int OFF_CN = OFF_CT + D * K * 8;                 // double [K]
    static constexpr int OFF_ACC = OFF_CN + K * 8;                    // long long [K*D + K]
    static constexpr int OFF_QV = OFF_ACC + (K * D + K) * 8;          // uint64 [CH]
    static constexpr int OFF_LST = OFF_QV + CH * 8;                   // u16 [2 CH]
    static constexpr int OFF_UND = OFF_LST + 2 * CH * 2;              // u16 [CH]
    static constexpr int OFF_CNT = OFF_UND + CH * 2;                  // int [2K] counts, [2K+1] starts, [2K] cursors, [1] nund
    static constexpr int OFF_NLAB = OFF_CNT + (6 * K + 2) * 4;        // int8 [CH]
    static constexpr int OFF_ROWS = (OFF_NLAB + CH + 15) / 16 * 16;   // float [NW][D]
    static constexpr int BYTES = OFF_ROWS + NW * D * 4;
};

// The queue is taken in chunks of CH entries per CTA.  In a chunk:
// (1) the near-tie rows are decided one LANE per row (the row in registers, f64
//     distances to its candidate clusters from a transposed shared copy of the
//     centroids); only rows the f64 filter cannot separate go to the
//     warp-cooperative reference-order decision (tc_refine_warp);
// (2) the rows whose label changed are bucketed by cluster (+x under the new
//     label, -x under the old one), a counting sort in shared memory;
// (3) the bucketed list is split evenly over the warps; each sums its range
//     in registers, eight rows in flight, and adds a run to the shared int64
//     sums only where its cluster changes (no atomic per row).
// Rows come from the queue (qx) or are read from X.  At the end the CTA adds
// its sums to racc; the last CTA converts racc into the partial row and
// resets the queue.
template <int D, int K>
__global__ void __launch_bounds__(DNDC_REFINE_THREADS) kmeans_tc_refine_kernel(TcRefineParams p) {
    using L = TcRefineSmem<D, K>;
    constexpr int KD = K * D, NT = tc_refine_threads<D, K>(), NW = L::NW, CH = L::CH;
    constexpr int FPL = (D + 31) / 32;
    static_assert(K <= 127 && D % 2 == 0, "int8 labels, float2 rows");
    extern __shared__ __align__(16) unsigned char rsm[];
    double* cT = reinterpret_cast<double*>(rsm + L::OFF_CT);
    double* cnS = reinterpret_cast<double*>(rsm + L::OFF_CN);
    long long* sacc = reinterpret_cast<long long*>(rsm + L::OFF_ACC);
    uint64_t* qv = reinterpret_cast<uint64_t*>(rsm + L::OFF_QV);
    unsigned short* lst = reinterpret_cast<unsigned short*>(rsm + L::OFF_LST);
    unsigned short* und = reinterpret_cast<unsigned short*>(rsm + L::OFF_UND);
    int* cnt = reinterpret_cast<int*>(rsm + L::OFF_CNT);
    int* start = cnt + 2 * K;
    int* cur = start + 2 * K + 1;
    int* nund = cur + 2 * K;
    signed char* nlab = reinterpret_cast<signed char*>(rsm + L::OFF_NLAB);
    float* rows = reinterpret_cast<float*>(rsm + L::OFF_ROWS);
    __shared__ bool last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool skip = p.done && *p.done;
    const unsigned count = skip ? 0u : min(p.ctl[0], p.cap);
    int e2 = 0;
    frexp(static_cast<double>(p.n) * (p.xabs ? *p.xabs : 1.0) + 1.0, &e2);
    const int shift = 61 - e2;
    const float qscale = ldexpf(1.f, shift);
    const float cmax = p.bounds[0], cnmax = p.bounds[1];
    constexpr uint64_t RMASK = (1ull << 48) - 1;
    auto src_of = [&](unsigned e, uint64_t v) -> const float* {
        return p.qx ? p.qx + static_cast<int64_t>(e) * D : p.x + static_cast<int64_t>(v & RMASK) * D;
    };
    const unsigned nchunks = (count + CH - 1) / CH;
    if (blockIdx.x < nchunks) {
        for (int e = tid; e < KD; e += NT) cT[(e % D) * K + e / D] = p.c64[e];
        for (int j = tid; j < K; j += NT) cnS[j] = p.cn64[j];
        for (int e = tid; e < KD + K; e += NT) sacc[e] = 0;
    }
    unsigned nref = 0;
    for (unsigned c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const unsigned e0 = c * CH;
        const int ne = static_cast<int>(min(static_cast<unsigned>(CH), count - e0));
        for (int i = tid; i < 2 * K; i += NT) cnt[i] = 0;
        if (tid == 0) *nund = 0;
        __syncthreads();
        for (int i = tid; i < ne; i += NT) {
            const uint64_t v = p.qrow[e0 + i];
            qv[i] = v;
            int dec = -2;
            if (v != TC_QHOLE) {
                dec = static_cast<int>((v >> 48) & 0xff) - 1;
                if (dec < 0) und[atomicAdd(nund, 1)] = static_cast<unsigned short>(i);
            }
            nlab[i] = static_cast<signed char>(dec);
        }
        __syncthreads();
        // (1) near-ties, lane per row
        const int nu = *nund;
        for (int base = warp * 32; base < nu; base += NW * 32) {
            const int k = base + lane;
            const bool active = k < nu;
            const int i = active ? und[k] : 0;
            const uint64_t v = qv[i];
            const uint64_t cm = active ? p.qcand[e0 + i] : 0ull;
            float xr[D];
            {
                const float* src = active ? src_of(e0 + i, v) : nullptr;
                if constexpr (D % 4 == 0) {
#pragma unroll
                    for (int q = 0; q < D / 4; ++q) {
                        const float4 t = active ? reinterpret_cast<const float4*>(src)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
                        xr[4 * q] = t.x;
                        xr[4 * q + 1] = t.y;
                        xr[4 * q + 2] = t.z;
                        xr[4 * q + 3] = t.w;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < D / 2; ++q) {
                        const float2 t = active ? reinterpret_cast<const float2*>(src)[q] : make_float2(0.f, 0.f);
                        xr[2 * q] = t.x;
                        xr[2 * q + 1] = t.y;
                    }
                }
            }
            double xn = 0.0;
#pragma unroll
            for (int f = 0; f < D; ++f) xn = fma(static_cast<double>(xr[f]), static_cast<double>(xr[f]), xn);
            double d1 = DBL_MAX, d2 = DBL_MAX;
            int best = K;
            for (uint64_t rest = cm; rest;) {
                int js[4];
                double g[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    js[q] = rest ? __ffsll(static_cast<long long>(rest)) - 1 : -1;
                    rest &= rest - 1;
                    g[q] = 0.0;
                }
                const int j0 = js[0] < 0 ? 0 : js[0], j1 = js[1] < 0 ? 0 : js[1];
                const int j2 = js[2] < 0 ? 0 : js[2], j3 = js[3] < 0 ? 0 : js[3];
#pragma unroll
                for (int f = 0; f < D; ++f) {
                    const double xf = static_cast<double>(xr[f]);
                    const double* col = cT + f * K;
                    g[0] = fma(xf, col[j0], g[0]);
                    g[1] = fma(xf, col[j1], g[1]);
                    g[2] = fma(xf, col[j2], g[2]);
                    g[3] = fma(xf, col[j3], g[3]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (js[q] < 0) continue;
                    const double dq = xn + cnS[js[q]] - 2.0 * g[q];
                    if (dq < d1) {
                        d2 = d1;
                        d1 = dq;
                        best = js[q];
                    } else if (dq < d2) {
                        d2 = dq;
                    }
                }
            }
            const double margin =
                0x1.0p-40 * (xn + static_cast<double>(cnmax) + 2.0 * sqrt(xn) * static_cast<double>(cmax));
            const bool decided = active && d1 > margin && d2 - d1 > margin;
            // not separable by the filter: the reference's operation order, one
            // row at a time, warp-cooperative
            unsigned fm = __ballot_sync(FULL, active && !decided);
            while (fm) {
                const int src = __ffs(fm) - 1;
                fm &= fm - 1;
                float* rw = rows + warp * D;
                if (lane == src) {
#pragma unroll
                    for (int f = 0; f < D; ++f) rw[f] = xr[f];
                }
                __syncwarp();
                const int b = tc_refine_warp<D, K>(rw, __shfl_sync(FULL, cm, src), p.c64, p.cn64, cnmax, cmax, nullptr);
                __syncwarp();
                if (lane == src) best = b;
            }
            if (active) {
                nlab[i] = static_cast<signed char>(best);
                ++nref;
                const int64_t r = static_cast<int64_t>(v & RMASK);
                if (p.labels) p.labels[r] = best;
                if (p.lab8) p.lab8[r] = static_cast<int8_t>(best);
            }
        }
        __syncthreads();
        if (p.partial) {
            // (2) buckets: + new label, - last label (rows whose label changed)
            for (int i = tid; i < ne; i += NT) {
                const int nl = nlab[i], old = static_cast<int8_t>(static_cast<uint8_t>(qv[i] >> 56));
                if (nl >= 0 && nl != old) {
                    atomicAdd(&cnt[nl], 1);
                    if (old >= 0) atomicAdd(&cnt[K + old], 1);
                }
            }
            __syncthreads();
            if (warp == 0) {
                int carry = 0;
                for (int b = 0; b < 2 * K; b += 32) {
                    const int v = b + lane < 2 * K ? cnt[b + lane] : 0;
                    int incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += t;
                    }
                    if (b + lane < 2 * K) {
                        start[b + lane] = carry + incl - v;
                        cur[b + lane] = carry + incl - v;
                    }
                    carry += __shfl_sync(FULL, incl, 31);
                }
                if (lane == 0) start[2 * K] = carry;
            }
            __syncthreads();
            for (int i = tid; i < ne; i += NT) {
                const int nl = nlab[i], old = static_cast<int8_t>(static_cast<uint8_t>(qv[i] >> 56));
                if (nl >= 0 && nl != old) {
                    lst[atomicAdd(&cur[nl], 1)] = static_cast<unsigned short>(i);
                    if (old >= 0) lst[atomicAdd(&cur[K + old], 1)] = static_cast<unsigned short>(i);
                }
            }
            __syncthreads();
            // (3) an even share of the bucketed list per warp, runs summed in registers
            const int total = start[2 * K];
            const int lo = static_cast<int>(static_cast<int64_t>(total) * warp / NW);
            const int hi = static_cast<int>(static_cast<int64_t>(total) * (warp + 1) / NW);
            if (lo < hi) {
                int bk = 0;
                while (start[bk + 1] <= lo) ++bk;
                int bend = start[bk + 1], runs = 0;
                long long acc[FPL];
#pragma unroll
                for (int f = 0; f < FPL; ++f) acc[f] = 0;
                auto flush = [&]() {
                    const int j = bk < K ? bk : bk - K;
                    const bool neg = bk >= K;
#pragma unroll
                    for (int f = 0; f < FPL; ++f) {
                        const int ff = lane + 32 * f;
                        if (ff < D && acc[f])
                            atomicAdd(reinterpret_cast<unsigned long long*>(sacc + j * D + ff),
                                      static_cast<unsigned long long>(neg ? -acc[f] : acc[f]));
                        acc[f] = 0;
                    }
                    if (lane == 0 && runs)
                        atomicAdd(reinterpret_cast<unsigned long long*>(sacc + KD + j),
                                  static_cast<unsigned long long>(neg ? -static_cast<long long>(runs) : runs));
                    runs = 0;
                };
                for (int b = lo; b < hi; b += 8) {
                    float xv[8][FPL];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int idx = b + q < hi ? lst[b + q] : -1;
                        const float* src = idx >= 0 ? src_of(e0 + idx, qv[idx]) : nullptr;
#pragma unroll
                        for (int f = 0; f < FPL; ++f) {
                            const int ff = lane + 32 * f;
                            xv[q][f] = (src && ff < D) ? src[ff] : 0.f;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (b + q >= hi) break;
                        while (b + q >= bend) {
                            flush();
                            ++bk;
                            bend = start[bk + 1];
                        }
#pragma unroll
                        for (int f = 0; f < FPL; ++f) acc[f] += __float2ll_rn(xv[q][f] * qscale);
                        ++runs;
                    }
                }
                flush();
            }
        }
        __syncthreads();
    }
    nref = __reduce_add_sync(FULL, nref);  // lane per row: every lane counted its own
    if (lane == 0 && nref) atomicAdd(p.refined, static_cast<unsigned long long>(nref));
    if (p.partial && blockIdx.x < nchunks) {
        for (int e = tid; e < KD + K; e += NT)
            if (sacc[e]) atomicAdd(reinterpret_cast<unsigned long long*>(p.racc + e), static_cast<unsigned long long>(sacc[e]));
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(p.ctl + 1, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int e = tid; e < KD + K; e += blockDim.x) {
        const long long v = static_cast<long long>(atomicExch(reinterpret_cast<unsigned long long*>(p.racc + e), 0ull));
        if (p.partial) p.partial[e] = e < KD ? ldexp(static_cast<double>(v), -shift) : static_cast<double>(v);
    }
    if (tid == 0) {
        p.ctl[0] = 0;
        p.ctl[1] = 0;
    }
}

// ------------------------------------------------ TMEM-operand delta / predict kernel
// kmeans_tcd_kernel: the same scores and decisions as kmeans_tc_kernel (P = 1),
// for the launches that accumulate nothing per row -- delta iterations (the
// changed rows go to the refine queue) and predict.  Laid out for the shared
// memory port, which bounds the smem-operand kernel (per 128-row tile it moved
// 240 KB through the 128 B/clk crossbar: the TMA write, the split's read and
// lo write, and the MMAs' A and B reads):
//   * the split writes BOTH halves of the row (raw = hi, the tensor core reads
//     tf32; lo = x - trunc(x)) into tensor memory with tcgen05.st (256 B/clk),
//     and the MMAs take A from TMEM: shared memory carries only the TMA tile,
//     its one read by the split, and the centroid operand B (112 KB per tile);
//   * the stage is released as soon as the split has read it;
//   * four epilogue warpgroups (tile it: warpgroup it % 4) for latency hiding;
//     TMEM: two A sets (hi | lo, tile it uses set it % 2, free again when the
//     MMAs of tile it - 2 retired) and one score block per warpgroup
//     (2 x 128 + 4 x 64 = 512 columns).  (Starting the score block at |c|^2
//     with tcgen05.st instead of one add per score measured slower.)
// kmeans_tcd_kernel's queue-overflow fallback, out of line (keeps the
// f64 decision's registers out of the kernel's main loop)
template <int D, int K>
__device__ __noinline__ int tcd_refine_row(const float* row, uint64_t cm, const double* __restrict__ c64,
                                           const double* __restrict__ cn64, float cnmax, float cmax) {
    return tc_refine_warp<D, K>(row, cm, c64, cn64, cnmax, cmax, nullptr);
}

#ifdef TCD_TRACE
// diagnostics (-DTCD_TRACE builds only): %globaltimer marks of CTA 0's first 64
// tiles: [0] MMAs issued, [2] A ready seen by the issuer, [4] A written,
// [5] scores ready, [6] scores read, [7] tile done
__device__ unsigned long long g_tcd_trace[64 * 8];
__device__ __forceinline__ void tcd_mark(int64_t it, int k) {
    if (blockIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tcd_trace[it * 8 + k] = t;
    }
}
#define TCD_MARK(it, k) tcd_mark(it, k)
#else
#define TCD_MARK(it, k) ((void)0)
#endif

template <int D, int K>
struct TcdCfg {
    static constexpr int KC = ((D + 7) / 8) * 8;
    static constexpr int NCH = KC / 4;
    static constexpr int NKB = (KC + 31) / 32;
    static constexpr int NS = K;
    static constexpr int PR = 128;
    static constexpr int WGS = 4;
    static constexpr int ASETS = 2;
    static constexpr int EPI = 128 * WGS;
    static constexpr int THREADS = EPI + 64;  // + the MMA warp + the TMA warp
    static constexpr int TILE_BYTES = NKB * PR * 128;
    static constexpr int B_BYTES = NCH * NS * 16;
    static constexpr int ROWB = (D * 4 + 15) / 16 * 16;
    static constexpr int SCR_BYTES = (EPI / 32) * ROWB;  // per-warp row (queue-overflow fallback)
    static constexpr int ACOLS = ((KC + 31) / 32) * 32;  // TMEM columns of one A half
    static constexpr int DBASE = ASETS * 2 * ACOLS;      // score blocks after the A sets
    static constexpr int TMEM_COLS = tc_pow2_cols(DBASE + WGS * NS);
    static constexpr int FIXED = 2 * B_BYTES + ((K * 4 + 15) / 16) * 16 + SCR_BYTES + 64 * 8 + 16;
    static constexpr int S = (232448 - FIXED) / TILE_BYTES > 6 ? 6 : (232448 - FIXED) / TILE_BYTES;
    static constexpr int OFF_TILE = 0;
    static constexpr int OFF_BHI = OFF_TILE + S * TILE_BYTES;
    static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
    static constexpr int OFF_CN = OFF_BLO + B_BYTES;
    static constexpr int OFF_SCR = OFF_CN + ((K * 4 + 15) / 16) * 16;
    static constexpr int OFF_BAR = OFF_SCR + SCR_BYTES;
    static constexpr int NBARS = 2 * S + 2 * WGS;
    static constexpr int OFF_TMEM = OFF_BAR + NBARS * 8;
    static constexpr int SMEM = OFF_TMEM + 16;
    static_assert(S >= 3, "kmeans_tcd: at least three TMA stages");
    static_assert(NS % 16 == 0 && DBASE + WGS * NS <= 512, "MMA N / TMEM columns");
    static_assert(D % 16 == 0 && D <= 64 && K <= 64, "kmeans_tcd shape (16-column TMEM stores)");
    static_assert(SMEM <= 232448, "shared memory");
    static_assert(TILE_BYTES % 1024 == 0, "SW128 tiles need 1024-byte alignment");
};

template <int D, int K>
__global__ void __launch_bounds__(TcdCfg<D, K>::THREADS, 1)
    kmeans_tcd_kernel(const __grid_constant__ CUtensorMap map, TcParams p) {
    using C = TcdCfg<D, K>;
    constexpr int NS = C::NS, PR = C::PR, S = C::S, KD = K * D, WGS = C::WGS;
    if (p.done && *p.done) return;

    extern __shared__ __align__(1024) unsigned char smem[];
    if (tc::smem_u32(smem) & 1023u) __trap();
    float* tiles = reinterpret_cast<float*>(smem + C::OFF_TILE);
    float* bhi = reinterpret_cast<float*>(smem + C::OFF_BHI);
    float* blo = reinterpret_cast<float*>(smem + C::OFF_BLO);
    float* cn = reinterpret_cast<float*>(smem + C::OFF_CN);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* full = bars;             // [S] TMA landed
    uint64_t* empty = bars + S;        // [S] stage read by the split (4 warp arrivals)
    uint64_t* aready = bars + 2 * S;   // [WGS] A hi/lo in TMEM (4 warp arrivals)
    uint64_t* dfull = aready + WGS;    // [WGS] scores ready (MMAs retired: A free again)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool accumulate = p.partials != nullptr;
    constexpr int CTRL = C::EPI / 32;

    if (warp == CTRL) {
        tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 4);
            }
            for (int w = 0; w < WGS; ++w) {
                tc::mbar_init(&aready[w], 4);
                tc::mbar_init(&dfull[w], 1);
            }
            tc::mbar_fence_init();
            tc::tma_prefetch_desc(&map);
        }
    } else if (warp < CTRL) {
        for (int e = tid; e < NS * C::KC; e += C::EPI) {
            const int j = e / C::KC, f = e % C::KC;
            const float v = f < D ? p.ctab[j * D + f] : 0.f;
            const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            const int off = (f / 4) * (NS * 4) + j * 4 + (f % 4);
            bhi[off] = hi;
            blo[off] = v - hi;
        }
        for (int j = tid; j < K; j += C::EPI) cn[j] = p.ctab[KD + j];
        tc::fence_async_smem();
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int64_t ntiles = ceil_div(p.n, static_cast<int64_t>(PR));
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == CTRL) {
        // ------------------------------------------------ MMA issuer
        // the whole warp runs the loop (converged: the MMAs are issued by an
        // elect.sync inside their asm, without a per-instruction divergence loop)
        constexpr uint32_t idesc = tc::idesc_tf32(128, NS, 0, 0);
        const uint64_t bh0 = tc::smem_desc(tc::smem_u32(bhi), NS * 16, 128);
        const uint64_t bl0 = tc::smem_desc(tc::smem_u32(blo), NS * 16, 128);
#pragma unroll 1
        for (int64_t it = 0; it < my_tiles; ++it) {
            const int w = static_cast<int>(it % WGS);
            if (lane == 0) TCD_MARK(it, 1);
            tc::mbar_wait(&aready[w], static_cast<uint32_t>((it / WGS) & 1));
            __syncwarp();
            if (lane == 0) TCD_MARK(it, 2);
            tc::tc_fence_after();
            const uint32_t ahi = tmem + static_cast<uint32_t>(it % C::ASETS) * 2 * C::ACOLS, alo = ahi + C::ACOLS;
            const uint32_t dt = tmem + C::DBASE + w * NS;
#pragma unroll
            for (int ks = 0; ks < C::KC / 8; ++ks)  // descriptor start address field: 16-byte units
                tc::mma3_tf32_ta_elect(dt, ahi + ks * 8, alo + ks * 8, bh0 + static_cast<uint64_t>(ks * 2 * NS),
                                       bl0 + static_cast<uint64_t>(ks * 2 * NS), idesc, ks > 0);
            tc::mma_commit_elect(&dfull[w]);
            if (lane == 0) TCD_MARK(it, 0);
        }
    } else if (warp == CTRL + 1) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            for (int64_t it = 0; it < my_tiles; ++it) {
                const int st = static_cast<int>(it % S);
                if (it >= S) tc::mbar_wait(&empty[st], static_cast<uint32_t>((it / S - 1) & 1));
                const int prow = static_cast<int>((blockIdx.x + it * gridDim.x) * PR);
                float* dst = tiles + st * (C::TILE_BYTES / 4);
                tc::mbar_expect_tx(&full[st], C::TILE_BYTES);
#pragma unroll
#ifndef DNDC_TC_NO_EVICT_FIRST  // X tiles leave L2 first (cfg3 shard: 0.532 -> 0.518 ms per iteration)
                for (int kb = 0; kb < C::NKB; ++kb)
                    tc::tma_load_2d_hint(dst + kb * PR * 32, &map, &full[st], kb * 32, prow, tc::l2_policy_evict_first());
#else
                for (int kb = 0; kb < C::NKB; ++kb) tc::tma_load_2d(dst + kb * PR * 32, &map, &full[st], kb * 32, prow);
#endif
            }
        }
    } else {
        // ------------------------------------------------ epilogue warpgroups
        const int wg = warp / 4, wq = warp % 4, t = tid % 128;
        const float cmax = p.bounds[0], cnmax = p.bounds[1];
        constexpr float ERR = 4.f * (static_cast<float>(3 * C::KC) * 0x1.0p-24f + 3.f * 0x1.0p-20f);
        float* wscr = reinterpret_cast<float*>(smem + C::OFF_SCR + warp * C::ROWB);
        unsigned long long refined = 0;
        constexpr unsigned QCHUNK = 64;
        unsigned qbase = 0, qleft = 0;
        auto qholes = [&]() {
            for (unsigned i = lane; i < qleft; i += 32)
                if (qbase + i < p.rq_cap) p.rq_row[qbase + i] = TC_QHOLE;
        };
        // queue-overflow fallback only: +x / -x of changed rows as int64 REDs
        // into the CTA's partial row (zero otherwise; converted at the end)
        long long* acc = accumulate ? reinterpret_cast<long long*>(p.partials + static_cast<int64_t>(blockIdx.x) * (KD + K))
                                    : nullptr;
        if (accumulate)
            for (int e = tid; e < KD + K; e += C::EPI) acc[e] = 0ll;
        __threadfence();
        int e2 = 0;
        frexp(static_cast<double>(p.n) * (p.xabs ? *p.xabs : 1.0) + 1.0, &e2);
        const int shift = 61 - e2;
        const float qscale = ldexpf(1.f, shift);
        tc::named_sync(15, C::EPI);

        const uint32_t lanes = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t trow = tmem + lanes + C::DBASE + wg * NS;
        auto park = [&](int64_t row) {
            for (int f = lane; f < D; f += 32) wscr[f] = __ldg(p.x + row * D + f);
            __syncwarp();
        };
        for (int64_t it = wg; it < my_tiles; it += WGS) {
            const int st = static_cast<int>(it % S);
            const int64_t use = it / WGS;
            const int64_t row = (blockIdx.x + it * gridDim.x) * PR + t;
            const bool live = row < p.n;
            const int oldl = (p.prev && live) ? static_cast<int>(p.prev[row]) : -1;
            const float* xt = tiles + st * (C::TILE_BYTES / 4);
            // A set it % 2 is free once the MMAs of tile it - 2 (another
            // warpgroup's) retired
            const uint32_t ahi = tmem + lanes + static_cast<uint32_t>(it % C::ASETS) * 2 * C::ACOLS, alo = ahi + C::ACOLS;
            if (it >= C::ASETS)
                tc::mbar_wait(&dfull[(it - C::ASETS) % WGS], static_cast<uint32_t>(((it - C::ASETS) / WGS) & 1));
            tc::mbar_wait(&full[st], static_cast<uint32_t>((it / S) & 1));
            tc::tc_fence_after();
            // split: 16 features at a time from the swizzled tile into TMEM,
            // raw (= hi: the tensor core reads tf32) and lo = x - trunc(x);
            // |x|^2 for the error bound on the way
            float4 xq = make_float4(0.f, 0.f, 0.f, 0.f);
            // the row's swizzle phase through an opaque shuffle: otherwise the
            // compiler hoists all 16 chunk offsets out of the tile loop and
            // spills them (the kernel runs at 128 registers)
            const int t7 = __shfl_sync(FULL, t & 7, lane);
            const float* xrow = xt + t * 32;
#pragma unroll
            for (int g = 0; g < C::KC / 16; ++g) {
                float hv[16], lv[16];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = g * 4 + u;
                    const float4 v = *reinterpret_cast<const float4*>(xrow + (c / 8) * PR * 32 + (((c % 8) ^ t7) * 4));
                    hv[4 * u] = v.x;
                    hv[4 * u + 1] = v.y;
                    hv[4 * u + 2] = v.z;
                    hv[4 * u + 3] = v.w;
                    xq.x = fmaf(v.x, v.x, xq.x);
                    xq.y = fmaf(v.y, v.y, xq.y);
                    xq.z = fmaf(v.z, v.z, xq.z);
                    xq.w = fmaf(v.w, v.w, xq.w);
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) lv[i] = hv[i] - __uint_as_float(__float_as_uint(hv[i]) & 0xFFFFE000u);
                tc::tmem_st16(ahi + g * 16, hv);
                tc::tmem_st16(alo + g * 16, lv);
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[st]);  // the stage is read: TMA may refill it
            tc::tmem_st_wait();
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&aready[wg]);
            if (t == 0) TCD_MARK(it, 4);
            const float xx = (xq.x + xq.y) + (xq.z + xq.w);

            tc::mbar_wait(&dfull[wg], static_cast<uint32_t>(use & 1));
            if (t == 0) TCD_MARK(it, 5);
            tc::tc_fence_after();
            float b1x[2] = {FLT_MAX, FLT_MAX}, b2x[2] = {FLT_MAX, FLT_MAX};
            int i1x[2] = {0, 0};
            constexpr int QC = NS % 32 == 0 ? 32 : 16;
#pragma unroll
            for (int q16 = 0; q16 < NS / QC; ++q16) {
                float v[QC];
                if constexpr (QC == 32) tc::tmem_ld32(trow + q16 * QC, v);
                else tc::tmem_ld16(trow + q16 * QC, v);
#pragma unroll
                for (int i = 0; i < QC; ++i) {
                    const int j = q16 * QC + i;
                    const float s = cn[j] + v[i];
                    float& c1 = b1x[i & 1];
                    const bool lt = s < c1;
                    b2x[i & 1] = fminf(b2x[i & 1], fmaxf(c1, s));
                    c1 = fminf(c1, s);
                    i1x[i & 1] = lt ? j : i1x[i & 1];
                }
            }
            const float b1 = fminf(b1x[0], b1x[1]);
            const float b2 = fminf(fmaxf(b1x[0], b1x[1]), fminf(b2x[0], b2x[1]));
            int label = live ? (b1x[1] < b1x[0] ? i1x[1] : i1x[0]) : K;
            const float tau = ERR * (cnmax + 2.f * sqrtf(xx) * cmax);
            const bool flag = live && K > 1 && !(b2 - b1 > tau);
            uint64_t cand = 0;
            const bool wflag = __any_sync(FULL, flag);
            if (wflag) {
#pragma unroll
                for (int q16 = 0; q16 < NS / QC; ++q16) {
                    float v[QC];
                    if constexpr (QC == 32) tc::tmem_ld32(trow + q16 * QC, v);
                    else tc::tmem_ld16(trow + q16 * QC, v);
#pragma unroll
                    for (int i = 0; i < QC; ++i) {
                        const int j = q16 * QC + i;
                        if (cn[j] + v[i] <= b1 + tau) cand |= 1ull << j;
                    }
                }
            }
            tc::tc_fence_before();
            if (t == 0) TCD_MARK(it, 6);

            auto enqueue = [&](bool want, uint64_t cm, int newl) -> bool {
                const unsigned fm = __ballot_sync(FULL, want);
                if (!p.rq_ctl || !fm) return false;
                const unsigned cnt = static_cast<unsigned>(__popc(fm));
                if (cnt > qleft) {
                    qholes();
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(p.rq_ctl, QCHUNK);
                    qbase = __shfl_sync(FULL, base, 0);
                    qleft = QCHUNK;
                }
                const unsigned pos = qbase + static_cast<unsigned>(__popc(fm & ((1u << lane) - 1u)));
                qbase += cnt;
                qleft -= cnt;
                if (!want || pos >= p.rq_cap) return false;
                p.rq_row[pos] = static_cast<uint64_t>(row) | (static_cast<uint64_t>(static_cast<uint8_t>(oldl)) << 56) |
                                (static_cast<uint64_t>(static_cast<uint8_t>(newl + 1)) << 48);
                p.rq_cand[pos] = cm;
                return true;
            };
            if (wflag) {
                if (enqueue(flag, cand, -1)) label = tc_deferred<K>();
                // queue overflow: the exact decision here, one row at a time
                unsigned fm = __ballot_sync(FULL, flag && label != tc_deferred<K>());
                while (fm) {
                    const int src = __ffs(fm) - 1;
                    fm &= fm - 1;
                    park(__shfl_sync(FULL, row, src));
                    const int best = tcd_refine_row<D, K>(wscr, __shfl_sync(FULL, cand, src), p.c64, p.cn64, cnmax, cmax);
                    __syncwarp();
                    if (lane == src) {
                        label = best;
                        ++refined;
                    }
                }
            }
            if (live && label < K) {
                if (p.labels) p.labels[row] = label;
                if (p.lab8) p.lab8[row] = static_cast<int8_t>(label);
            }
            if (accumulate && p.prev) {
                // changed rows: +x into the new cluster, -x out of the old one,
                // by the refine kernel (queue overflow: REDs here)
                bool ch = label < K && label != oldl;
                if (enqueue(ch, 0ull, label)) ch = false;
                unsigned fm = __ballot_sync(FULL, ch);
                while (fm) {
                    const int src = __ffs(fm) - 1;
                    fm &= fm - 1;
                    park(__shfl_sync(FULL, row, src));
                    const int jn = __shfl_sync(FULL, label, src), jo = __shfl_sync(FULL, oldl, src);
                    for (int f = lane; f < D; f += 32) {
                        const long long qv = __float2ll_rn(wscr[f] * qscale);
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + jn * D + f), static_cast<unsigned long long>(qv));
                        if (jo >= 0)
                            atomicAdd(reinterpret_cast<unsigned long long*>(acc + jo * D + f), static_cast<unsigned long long>(-qv));
                    }
                    if (lane == 0) {
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + KD + jn), 1ull);
                        if (jo >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc + KD + jo), ~0ull);
                    }
                    __syncwarp();
                }
            }
            if (t == 0) TCD_MARK(it, 7);
        }
        if (refined) atomicAdd(p.refined, refined);
        qholes();
        if (accumulate) {
            __threadfence();
            tc::named_sync(15, C::EPI);
            double* out = p.partials + static_cast<int64_t>(blockIdx.x) * (KD + K);
            for (int e = tid; e < KD + K; e += C::EPI) {
                const long long v = __ldcg(acc + e);
                out[e] = e < KD ? ldexp(static_cast<double>(v), -shift) : static_cast<double>(v);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == CTRL) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ------------------------------------------------ full-iteration accumulation
// kmeans_tc_accum_kernel: the per-cluster sums of EVERY row from the final
// labels (lab8), for the full iterations of the tc path: kmeans_tcd_kernel
// (labels only) + the refine kernel (near-ties) decide, then this kernel
// streams X once more.  Chunks of ROWS rows and their labels arrive by 1-D
// bulk copy into a three-stage ring; each chunk is counting-sorted by label in
// shared memory and warp w sums the rows of its clusters (w, w + 16, ...) from
// shared memory into int64 registers kept across all chunks (lanes over the
// features; no atomics).  The sums become the CTA's partial row (f64 of the
// exact integers, summed over CTAs in CTA order as before);
// CTA 0 also clears the refine kernel's row.  Deterministic: static chunk
// assignment, integer sums.
struct TcAccumParams {
    const float* x;
    int64_t n;
    const int8_t* lab8;
    const double* xabs;
    double* partials;   // rows [0, gridDim.x) + the zeroed row gridDim.x
    const int* done;
};

template <int D, int K>
struct TcAccumCfg {
    static constexpr int ROWS = 256, S = 3, THREADS = 512, NW = THREADS / 32;  // 3 x 64 KB stages
    static constexpr int OFF_X = 0;                                   // float [S][ROWS][D]
    static constexpr int OFF_LST = OFF_X + S * ROWS * D * 4;          // u16 [ROWS]
    static constexpr int OFF_LAB = OFF_LST + ROWS * 2;                // int8 [S][ROWS] (bulk-copied with the rows)
    static constexpr int OFF_CNT = (OFF_LAB + S * ROWS + 15) / 16 * 16;  // int [K] counts, [K+1] starts, [K] cursors
    static constexpr int OFF_BAR = (OFF_CNT + (3 * K + 1) * 4 + 15) / 16 * 16;
    static constexpr int SMEM = OFF_BAR + S * 8;
    static_assert(SMEM <= 232448, "shared memory");
};

template <int D, int K>
__global__ void __launch_bounds__(512, 1) kmeans_tc_accum_kernel(TcAccumParams p) {
    using C = TcAccumCfg<D, K>;
    constexpr int KD = K * D, ROWS = C::ROWS, S = C::S, NT = C::THREADS, NW = C::NW;
    constexpr int FPL = (D + 31) / 32;
    if (p.done && *p.done) return;
    extern __shared__ __align__(16) unsigned char asmem[];
    float* xs = reinterpret_cast<float*>(asmem + C::OFF_X);
    unsigned short* lst = reinterpret_cast<unsigned short*>(asmem + C::OFF_LST);
    signed char* lab = reinterpret_cast<signed char*>(asmem + C::OFF_LAB);
    int* cnt = reinterpret_cast<int*>(asmem + C::OFF_CNT);
    int* start = cnt + K;
    int* cur = start + K + 1;
    uint64_t* full = reinterpret_cast<uint64_t*>(asmem + C::OFF_BAR);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int e2 = 0;
    frexp(static_cast<double>(p.n) * (p.xabs ? *p.xabs : 1.0) + 1.0, &e2);
    const int shift = 61 - e2;
    const float qscale = ldexpf(1.f, shift);
    const int64_t nchunks = (p.n + ROWS - 1) / ROWS;
    const int64_t my = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    constexpr int CPW = (K + NW - 1) / NW;  // clusters per warp
    long long acc[CPW][FPL], accn[CPW];
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
        accn[u] = 0;
#pragma unroll
        for (int f = 0; f < FPL; ++f) acc[u][f] = 0;
    }
    if (tid == 0) {
        for (int s = 0; s < S; ++s) tc::mbar_init(&full[s], 1);
        tc::mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int64_t k) {  // chunk k of this CTA into stage k % S
        const int64_t r0 = (blockIdx.x + k * gridDim.x) * ROWS;
        const int64_t nr = min(static_cast<int64_t>(ROWS), p.n - r0);
        const uint32_t bytes = static_cast<uint32_t>(nr * D * 4);
        const uint32_t lbytes = static_cast<uint32_t>((nr + 15) / 16 * 16);  // labels: 16-byte multiple (r0 % 16 == 0)
        const int st = static_cast<int>(k % S);
        tc::mbar_expect_tx(&full[st], bytes + lbytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                tc::smem_u32(xs + st * ROWS * D)),
            "l"(p.x + r0 * D), "r"(bytes), "r"(tc::smem_u32(&full[st]))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                tc::smem_u32(lab + st * ROWS)),
            "l"(p.lab8 + r0), "r"(lbytes), "r"(tc::smem_u32(&full[st]))
            : "memory");
    };
    if (tid == 0)
        for (int64_t k = 0; k < min(my, static_cast<int64_t>(S)); ++k) issue(k);
    for (int64_t k = 0; k < my; ++k) {
        const int st = static_cast<int>(k % S);
        const int64_t r0 = (blockIdx.x + k * gridDim.x) * ROWS;
        const int nr = static_cast<int>(min(static_cast<int64_t>(ROWS), p.n - r0));
        for (int i = tid; i < K; i += NT) cnt[i] = 0;
        const signed char* lb = lab + st * ROWS;
        tc::mbar_wait(&full[st], static_cast<uint32_t>((k / S) & 1));
        __syncthreads();
        for (int i = tid; i < nr; i += NT) {
            const int l = lb[i];
            if (l >= 0 && l < K) atomicAdd(&cnt[l], 1);
        }
        __syncthreads();
        if (warp == 0) {
            int carry = 0;
            for (int b = 0; b < K; b += 32) {
                const int v = b + lane < K ? cnt[b + lane] : 0;
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += t;
                }
                if (b + lane < K) {
                    start[b + lane] = carry + incl - v;
                    cur[b + lane] = carry + incl - v;
                }
                carry += __shfl_sync(FULL, incl, 31);
            }
            if (lane == 0) start[K] = carry;
        }
        __syncthreads();
        for (int i = tid; i < nr; i += NT) {
            const int l = lb[i];
            if (l >= 0 && l < K) lst[atomicAdd(&cur[l], 1)] = static_cast<unsigned short>(i);
        }
        __syncthreads();
        const float* xc = xs + st * ROWS * D;
        // warp w owns clusters w, w + NW, ...: their sorted rows from shared
        // memory into int64 registers kept across chunks (no atomics)
#pragma unroll
        for (int u = 0; u < CPW; ++u) {
            const int j = warp + NW * u;
            if (j >= K) continue;
            const int b0 = start[j], b1 = start[j + 1];
            for (int b = b0; b < b1; b += 8) {
                float xv[8][FPL];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int idx = b + q < b1 ? lst[b + q] : 0;
#pragma unroll
                    for (int f = 0; f < FPL; ++f) {
                        const int ff = lane + 32 * f;
                        xv[q][f] = (ff < D && b + q < b1) ? xc[idx * D + ff] : 0.f;
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int f = 0; f < FPL; ++f) acc[u][f] += __float2ll_rn(xv[q][f] * qscale);
            }
            accn[u] += b1 - b0;
        }
        __syncthreads();  // the stage is read: refill it
        if (tid == 0 && k + S < my) issue(k + S);
    }
    // each warp's clusters -> the CTA's partial row (f64 of the exact int64)
    double* out = p.partials + static_cast<int64_t>(blockIdx.x) * (KD + K);
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
        const int j = warp + NW * u;
        if (j >= K) continue;
#pragma unroll
        for (int f = 0; f < FPL; ++f) {
            const int ff = lane + 32 * f;
            if (ff < D) out[j * D + ff] = ldexp(static_cast<double>(acc[u][f]), -shift);
        }
        if (lane == 0) out[KD + j] = static_cast<double>(accn[u]);
    }
    if (blockIdx.x == 0) {
        double* zr = p.partials + static_cast<int64_t>(gridDim.x) * (KD + K);
        for (int e = tid; e < KD + K; e += NT) zr[e] = 0.0;
    }
}
