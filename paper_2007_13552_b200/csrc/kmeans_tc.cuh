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
                    for (int kb = 0; kb < C::NKB; ++kb) tc::tma_load_2d(dst + kb * PR * 32, &map, &full[st], kb * 32, prow);
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

template <int D, int K>
__host__ __device__ constexpr int tc_refine_threads() { return 512; }

// rows are accumulated in a per-CTA shared int64 copy first (global atomics
// on the K*D sums from every warp contended at L2: 200 us per launch at cfg3),
// then the CTA adds its nonzero entries to racc once
template <int D, int K>
__global__ void __launch_bounds__(512) kmeans_tc_refine_kernel(TcRefineParams p) {
    constexpr int KD = K * D, WPB = tc_refine_threads<D, K>() / 32;
    __shared__ float rows[WPB][D];
    __shared__ long long sacc[KD + K];
    __shared__ bool last;
    for (int e = threadIdx.x; e < KD + K; e += blockDim.x) sacc[e] = 0ll;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool skip = p.done && *p.done;
    const unsigned count = skip ? 0u : min(p.ctl[0], p.cap);
    int e2 = 0;
    frexp(static_cast<double>(p.n) * (p.xabs ? *p.xabs : 1.0) + 1.0, &e2);
    const int shift = 61 - e2;
    const float qscale = ldexpf(1.f, shift);
    const float cmax = p.bounds[0], cnmax = p.bounds[1];
    float* row = rows[warp];
    constexpr int FPL = (D + 31) / 32;
    // the next entry is loaded while this one is decided (the queue is
    // contiguous and L2-resident: it was written by the tc kernel just before)
    auto fetch = [&](unsigned ee, uint64_t& v, uint64_t& c, float (&xv)[FPL]) {
        v = p.qrow[ee];
        c = p.qcand[ee];
        // the row from the queue, or (queues without rows) gathered from X
        const float* src = p.qx ? p.qx + static_cast<int64_t>(ee) * D
                                : (v == TC_QHOLE ? nullptr : p.x + static_cast<int64_t>(v & ((1ull << 48) - 1)) * D);
#pragma unroll
        for (int u = 0; u < FPL; ++u) {
            const int f = lane + 32 * u;
            xv[u] = (f < D && src) ? src[f] : 0.f;
        }
    };
    const unsigned stride = gridDim.x * WPB;
    unsigned e = blockIdx.x * WPB + warp;
    uint64_t v = 0, cm = 0;
    unsigned nref = 0;  // entries decided here (the rest only accumulate)
    float xa[FPL];
    if (e < count) fetch(e, v, cm, xa);
    for (; e < count; e += stride) {
        uint64_t vn = 0, cn = 0;
        float xn[FPL];
        if (e + stride < count) fetch(e + stride, vn, cn, xn);
#pragma unroll
        for (int u = 0; u < FPL; ++u)
            if (lane + 32 * u < D) row[lane + 32 * u] = xa[u];
        __syncwarp();
        if (v == TC_QHOLE) {
            v = vn;
            cm = cn;
#pragma unroll
            for (int u = 0; u < FPL; ++u) xa[u] = xn[u];
            continue;
        }
        const int64_t r = static_cast<int64_t>(v & ((1ull << 48) - 1));
        const int old = static_cast<int>(static_cast<int8_t>(static_cast<uint8_t>(v >> 56)));
        const int dec = static_cast<int>((v >> 48) & 0xff) - 1;  // decided label (changed row) or -1
        int best = dec;
        if (dec < 0) {
            best = tc_refine_warp<D, K>(row, cm, p.c64, p.cn64, cnmax, cmax, nullptr);
            ++nref;
            if (lane == 0) {
                if (p.labels) p.labels[r] = best;
                if (p.lab8) p.lab8[r] = static_cast<int8_t>(best);
            }
        }
        __syncwarp();
        if (p.partial && best != old) {
            for (int f = lane; f < D; f += 32) {
                const long long qv = __float2ll_rn(row[f] * qscale);
                atomicAdd(reinterpret_cast<unsigned long long*>(sacc + best * D + f), static_cast<unsigned long long>(qv));
                if (old >= 0)
                    atomicAdd(reinterpret_cast<unsigned long long*>(sacc + old * D + f), static_cast<unsigned long long>(-qv));
            }
            if (lane == 0) {
                atomicAdd(reinterpret_cast<unsigned long long*>(sacc + KD + best), 1ull);
                if (old >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(sacc + KD + old), ~0ull);
            }
        }
        __syncwarp();
        v = vn;
        cm = cn;
#pragma unroll
        for (int u = 0; u < FPL; ++u) xa[u] = xn[u];
    }
    if (lane == 0 && nref) atomicAdd(p.refined, static_cast<unsigned long long>(nref));
    __syncthreads();
    if (p.partial && blockIdx.x * WPB < count) {
        for (int e = threadIdx.x; e < KD + K; e += blockDim.x)
            if (sacc[e]) atomicAdd(reinterpret_cast<unsigned long long*>(p.racc + e), static_cast<unsigned long long>(sacc[e]));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(p.ctl + 1, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int e = threadIdx.x; e < KD + K; e += blockDim.x) {
        const long long v = static_cast<long long>(atomicExch(reinterpret_cast<unsigned long long*>(p.racc + e), 0ull));
        if (p.partial) p.partial[e] = e < KD ? ldexp(static_cast<double>(v), -shift) : static_cast<double>(v);
    }
    if (threadIdx.x == 0) {
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
                for (int kb = 0; kb < C::NKB; ++kb) tc::tma_load_2d(dst + kb * PR * 32, &map, &full[st], kb * 32, prow);
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
