// kmeans_persist.cuh -- the whole Lloyd loop of a small-(D, K) k-means fit in
// ONE cooperative launch (BASELINE config 1: 5M x 18 fp32, k = 8, 20 iterations).
// Included by kmeans.cu (shares its helpers).
//
// Reference: kmeans_fit's loop body (cluster.cpp:105-151) over assign_local
// (:44-56) and cdist_xy (pairwise.cpp:87-100); the per-iteration allreduce of
// sums/counts (:123, transport.hpp:136-148) becomes a grid barrier plus, with
// world > 1, an NVLink exchange between the ranks' kernels.
//
// Why one launch: one cfg1 iteration streams 360 MB (55.8 us at the measured
// copy bandwidth).  A launch per iteration paid a tail, a table-copy node and a
// relaunch gap every iteration.  Here every CTA keeps a private copy of the
// Lloyd state (f64 master centroids, reference-order |c|^2, running sums, the
// fp32 score table) in shared memory; after each grid barrier every CTA
// applies the same update to the same folded stats, so the copies stay
// bit-identical without a broadcast.  The TMA ring is never drained between
// iterations: X does not change, so a CTA that has no tile left in iteration
// i already streams its first tiles of iteration i + 1 while the grid waits.
//
// Tile schedule per iteration (measured, profiles/: with a fully static
// schedule the CTAs finished their equal shares between 52 and 85 us -- HBM
// does not serve the SMs evenly): CTA b first takes the static tiles
// b + j G (j < J0, about 70% of the work, no atomics, prefetchable across the
// barrier), then grabs the rest dynamically from a per-iteration counter.
// Which CTA adds which rows therefore varies from run to run, so the sums are
// made ORDER-INDEPENDENT: every row's contribution (delta iterations) or every
// tile's f64 run sum (full iterations) is rounded to int64 fixed point at
// 2^-(61-e) with n max|x| < 2^e (2^-38 at cfg1, far below the f64 rounding of
// the sums themselves) and added as integers -- the fit is bit-identical from
// run to run.  The rows' int8 labels live in HBM, two buffers by
// iteration parity (written in i, read as "previous" in i + 1, fetched with the
// tile by the same bulk copy, or right after the barrier for a tile that was
// prefetched across it).
//
// Per-iteration protocol (S = k*m + k stats):
//   tiles    -> CTA int64 partials -> atomicAdd into acc[it % 3] (integer adds commute)
//   barrier  world == 1: arrival counter reaches G (it + 1), every CTA reads
//            acc[it % 3] from L2.  world > 1: the last CTA to arrive converts
//            and stores the rank's stats into every rank's exchange region over
//            NVLink, then releases one flag per rank; every CTA of every rank
//            waits for all ranks' flags in its own region (bounded: ~20 s, then
//            flags[3] = timeout instead of a trap) and folds ranks 0..p-1 in
//            order itself -- one NVLink hop, no second release word.
//   update   every CTA: running sums (+= changes in delta iterations),
//            c_j = S_j / n_j or kept when empty (cluster.cpp:125-133), reference
//            order |c_j|^2, fp32 table, the fp32 error-bound inputs; CTA 0
//            writes the inertia trace, displacement and iteration count.
// acc[(it+1) % 3] is zeroed by CTA 0 at the start of iteration it (its last
// readers passed barrier it-1; its first writers wait for barrier it).
#pragma once

// -DDNDC_CHECKS: device-side bounds checks of the persistent kernel (labels,
// tiles, queue slots, accumulator indices) for the checked build that
// tools/sanitize_smoke.py runs (compute-sanitizer is closed on this pool)
#ifdef DNDC_CHECKS
#define PCHECK(cond)                                                                              \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("PCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x, #cond);                                                           \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define PCHECK(cond) \
    do {             \
    } while (0)
#endif

namespace persist {
// SCR: changed rows a warp queues (values + labels) before it moves them
// between the clusters' sums in one pass (the per-row cost of small batches
// was ~70 issue slots per changed row, r2 ncu)
constexpr int THREADS = 128, W = THREADS / 32, SCR = 32;
// tensor-core scores (TCS instantiations): MMA N (K centroids padded to 16),
// TMEM columns per CTA (4 CTAs per SM share the 512)
constexpr int TC_NS = 16, TC_COLS = 128;
// MODE of an instantiation: iterations that accumulate every row (full), only
// the rows whose label changed (delta), or both in one launch
enum { BOTH = 0, FULL_ONLY = 1, DELTA_ONLY = 2 };
}

struct PersistParams {
    const float* x;
    int64_t n;                   // rows of this rank's shard
    int max_iter, full_iters;
    int it_begin, it_end;        // this launch runs iterations [it_begin, it_end)
    double tol;
    const double* c64_init;      // centroids before iteration it_begin (k*m)
    double* c64_out;             // centroids after the last iteration run (may alias c64_init)
    double* run_io;              // running sums/counts [S]: read at it_begin (delta), written at the end
    double* trace;               // [max_iter] inertia
    double* disp;                // [max_iter] max centroid displacement
    int* flags;                  // [0] stopped early, [1] iterations run, [2] invalid input, [3] timeout
    const double* sx2;           // [2] global sum |x|^2, [3] max |x| of the shard
    unsigned long long* acc;     // 3 x S fixed-point accumulators (zero at launch)
    unsigned* arrive;            // [33] grid arrival: root + 32 group counters (zero at launch)
    unsigned* go;                // world > 1: iterations released by the finaliser (zero at launch)
    double* gstats;              // world > 1: 2 x S rank-folded stats
    unsigned long long* refined; // rows re-decided in f64 (all iterations)
    int world, rank;
    void* const* peers;          // world > 1: exchange regions of every rank (NVLink)
    int8_t* labels;              // [n] each row's label, updated in place (delta: changed rows only)
    unsigned* tile_ctr;          // [max_iter] dynamic tile counters (zero at launch)
    int static_tiles;            // J0: static tiles per CTA per iteration
    // optional %globaltimer trace (DNDC_PERSIST_TRACE): per iteration and CTA
    // [0] tiles done, [1] barrier passed; per iteration (CTA 0) [2] start, [3] update done
    unsigned long long* trace_marks;
    int trace_grid;  // row stride of trace_marks: 2 * trace_grid + 2 per iteration
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// The barrier of one virtual CTA: the whole CTA (WG = 1) or warpgroup wg of
// a WG-warpgroup CTA (named barrier 1 + wg) -- see kmeans_persist_kernel.
template <int WG>
__device__ __forceinline__ void persist_sync(int wg) {
    if constexpr (WG == 1) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(wg + 1), "r"(persist::THREADS) : "memory");
    }
}

struct PersistLayout {
    int tiles, slab, wacc, scr, scl, cnt, tab, bop, run, c64, cn64, misc, stile, siter, sdef, lcnt, consumed, bars,
        lbars, total;
};

template <int D, int K, int R, int NST, bool TCS = false>
__host__ __device__ constexpr PersistLayout persist_layout() {
    using namespace persist;
    constexpr int KD = K * D, S = KD + K, TILE = THREADS * R, VW = W * R;
    PersistLayout l{};
    int o = 0;
    auto take = [&](int bytes) {
        const int at = o;
        o = (o + bytes + 15) / 16 * 16;
        return at;
    };
    l.tiles = take(NST * TILE * D * 4);
    l.slab = take(NST * TILE);           // previous labels of each staged tile
    l.wacc = take(W * KD * 8);           // int64 per-warp changes (delta iterations)
    l.scr = take(W * SCR * D * 4 > (KD + K) * 8 ? W * SCR * D * 4 : (KD + K) * 8);  // also old c / |c|^2 in the update
    l.scl = take(W * 2 * SCR * 4);
    l.cnt = take(VW * K * 4);
    l.tab = take((K * D + K) * 4);
    // TCS: the centroid operand -2c as tf32 hi then lo, K-major SWIZZLE_NONE
    // core matrices of 8 rows x 16 B: chunk c (4 features) of rows 0..7 at
    // c * 128 B, TC_BSTRIDE bytes per part.  The MMA's second 8-row group
    // (N = 16 > K) reads the next TC_BSTRIDE bytes (hi: the lo part; lo: the
    // start of `run`) -- score columns >= K are never read, so those rows need
    // no zeros of their own (and cost no shared memory: 4 CTAs per SM fit)
    l.bop = TCS ? take(2 * (D + 7) / 8 * 8 / 4 * 128) : o;
    l.run = take(S * 8);
    l.c64 = take(KD * 8);
    l.cn64 = take(K * 8);
    l.misc = take(16 * 8);
    l.stile = take(NST * 8);
    l.siter = take(NST * 4);
    l.sdef = take(NST * 4);
    l.lcnt = take(NST * 4);
    l.consumed = take(NST * 4);
    l.bars = take(NST * 8);
    l.lbars = take(NST * 8);
    l.total = o;
    return l;
}

__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// fp32 top-2 of R rows against the table in shared memory, clusters in pairs:
// T[p*2D + 2f + (j&1)] = -2 c_j,f for the pair p = j/2 (one LDS.128 = two
// features of both clusters), T[K*D + j] = |c_j|^2.  A pair's two scores
// accumulate in one float2: FFMA2 with the feature x_f as a broadcast scalar
// operand and the (|c_j|^2, |c_j+1|^2) pair as the first addend -- no
// accumulator moves, no combining add.  s_j = |c_j|^2 + sum_f x_f (-2 c_j,f)
// is one sequential fp32 chain of D FMAs (the error bound's model).
template <int D, int K, int R>
__device__ __forceinline__ void persist_top2(const float2 (&xv)[R][D / 2], const float* __restrict__ T,
                                             float (&b1)[R], float (&b2)[R], int (&i1)[R]) {
    static_assert(K % 2 == 0 && D % 2 == 0, "cluster pairs, feature pairs");
    constexpr int L = D / 2;
#pragma unroll
    for (int h = 0; h < R; ++h) {
        b1[h] = FLT_MAX;
        b2[h] = FLT_MAX;
        i1[h] = 0;
    }
#pragma unroll
    for (int pr = 0; pr < K / 2; ++pr) {
        const float2 cn = *reinterpret_cast<const float2*>(T + K * D + 2 * pr);
        float2 sp[R];
#pragma unroll
        for (int h = 0; h < R; ++h) sp[h] = cn;
#pragma unroll
        for (int g = 0; g < L; ++g) {
            const float4 c = *reinterpret_cast<const float4*>(T + pr * 2 * D + 4 * g);
#pragma unroll
            for (int h = 0; h < R; ++h) {
                sp[h] = __ffma2_rn(make_float2(xv[h][g].x, xv[h][g].x), make_float2(c.x, c.y), sp[h]);
                sp[h] = __ffma2_rn(make_float2(xv[h][g].y, xv[h][g].y), make_float2(c.z, c.w), sp[h]);
            }
        }
#pragma unroll
        for (int h = 0; h < R; ++h) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float sc = u ? sp[h].y : sp[h].x;
                const bool lt = sc < b1[h];
                b2[h] = fminf(b2[h], fmaxf(b1[h], sc));
                b1[h] = fminf(b1[h], sc);
                i1[h] = lt ? 2 * pr + u : i1[h];
            }
        }
    }
}

// The same top-2 with the K*D score products on the tensor core (TCS
// instantiations).  Every thread writes its R rows into tensor memory (lane =
// row of the 128-row half h; the raw fp32 is the tf32 hi part -- the tensor
// core truncates -- and lo = x - trunc(x); KCP = D padded to the K = 8 step,
// padding columns zero), then one warp issues, per half, the 3xTF32 MMAs
// hi.Bhi + hi.Blo + lo.Bhi with A from TMEM (kmeans_tcd_kernel's scheme:
// shared memory carries only B = -2c) and every thread reads its rows' K
// scores back (tcgen05.ld) and adds |c_j|^2 in fp32.  Error bound per row
// (kmeans_tcd_kernel's model): tau = 4 (3 KCP 2^-24 + 3 2^-20)
// (max|c|^2 + 2 |x| max|c|).  Replaces 72 FFMA2 and ~25 table loads per row
// by ~40 instructions; the CTA waits for its MMAs once per tile (the other
// CTAs of the SM fill the gap).
template <int D, int K, int R, int WG>
__device__ __forceinline__ void persist_top2_tc(const float2 (&xv)[R][D / 2], const float* __restrict__ T,
                                                uint32_t tmem, uint64_t bh, uint64_t bl, uint64_t* tbar,
                                                uint32_t& tph, float cnmax, float cmax, float (&b1)[R],
                                                float (&b2)[R], int (&i1)[R], float (&tau)[R], int wg) {
    using namespace persist;
    constexpr int L = D / 2, KCP = (D + 7) / 8 * 8, DCOL = R * 2 * KCP;
    static_assert(K <= 8 && DCOL + R * TC_NS <= TC_COLS, "persistent tc scores: TMEM columns");
    constexpr float ERR = 4.f * (static_cast<float>(3 * KCP) * 0x1.0p-24f + 3.f * 0x1.0p-20f);
    const int warp = (threadIdx.x >> 5) & 3;  // TMEM lane quarter = warp within the warpgroup
    const uint32_t lanes = static_cast<uint32_t>(warp * 32) << 16;
#pragma unroll
    for (int h = 0; h < R; ++h) {
        float2 q = make_float2(0.f, 0.f);
#pragma unroll
        for (int f = 0; f < L; ++f) q = __ffma2_rn(xv[h][f], xv[h][f], q);
        tau[h] = ERR * (cnmax + 2.f * sqrtf(q.x + q.y) * cmax);
        const uint32_t ahi = tmem + lanes + static_cast<uint32_t>(h * 2 * KCP), alo = ahi + KCP;
#pragma unroll
        for (int g = 0; g < KCP; g += 8) {
            float hv[8], lv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = g + i;
                const float v = c < D ? ((c & 1) ? xv[h][c / 2].y : xv[h][c / 2].x) : 0.f;
                hv[i] = v;
                lv[i] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            }
            tc::tmem_st8(ahi + g, hv);
            tc::tmem_st8(alo + g, lv);
        }
    }
    tc::tmem_st_wait();
    tc::tc_fence_before();
    persist_sync<WG>(wg);
    if (warp == 0) {
        tc::tc_fence_after();
        constexpr uint32_t idesc = tc::idesc_tf32(128, TC_NS, 0, 0);
#pragma unroll
        for (int h = 0; h < R; ++h)
#pragma unroll
            for (int ks = 0; ks < KCP / 8; ++ks)  // descriptor start address: 16-byte units
                tc::mma3_tf32_ta_elect(tmem + DCOL + h * TC_NS, tmem + h * 2 * KCP + ks * 8,
                                       tmem + h * 2 * KCP + KCP + ks * 8, bh + static_cast<uint64_t>(ks * 16),
                                       bl + static_cast<uint64_t>(ks * 16), idesc, ks > 0);
        tc::mma_commit_elect(tbar);
    }
    tc::mbar_wait(tbar, tph);  // plain poll (the suspend-hint wait is for TMA completions)
    tph ^= 1u;
    tc::tc_fence_after();
    float v[R][8];
    if constexpr (R == 2) {
        tc::tmem_ld8x2(tmem + lanes + DCOL, tmem + lanes + DCOL + TC_NS, v[0], v[1]);
    } else {
#pragma unroll
        for (int h = 0; h < R; ++h) tc::tmem_ld8(tmem + lanes + DCOL + h * TC_NS, v[h]);
    }
    tc::tc_fence_before();
#pragma unroll
    for (int h = 0; h < R; ++h) {
        b1[h] = FLT_MAX;
        b2[h] = FLT_MAX;
        i1[h] = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const float sc = T[K * D + j] + v[h][j];
            const bool lt = sc < b1[h];
            b2[h] = fminf(b2[h], fmaxf(b1[h], sc));
            b1[h] = fminf(b1[h], sc);
            i1[h] = lt ? j : i1[h];
        }
    }
}

// Tables of the current centroids c64 (shared memory), thread j < K (K <= 32:
// all in warp 0): reference-order |c_j|^2 (pairwise.cpp:13-18), the fp32 score
// table and the error-bound inputs (misc[0] max |c|, misc[1] max fp32 |c|^2).
// TCS: also the MMA operand B = -2c (rows j < K of bhi / blo; the padding
// rows and columns stay zero) for persist_top2_tc, made visible to the
// tensor core (async proxy) before the caller's barrier.
template <int D, int K>
__device__ __forceinline__ void persist_tables(const double* c64, double* cn64, float* tab, double* misc,
                                               float* bhi = nullptr, float* blo = nullptr) {
    const int j = threadIdx.x % persist::THREADS;  // thread of the (virtual) CTA
    double cmax = 0.0, cnmax = 0.0;
    if (j < K) {
        double n64 = 0.0, n32 = 0.0;
        for (int f = 0; f < D; ++f) {
            const double cf = c64[j * D + f];
            n64 = add_rn(n64, mul_rn(cf, cf));
            const float c32 = static_cast<float>(cf);
            tab[(j / 2) * 2 * D + 2 * f + (j & 1)] = -2.f * c32;  // cluster-pair layout (persist_top2)
            if (bhi) {  // persist_layout's bop (j < K <= 8: the first 8-row group)
                const float v = -2.f * c32;
                const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
                const int off = (f / 4) * 32 + j * 4 + (f % 4);
                bhi[off] = hi;
                blo[off] = v - hi;
            }
            n32 += static_cast<double>(c32) * static_cast<double>(c32);
        }
        if (bhi) tc::fence_async_smem();
        tab[K * D + j] = static_cast<float>(n32);
        cn64[j] = n64;
        cmax = sqrt(n32);
        cnmax = static_cast<double>(static_cast<float>(n32));
    }
    if (j < 32) {
        cmax = warp_max(cmax);
        cnmax = warp_max(cnmax);
        if (j == 0) {
            misc[0] = static_cast<double>(static_cast<float>(cmax) * (1.f + 0x1.0p-20f));
            misc[1] = static_cast<double>(static_cast<float>(cnmax) * (1.f + 0x1.0p-20f));
        }
    }
}

// WG > 1: one CTA of WG warpgroups per SM, each warpgroup one virtual CTA of
// the algorithm above (its own shared-memory block, tiles, state copy and
// named barrier; virtual block id blockIdx.x * WG + wg).  The tensor-core
// score instantiations need it: a kernel that uses tcgen05 is resident one
// CTA per SM, and the four virtual CTAs share the SM's 512 TMEM columns.
template <int D, int K, int R, int NST, int MINB, int MODE, bool TCS = false, int WG = 1>
__global__ void __launch_bounds__(persist::THREADS * WG, WG == 1 ? MINB : 1) kmeans_persist_kernel(PersistParams p) {
    using namespace persist;
    static_assert(D % 2 == 0 && D <= 64 && K <= 32, "persistent kernel shape");
    constexpr int TILE = THREADS * R, VW = W * R;
    constexpr int L = D / 2;                 // lanes per row in the run sums (float2 each)
    constexpr int GR = L <= 32 ? 32 / L : 1; // rows summed in parallel per warp
    constexpr int KD = K * D, S = KD + K;
    constexpr int JW = (K + W - 1) / W;      // clusters owned per warp in the run sums
    constexpr PersistLayout LY = persist_layout<D, K, R, NST, TCS>();

    extern __shared__ __align__(16) unsigned char smem_base[];
    const int wg = WG == 1 ? 0 : static_cast<int>(threadIdx.x) / THREADS;
    unsigned char* smem_raw = smem_base + wg * LY.total;
    float* tiles = reinterpret_cast<float*>(smem_raw + LY.tiles);
    int8_t* slab = reinterpret_cast<int8_t*>(smem_raw + LY.slab);
    long long* wacc = reinterpret_cast<long long*>(smem_raw + LY.wacc);
    float* scr = reinterpret_cast<float*>(smem_raw + LY.scr);
    int* scl = reinterpret_cast<int*>(smem_raw + LY.scl);
    int* cnt = reinterpret_cast<int*>(smem_raw + LY.cnt);
    float* tab = reinterpret_cast<float*>(smem_raw + LY.tab);
    double* run = reinterpret_cast<double*>(smem_raw + LY.run);
    double* c64s = reinterpret_cast<double*>(smem_raw + LY.c64);
    double* cn64s = reinterpret_cast<double*>(smem_raw + LY.cn64);
    double* misc = reinterpret_cast<double*>(smem_raw + LY.misc);
    volatile long long* stile = reinterpret_cast<volatile long long*>(smem_raw + LY.stile);
    volatile int* siter = reinterpret_cast<volatile int*>(smem_raw + LY.siter);
    volatile int* sdef = reinterpret_cast<volatile int*>(smem_raw + LY.sdef);
    volatile int* lcnt = reinterpret_cast<volatile int*>(smem_raw + LY.lcnt);  // deferred label loads per stage
    unsigned* consumed = reinterpret_cast<unsigned*>(smem_raw + LY.consumed);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + LY.bars);
    uint64_t* lbars = reinterpret_cast<uint64_t*>(smem_raw + LY.lbars);
    constexpr int BPART = (D + 7) / 8 * 8 / 4 * 128;  // bytes of one part (hi or lo) of the MMA operand
    float* bhi = TCS ? reinterpret_cast<float*>(smem_raw + LY.bop) : nullptr;
    float* blo = TCS ? reinterpret_cast<float*>(smem_raw + LY.bop + BPART) : nullptr;
    double* cold = reinterpret_cast<double*>(scr);  // update only: previous centroids [KD] and |c|^2 [K]
    double* cnold = cold + KD;
    int* s_last = reinterpret_cast<int*>(misc + 8);
    volatile int* s_tmo = reinterpret_cast<volatile int*>(misc + 8) + 1;  // this CTA timed out at a barrier
    uint64_t* tbar = reinterpret_cast<uint64_t*>(misc + 4);    // TCS: MMA completion
    uint32_t* tslot = reinterpret_cast<uint32_t*>(misc + 5);   // TCS: TMEM base address
    // the producer's position: iteration being grabbed and its next static index
    volatile int* s_git = reinterpret_cast<volatile int*>(misc + 12);
    volatile int* s_gj = reinterpret_cast<volatile int*>(misc + 12) + 1;

    const int tid = static_cast<int>(threadIdx.x) % THREADS, warp = tid >> 5, lane = tid & 31;
    const int vb = static_cast<int>(blockIdx.x) * WG + wg;  // virtual block
    const int G = static_cast<int>(gridDim.x) * WG;
    const int64_t ntiles = ceil_div(p.n, TILE);
    const int J0 = p.static_tiles;                       // static tiles of every CTA
    const int64_t nstatic = static_cast<int64_t>(J0) * G;  // tiles [0, nstatic) are static

    if constexpr (TCS) {
        if (threadIdx.x < 32) tc::tmem_alloc(tslot, TC_COLS * WG);  // warpgroup 0's slot
        for (int e = tid; e < 2 * BPART / 4; e += THREADS) bhi[e] = 0.f;  // padding features
    }
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&lbars[s], 1);
        }
        if (TCS) mbar_init(tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        *s_git = p.it_begin;
        *s_gj = 0;
        *s_tmo = 0;
    }
    if (tid < NST) {
        consumed[tid] = 0u;
        sdef[tid] = 0;
        lcnt[tid] = 0;
    }
    for (int e = tid; e < KD; e += THREADS) c64s[e] = p.c64_init[e];
    if (MODE == DELTA_ONLY)
        for (int e = tid; e < S; e += THREADS) run[e] = p.run_io[e];
    if (TCS) tc::tc_fence_before();
    __syncthreads();  // the whole CTA (every warpgroup)
    if (TCS) tc::tc_fence_after();
    // this warpgroup's TMEM columns
    const uint32_t tmem =
        TCS ? *reinterpret_cast<const uint32_t*>(smem_base + (reinterpret_cast<unsigned char*>(tslot) - smem_raw)) +
                  static_cast<uint32_t>(wg * TC_COLS)
            : 0u;
    persist_tables<D, K>(c64s, cn64s, tab, misc, bhi, blo);
    // TCS: the MMA operand descriptors (fixed addresses) and the barrier phase
    // (LBO: the two 16-byte K chunks of a K = 8 step; SBO: the 8-row groups)
    const uint64_t bh_desc = TCS ? tc::smem_desc(tc::smem_u32(bhi), 128, BPART) : 0ull;
    const uint64_t bl_desc = TCS ? tc::smem_desc(tc::smem_u32(blo), 128, BPART) : 0ull;
    uint32_t tph = 0u;
    // fixed-point scale of the sums: n max|x| < 2^e
    const double xabs = p.sx2[3];
    int e2 = 0;
    frexp(static_cast<double>(p.n) * xabs + 1.0, &e2);
    const int shift = 61 - e2;
    const float xabs_f = static_cast<float>(xabs);
    const float qscale = ldexpf(1.f, shift);  // exact power of two (shift <= 61 < 127)

    // Fills stage s with the producer's next tile: the static ones of the grab
    // iteration first, then the dynamic counter; past the last tile of the
    // iteration it moves to the next one.  `cur` is the caller's iteration:
    // a tile of a later iteration gets its previous labels only after the
    // barrier (sdef), since they are still being written.  Called by one
    // thread at a time, in load order (stage releases are ordered).
    auto issue = [&](int s, int cur) {
        int git = *s_git;
        int64_t tile = -1;
        while (git < p.it_end) {
            const int j = *s_gj;
            if (j < J0) {
                const int64_t t = vb + static_cast<int64_t>(j) * G;
                *s_gj = j + 1;
                if (t < ntiles) {
                    tile = t;
                    break;
                }
                continue;
            }
            const int64_t t = nstatic + atomicAdd(p.tile_ctr + git, 1u);
            if (t < ntiles) {
                tile = t;
                break;
            }
            ++git;
            *s_git = git;
            *s_gj = 0;
        }
        PCHECK(tile < ntiles && git <= p.it_end);
        stile[s] = tile;
        siter[s] = git;
        if (tile < 0) {  // nothing left in the fit: an empty stage ends the consumer's loop
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
            return;
        }
        const int64_t rows = min(static_cast<int64_t>(TILE), p.n - tile * TILE);
        const bool want_lab = MODE == DELTA_ONLY || (MODE == BOTH && git >= p.full_iters);  // delta: previous labels
        if (want_lab && git <= cur) {
            bulk_load2(tiles + s * TILE * D, p.x + tile * TILE * D, static_cast<uint32_t>(rows * D * 4),
                       slab + s * TILE, p.labels + tile * TILE,
                       static_cast<uint32_t>(rows), &bars[s]);
        } else {
            bulk_load(tiles + s * TILE * D, p.x + tile * TILE * D, static_cast<uint32_t>(rows * D * 4), &bars[s]);
            if (want_lab) sdef[s] = 1;  // fetched after barrier git - 1
        }
    };
    auto issue_labels = [&](int s) {  // the deferred previous labels of stage s
        const int git = siter[s];
        const int64_t tile = stile[s];
        const int64_t rows = min(static_cast<int64_t>(TILE), p.n - tile * TILE);
        int8_t* dst = slab + s * TILE;
        const int8_t* src = p.labels + tile * TILE;
        const uint32_t body = static_cast<uint32_t>(rows) & ~15u;
        for (uint32_t b = body; b < static_cast<uint32_t>(rows); ++b) dst[b] = src[b];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        lcnt[s] = lcnt[s] + 1;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&lbars[s])), "r"(body)
                     : "memory");
        if (body)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(dst)),
                "l"(src), "r"(body), "r"(smem_u32(&lbars[s]))
                : "memory");
    };
    if (tid == 0)
        for (int s = 0; s < NST; ++s) issue(s, p.it_begin);
    persist_sync<WG>(wg);

    const bool invalid = p.flags[0] != 0;  // invalid input, or converged in an earlier launch
    // exchange epoch before this launch's first iteration (read before barrier 0)
    const unsigned long long xbase = p.world > 1 ? *(xchg_flags(p.peers[p.rank], p.world) + p.world) : 0ull;
    unsigned long long refined = 0;
    int64_t g = 0;  // stages consumed so far (stage g % NST, phase (g / NST) & 1)
    const int gq = lane / L, q = lane % L;
    bool stop = invalid;
    for (int it = p.it_begin; it < p.it_end && !stop; ++it) {
        const bool full = MODE == FULL_ONLY || (MODE == BOTH && it < p.full_iters);
        const int TG = p.trace_grid;
        unsigned long long* tm = p.trace_marks ? p.trace_marks + static_cast<int64_t>(it) * (2 * TG + 2) : nullptr;
        if (tm && vb == 0 && tid == 0) tm[2 * TG] = gtimer();
        const float tau = 4.f * static_cast<float>(D + 3) * 0x1.0p-24f *
                          (static_cast<float>(misc[1]) +
                           2.f * sqrtf(static_cast<float>(D)) * xabs_f * static_cast<float>(misc[0]));
        const float cnmax_f = static_cast<float>(misc[1]), cmax_f = static_cast<float>(misc[0]);
        if (!full)
            for (int e = tid; e < W * KD; e += THREADS) wacc[e] = 0ll;
        if (vb == 0 && it >= 1)
            for (int e = tid; e < S; e += THREADS) p.acc[((it + 1) % 3) * S + e] = 0ull;
        persist_sync<WG>(wg);

        long long count_acc = 0;
        int cnt_delta = 0;
        long long wsum[JW][2];
#pragma unroll
        for (int jj = 0; jj < JW; ++jj) wsum[jj][0] = wsum[jj][1] = 0ll;
        int8_t* lab_out = p.labels;
        int qn = 0;  // rows in this warp's change queue (warp-uniform)
        auto flush_queue = [&]() {
            __syncwarp();
            const float* wscr = scr + warp * SCR * D;
            const int* wscl = scl + warp * 2 * SCR;
            long long* acc = wacc + warp * KD;
            for (int c = 0; c < qn; ++c) {
                const int nl = wscl[2 * c], ol = wscl[2 * c + 1];
                PCHECK(nl >= 0 && nl < K && ol >= -1 && ol < K && nl != ol);
                if (lane < K) cnt_delta += (lane == nl) - (lane == ol);
#pragma unroll
                for (int f = lane; f < D; f += 32) {
                    const long long v = __float2ll_rn(wscr[c * D + f] * qscale);
                    acc[nl * D + f] += v;
                    if (ol >= 0) acc[ol * D + f] -= v;
                }
            }
            __syncwarp();
        };

        for (;; ++g) {
            const int s = static_cast<int>(g % NST);
            float* xt = tiles + s * TILE * D;
            mbar_wait(&bars[s], static_cast<uint32_t>((g / NST) & 1));
            const int64_t tile = stile[s];
            if (tile < 0 || siter[s] != it) break;  // this CTA has no tile left in iteration it
            const int64_t row0 = tile * TILE;
            float2 xv[R][L];
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const int row = tid + h * THREADS;
#pragma unroll
                for (int f = 0; f < L; ++f) xv[h][f] = *reinterpret_cast<const float2*>(xt + row * D + 2 * f);
            }
            if (!full) {
                // ---- delta iteration: rows in registers, stage handed back at once
                if (sdef[s]) mbar_wait(&lbars[s], static_cast<uint32_t>((lcnt[s] - 1) & 1));
                int prevl[R], label[R];
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const int row = tid + h * THREADS;
                    prevl[h] = row0 + row < p.n ? static_cast<int>(slab[s * TILE + row]) : -1;
                    PCHECK(prevl[h] >= -1 && prevl[h] < K);
                }
                __threadfence_block();
                __syncwarp();
                if (lane == 0) {
                    const unsigned done = atomicAdd(&consumed[s], 1u);
                    if (done == W - 1) {
                        consumed[s] = 0u;
                        sdef[s] = 0;
                        issue(s, it);
                    }
                }
                float b1[R], b2[R], tr[R];
                int i1[R];
#ifdef KP_EXP_STREAM
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
                if constexpr (TCS) {
                    persist_top2_tc<D, K, R, WG>(xv, tab, tmem, bh_desc, bl_desc, tbar, tph, cnmax_f, cmax_f, b1, b2, i1, tr, wg);
                } else {
                    persist_top2<D, K, R>(xv, tab, b1, b2, i1);
#pragma unroll
                    for (int h = 0; h < R; ++h) tr[h] = tau;
                }
#endif
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const int row = tid + h * THREADS;
                    const int64_t gr = row0 + row;
                    label[h] = K;
                    if (gr < p.n) {
                        label[h] = i1[h];
                        if (K > 1 && !(b2[h] - b1[h] > tr[h])) {
                            // the stage may be refilled already: the row from global (L2)
                            label[h] = ref_argmin<float>(p.x + gr * D, D, c64s, cn64s, K);
                            ++refined;
                        }
                        if (label[h] != prevl[h]) lab_out[gr] = static_cast<int8_t>(label[h]);
                    }
                }
                // changed rows: queued per warp (values + labels), moved from the
                // old cluster's sums to the new one's when the queue fills or the
                // iteration ends, lane = feature, int64 fixed point (any order)
#ifdef KP_EXP_NOACC
                continue;  // timing experiment only: no accumulation of changed rows
#endif
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const bool ch = label[h] < K && label[h] != prevl[h];
                    const unsigned mask = __ballot_sync(FULL, ch);
                    if (!mask) continue;
                    if (qn + __popc(mask) > SCR) {
                        flush_queue();
                        qn = 0;
                    }
                    if (ch) {
                        const int pos = qn + __popc(mask & ((1u << lane) - 1u));
                        PCHECK(pos < SCR && label[h] >= 0 && label[h] < K);
                        float* dst = scr + (warp * SCR + pos) * D;
#pragma unroll
                        for (int f = 0; f < L; ++f) *reinterpret_cast<float2*>(dst + 2 * f) = xv[h][f];
                        scl[(warp * SCR + pos) * 2] = label[h];
                        scl[(warp * SCR + pos) * 2 + 1] = prevl[h];
                    }
                    qn += __popc(mask);
                }
                continue;
            }

            // ---- full iteration: every row summed (counting sort of the tile)
            int label[R];
            {
                float b1[R], b2[R], tr[R];
                int i1[R];
                if constexpr (TCS) {
                    persist_top2_tc<D, K, R, WG>(xv, tab, tmem, bh_desc, bl_desc, tbar, tph, cnmax_f, cmax_f, b1, b2, i1, tr, wg);
                } else {
                    persist_top2<D, K, R>(xv, tab, b1, b2, i1);
#pragma unroll
                    for (int h = 0; h < R; ++h) tr[h] = tau;
                }
#pragma unroll
                for (int h = 0; h < R; ++h) {
                    const int row = tid + h * THREADS;
                    label[h] = K;  // rows past the end sort last
                    if (row0 + row < p.n) {
                        label[h] = i1[h];
                        if (K > 1 && !(b2[h] - b1[h] > tr[h])) {
                            label[h] = ref_argmin<float>(xt + row * D, D, c64s, cn64s, K);
                            ++refined;
                        }
                        lab_out[row0 + row] = static_cast<int8_t>(label[h]);
                    }
                }
            }
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
            persist_sync<WG>(wg);  // counts visible; every warp is done with the previous tile's stage
            if (tid == 0 && g > 0 && consumed[(g - 1) % NST] == 0xFFFFFFFFu) {
                consumed[(g - 1) % NST] = 0u;  // the previous full tile's stage: sort buffer no more
                sdef[(g - 1) % NST] = 0;
                issue(static_cast<int>((g - 1) % NST), it);
            }
            int tot = 0, before[R];
#pragma unroll
            for (int h = 0; h < R; ++h) before[h] = 0;
            if (lane < K) {
#pragma unroll
                for (int v = 0; v < VW; ++v) {
                    const int c = cnt[v * K + lane];
                    tot += c;
#pragma unroll
                    for (int h = 0; h < R; ++h) before[h] += v < h * W + warp ? c : 0;
                }
            }
            int start = tot;
#pragma unroll
            for (int o = 1; o < K; o <<= 1) {
                const int v = __shfl_up_sync(FULL, start, o);
                if (lane >= o) start += v;
            }
            start -= tot;
            if (warp == 0 && lane < K) count_acc += tot;
            // scatter into label order, in place (every row is in registers)
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const int pos = __shfl_sync(FULL, start + before[h], label[h] < K ? label[h] : 0) + rank[h];
                if (label[h] < K) {
#pragma unroll
                    for (int f = 0; f < L; ++f) *reinterpret_cast<float2*>(xt + pos * D + 2 * f) = xv[h][f];
                }
            }
            persist_sync<WG>(wg);
            // warp w sums the sorted runs of clusters w, w+W, ... in f64 and
            // adds the tile's run sums as int64 fixed point
#pragma unroll
            for (int jj = 0; jj < JW; ++jj) {
                const int cl = warp + jj * W;
                if (cl >= K) break;
                const int r0 = __shfl_sync(FULL, start, cl);
                const int r1 = r0 + __shfl_sync(FULL, tot, cl);
                double2 part = make_double2(0.0, 0.0), part2 = make_double2(0.0, 0.0);
                if (gq < GR) {
                    const float* src = xt + 2 * q;
                    int r = r0 + gq;
#pragma unroll 2
                    for (; r + GR < r1; r += 2 * GR) {
                        const float2 v = *reinterpret_cast<const float2*>(src + r * D);
                        const float2 u = *reinterpret_cast<const float2*>(src + (r + GR) * D);
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
#pragma unroll
                for (int o = 1; o < GR; o <<= 1) {
                    const double vx = __shfl_down_sync(FULL, part.x, o * L);
                    const double vy = __shfl_down_sync(FULL, part.y, o * L);
                    if (gq + o < GR) {
                        part.x += vx;
                        part.y += vy;
                    }
                }
                if (gq == 0) {
                    wsum[jj][0] += llrint(ldexp(part.x, shift));
                    wsum[jj][1] += llrint(ldexp(part.y, shift));
                }
            }
            if (tid == 0) consumed[s] = 0xFFFFFFFFu;  // released at the next tile's count barrier
        }
        if (!full && qn > 0) flush_queue();
        persist_sync<WG>(wg);  // every warp is done with this iteration's tiles
        // a full iteration hands its last stage back only now (it was the sort buffer)
        if (full && tid == 0 && g > 0 && consumed[(g - 1) % NST] == 0xFFFFFFFFu) {
            consumed[(g - 1) % NST] = 0u;
            sdef[(g - 1) % NST] = 0;
            issue(static_cast<int>((g - 1) % NST), it);
        }
        if (tm && tid == 0) tm[vb] = gtimer();
        asm volatile("fence.proxy.async.global;" ::: "memory");  // this iteration's labels -> later bulk reads

        // ---- this CTA's int64 partial stats -> global accumulator
        unsigned long long* acc_it = p.acc + (it % 3) * S;
        if (!full) {
            if (lane < K) cnt[warp * K + lane] = cnt_delta;
            persist_sync<WG>(wg);
            for (int e = tid; e < KD; e += THREADS) {
                long long v = 0;
#pragma unroll
                for (int c = 0; c < W; ++c) v += wacc[c * KD + e];
                if (v != 0) atomicAdd(acc_it + e, static_cast<unsigned long long>(v));
            }
            if (tid < K) {
                long long c = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) c += cnt[w * K + tid];
                if (c != 0) atomicAdd(acc_it + KD + tid, static_cast<unsigned long long>(c));
            }
        } else {
#pragma unroll
            for (int jj = 0; jj < JW; ++jj) {
                const int cl = warp + jj * W;
                if (cl < K && gq == 0 && q < L) {
                    if (wsum[jj][0]) atomicAdd(acc_it + cl * D + 2 * q, static_cast<unsigned long long>(wsum[jj][0]));
                    if (wsum[jj][1])
                        atomicAdd(acc_it + cl * D + 2 * q + 1, static_cast<unsigned long long>(wsum[jj][1]));
                }
            }
            if (warp == 0 && lane < K && count_acc)
                atomicAdd(acc_it + KD + lane, static_cast<unsigned long long>(count_acc));
        }
        persist_sync<WG>(wg);

        // ---- grid barrier (+ the cross-rank exchange on the last arrival)
        // two-level arrival: CTA b counts in group b % NG, the last of a group in
        // the root word (592 same-address atomics serialised at one L2 slice)
        const int NG = G < 32 ? G : 32;
        const unsigned round = static_cast<unsigned>(it + 1 - p.it_begin);
        const unsigned target = static_cast<unsigned>(NG) * round;
        if (tid == 0) {
            __threadfence();
            const int grp = vb % NG;
            const unsigned gsize = static_cast<unsigned>((G - 1 - grp) / NG + 1);
            const unsigned oldg = atomicAdd(p.arrive + 1 + grp, 1u);
            int last = 0;
            if (oldg == gsize * round - 1u) last = atomicAdd(p.arrive, 1u) == target - 1u ? 1 : 0;
            *s_last = last;
        }
        persist_sync<WG>(wg);
        // world > 1: the exchange epoch of this iteration (every CTA read the
        // base before barrier 0; only the finaliser advances the stored epoch)
        const unsigned long long epoch = xbase + static_cast<unsigned long long>(it + 1 - p.it_begin);
        const int xslot = static_cast<int>(epoch & 1);
        if (p.world > 1 && *s_last) {
            // finaliser: this rank's stats into every rank's exchange region
            // (NVLink stores; its own too), then one release flag per rank
            if (tid == 0) *(xchg_flags(p.peers[p.rank], p.world) + p.world) = epoch;
            for (int e = tid; e < S; e += THREADS) {
                const long long qv = static_cast<long long>(__ldcg(acc_it + e));
                const double v = e < KD ? ldexp(static_cast<double>(qv), -shift) : static_cast<double>(qv);
                for (int r = 0; r < p.world; ++r) xchg_recv(p.peers[r], xslot, p.world, p.rank)[e] = v;
            }
            // the CTA barrier orders every thread's stores before the flag
            // writers' system-scope release (cumulative, as in a grid sync:
            // no fence per storing thread -- one NVLink round trip less)
            persist_sync<WG>(wg);
            if (tid < p.world) st_release_sys(xchg_flags(p.peers[tid], p.world) + p.rank, epoch);
        }
        if (p.world > 1) {
            // every CTA waits for every rank's stats in its own region (no
            // second hop through a release word) and folds them itself below
            if (tid < p.world) {
                const unsigned long long* mine_f = xchg_flags(p.peers[p.rank], p.world) + tid;
                const long long t0 = clock64();
                while (ld_acquire_sys(mine_f) < epoch) {
                    __nanosleep(32);
                    if (clock64() - t0 > 40000000000ll) {  // a rank never arrived (~20 s): TimeoutError, no trap
                        atomicExch(p.flags + 3, 1);
                        *s_tmo = 1;
                        break;
                    }
                }
            }
        } else if (tid == 0) {
            const long long t0 = clock64();
            while (ld_acquire_gpu_u32(p.arrive) < target) {
                __nanosleep(20);
                if (clock64() - t0 > 40000000000ll) {
                    atomicExch(p.flags + 3, 1);
                    *s_tmo = 1;
                    break;
                }
            }
        }
        persist_sync<WG>(wg);
        if (tm && tid == 0) tm[TG + vb] = gtimer();
        // ---- the folded stats of this iteration, added to the running sums
        // (delta iterations) -- every CTA the same bits -- and the old state
        const double* xrecv = p.world > 1 ? xchg_recv(p.peers[p.rank], xslot, p.world, 0) : nullptr;
        auto folded = [&](int e) {  // this iteration's stat e, plus the running value (delta iterations)
            double v;
            if (p.world > 1) {  // rank-order fold (transport.hpp:136-148), identical in every CTA of every rank
                v = 0.0;
                for (int r = 0; r < p.world; ++r) v += __ldcv(xrecv + static_cast<int64_t>(r) * XCHG_STATS + e);
            } else {
                const long long qv = static_cast<long long>(__ldcg(acc_it + e));
                v = e < KD ? ldexp(static_cast<double>(qv), -shift) : static_cast<double>(qv);
            }
            if (!full) v += run[e];  // delta iterations: changes added to the running sums
            return v;
        };
        // the new centroids in the same pass (cluster.cpp:125-133): the thread of
        // entry e folds its cluster's count itself (the same bits as the count's
        // own entry); counts go to ncnt, so run[KD..] stays the old value until
        // every thread has read it
        double* ncnt = cnold + K;
        for (int e = tid; e < S; e += THREADS) {
            const double v = folded(e);
            if (e < KD) {
                const double count = folded(KD + e / D);
                run[e] = v;
                const double c_old = c64s[e];
                cold[e] = c_old;
                c64s[e] = count > 0.0 ? v / count : c_old;  // empty cluster keeps its centroid
            } else {
                ncnt[e - KD] = v;
            }
        }
        if (tid < K) cnold[tid] = cn64s[tid];
        persist_sync<WG>(wg);
        if (*s_tmo) {  // (flags[3] tells the host; the other CTAs time out at their own waits)
            stop = true;
            break;
        }
        // ---- rest of the update (cluster.cpp:123-150), identical in every CTA:
        // warp 0 the tables, warp 1 inertia / displacement, warp 2 the counts
        if (warp == 0) {
            persist_tables<D, K>(c64s, cn64s, tab, misc, bhi, blo);
        } else if (warp == 2) {
            if (lane < K) run[KD + lane] = ncnt[lane];
        } else if (warp == 1) {
            double inertia_part = 0.0, dmax = 0.0;
            if (lane < K) {
                const double count = ncnt[lane];
                double dot = 0.0, dsq = 0.0;
                for (int f = 0; f < D; ++f) {
                    const int e = lane * D + f;
                    dot += cold[e] * run[e];
                    const double diff = c64s[e] - cold[e];
                    dsq = add_rn(dsq, mul_rn(diff, diff));  // cluster.cpp:142-146 order
                }
                inertia_part = count * cnold[lane] - 2.0 * dot;  // uses the old |c_j|^2
                dmax = __dsqrt_rn(dsq);
            }
            inertia_part = warp_sum(inertia_part);
            dmax = warp_max(dmax);
            if (lane == 0) {
                if (vb == 0) {
                    p.trace[it] = p.sx2[2] + inertia_part;
                    p.disp[it] = dmax;
                    p.flags[1] = it + 1;
                    if (dmax < p.tol) p.flags[0] = 1;
                }
                misc[2] = dmax < p.tol ? 1.0 : 0.0;
            }
        }
        persist_sync<WG>(wg);
        if (tm && vb == 0 && tid == 0) tm[2 * TG + 1] = gtimer();
        stop = misc[2] != 0.0;
        // tiles of the next iteration already staged: their previous labels are final now
        if (!stop && tid == 0) {
            for (int64_t h = g; h < g + NST; ++h) {
                const int s = static_cast<int>(h % NST);
                if (sdef[s] && siter[s] == it + 1) issue_labels(s);
            }
        }
        persist_sync<WG>(wg);
    }
    // loads issued but never consumed (early stop): let them land before exit
    if (tid == 0) {
        for (int64_t h = g; h < g + NST; ++h)
            mbar_wait(&bars[h % NST], static_cast<uint32_t>((h / NST) & 1));
    }
    if (refined) atomicAdd(p.refined, refined);
    if (vb == 0) {
        for (int e = tid; e < KD; e += THREADS) p.c64_out[e] = c64s[e];
        for (int e = tid; e < S; e += THREADS) p.run_io[e] = run[e];
    }
    if constexpr (TCS) {
        tc::tc_fence_before();
        __syncthreads();  // every warpgroup done with its columns
        if (threadIdx.x < 32) {
            tc::tc_fence_after();
            tc::tmem_dealloc(tmem, TC_COLS * WG);  // warpgroup 0's base = the allocation
        }
    }
}
