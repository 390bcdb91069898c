// cdist_tc.cu -- tcgen05 3xTF32 distance tiles for large feature counts
// (BASELINE config 4: 100k x 1024 vs 100k x 1024; north_star (3): tensor cores
// "only when the feature dimension makes it a real dense contraction").
//
// Reference: distance_block / matmul_local (pairwise.cpp:22-33,
// ndarray.hpp:400-418), place_chunk (tile.hpp:90-107).
//
// Persistent CTAs, one per SM, 14 warps (2-5 idle):
//   warp 0      TMA producer: 32-column K chunks of a 128-row X tile and a
//               256-row Y tile, SWIZZLE_128B K-major, 2-stage ring.
//   warp 1      TMEM allocator + MMA issuer: per K=8 step three
//               tcgen05.mma.kind::tf32 (M=128, N=256): hi.hi + hi.lo + lo.hi into
//               a 128x256 fp32 TMEM accumulator (double-buffered: 512 columns).
//   (both operands are first centred on a common mu (centre_sample_kernel):
//    hi = fl(x - mu) and lo = hi - trunc_tf32(hi) are made once per operand by
//    centre_split_kernel into 16-byte-pitched copies and loaded by TMA side by
//    side; the tensor core truncates hi to tf32 itself -- pinned by
//    tests/test_gpu_tc.py.  Centring keeps the norms and dot products small, so
//    the fp32 accumulation over K stays inside BASELINE's 1e-5 gate at d = 1024.
//    Splitting in shared memory per tile cost as much smem bandwidth as the MMAs.)
//   warps 6-13  epilogue: tcgen05.ld of each accumulator row, then
//               d = sqrt(max(xn + yn - 2g, 0)) into swizzled smem boxes written
//               by TMA bulk stores (+ the self block's zero diagonal); rows
//               whose window is not 16-byte aligned use direct stores (warps 6-9).
// The row norms come from the SAME tensor-core path (a diagonal-tile pass), so a
// row's dot product with itself equals its norm bit for bit and duplicate rows
// cancel to exactly 0, as in the reference.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "tc.cuh"

namespace dndc {

namespace cdtc {
constexpr int BM = 128, BN = 256, BK = 32, STAGES = 2;
constexpr int A_BYTES = BM * BK * 4;   // 16 KB
constexpr int B_BYTES = BN * BK * 4;   // 32 KB
constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);  // raw + lo
constexpr int EPI_MAX = 12;                             // epilogue warps: 8 (2 stages) or 12 (1 stage)
// store boxes: 32 rows x BC columns (BC = 16: SWIZZLE_64B, 32: SWIZZLE_128B),
// double-buffered per epilogue warp
#ifndef CDTC_NBUF1
#define CDTC_NBUF1 2  // store boxes in flight per warp in the one-stage layout
#endif
#ifndef CDTC_EPI1
#define CDTC_EPI1 12
#endif
#ifndef CDTC_BC1
#define CDTC_BC1 32
#endif
__host__ __device__ constexpr int stg_bytes(int bc, int nbuf = 2) { return nbuf * bc * 32 * 4; }
constexpr int NBARS = 3 * STAGES + 4;
constexpr int THREADS = (2 + EPI_MAX) * 32;
// shared-memory layout for `nst` stages and `epi` TMA-store epilogue warps
__host__ __device__ constexpr int off_stg(int nst) { return nst * STAGE_BYTES; }
__host__ __device__ constexpr int nbuf_of(int nst) { return nst == 1 ? CDTC_NBUF1 : 2; }
__host__ __device__ constexpr int off_bar(int nst, int epi, int bc) {
    return off_stg(nst) + epi * stg_bytes(bc, nbuf_of(nst));
}
__host__ __device__ constexpr int smem_bytes(int nst, int epi, int bc) {
    return off_bar(nst, epi, bc) + NBARS * 8 + 16 + 1024;
}
constexpr int SMEM = smem_bytes(2, 8, 16);  // the largest configuration
static_assert(smem_bytes(1, CDTC_EPI1, CDTC_BC1) <= SMEM, "smem layouts");
constexpr int TMEM_COLS = 512;
#ifndef CDTC_GROUP
#define CDTC_GROUP 16
#endif
constexpr int GROUP = CDTC_GROUP;  // rasterisation: GROUP row blocks x all column blocks per super-block
}  // namespace cdtc

struct CdtcParams {
    int nst;          // TMA stages (1 when a tile is one K chunk: the MMAs are short)
    int epi;          // TMA-store epilogue warps (MODE 2): 8 = warps 6-13, 12 = warps 2-13
    int64_t nx, ny;
    int m;
    const float* xn;   // norms (null in NORM mode)
    const float* yn;
    const float* xd;   // norm-bias model (null: off): tensor-core norm minus the f64-exact one
    const float* yd;
    float* out;        // distances (DIST) or norms (NORM)
    int64_t ld, col_off, diag_offset;
    bool vec;
};

__device__ __forceinline__ void cdtc_tile_of(int64_t t, int64_t nrb, int64_t ncb, int64_t& rb, int64_t& cb) {
    using namespace cdtc;
    const int64_t per_group = static_cast<int64_t>(GROUP) * ncb;  // GROUP row blocks x all column blocks
    const int64_t g = t / per_group, r = t % per_group;
    const int64_t rows_in_group = min(static_cast<int64_t>(GROUP), nrb - g * GROUP);
    rb = g * GROUP + r % rows_in_group;
    cb = r / rows_in_group;
}

// MODE 0: row norms (diagonal tiles); 1: distances with direct stores (any
// alignment); 2: distances staged in swizzled shared memory and written by TMA
// bulk stores (32x32 boxes, out-of-range rows/columns clipped by the unit).
template <int MODE, int BC = 16>
__global__ void __launch_bounds__(cdtc::THREADS, 1)
    cdist_tc_kernel(const __grid_constant__ CUtensorMap mapx, const __grid_constant__ CUtensorMap mapy,
                    const __grid_constant__ CUtensorMap mapxl, const __grid_constant__ CUtensorMap mapyl,
                    const __grid_constant__ CUtensorMap mapo, CdtcParams p) {
    using namespace cdtc;
    constexpr bool NORM = MODE == 0;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int nst = p.nst, epi = MODE == 2 ? p.epi : 8;
    const int STG = nst;  // stages in use
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar(nst, epi, BC));
    uint64_t* full = bars;                 // [STAGES] TMA landed
    uint64_t* split = bars + STAGES;       // [STAGES] lo written
    uint64_t* empty = bars + 2 * STAGES;   // [STAGES] MMAs done with the stage
    uint64_t* tfull = bars + 3 * STAGES;   // [2] accumulator ready
    uint64_t* tempty = tfull + 2;          // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nrb = ceil_div(p.nx, BM);
    const int64_t ncb = NORM ? 1 : ceil_div(p.ny, BN);
    const int64_t ntiles = nrb * ncb;
    const int kchunks = (p.m + BK - 1) / BK;

    if (warp == 1) {
        tc::tmem_alloc(tmem_slot, TMEM_COLS);
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&split[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(&tfull[b], 1);
                // MODE 2: every epilogue warp arrives on its own (no CTA-wide
                // named barrier per tile); otherwise one arrival after a barrier
                tc::mbar_init(&tempty[b], MODE == 2 ? epi : 1);
            }
            tc::mbar_fence_init();
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto stage_ptr = [&](int s) { return smem + s * STAGE_BYTES; };  // A, B, Alo, Blo

    if (warp == 0) {
        // ------------------------------------------------------- producer
        if (lane == 0) {
            tc::tma_prefetch_desc(&mapx);
            tc::tma_prefetch_desc(&mapy);
            int64_t g = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int64_t rb, cb;
                if (NORM) { rb = t; cb = 0; } else cdtc_tile_of(t, nrb, ncb, rb, cb);
                const int row0 = static_cast<int>(rb * BM);
                const int col0 = NORM ? row0 : static_cast<int>(cb * BN);
                for (int kc = 0; kc < kchunks; ++kc, ++g) {
                    const int s = static_cast<int>(g % STG);
                    if (g >= STG) tc::mbar_wait(&empty[s], static_cast<uint32_t>((g / STG - 1) & 1));
                    unsigned char* st = stage_ptr(s);
                    // hi = the raw tile (the tensor core truncates to tf32), lo from
                    // the pre-split copies: no generic-proxy pass over the stage
                    tc::mbar_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
                    tc::tma_load_2d(st, &mapx, &full[s], kc * BK, row0);
                    tc::tma_load_2d(st + A_BYTES, &mapy, &full[s], kc * BK, col0);
                    tc::tma_load_2d(st + A_BYTES + B_BYTES, &mapxl, &full[s], kc * BK, row0);
                    tc::tma_load_2d(st + 2 * A_BYTES + B_BYTES, &mapyl, &full[s], kc * BK, col0);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(BM, BN, 0, 0);
            int64_t g = 0, tcount = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tcount) {
                const int b = static_cast<int>(tcount & 1);
                if (tcount >= 2) tc::mbar_wait(&tempty[b], static_cast<uint32_t>((tcount / 2 - 1) & 1));
                const uint32_t dt = tmem + b * BN;
                for (int kc = 0; kc < kchunks; ++kc, ++g) {
                    const int s = static_cast<int>(g % STG);
                    tc::mbar_wait(&full[s], static_cast<uint32_t>((g / STG) & 1));
                    tc::tc_fence_after();
                    const uint32_t a = tc::smem_u32(stage_ptr(s));
                    const uint32_t bsm = a + A_BYTES, alo = a + A_BYTES + B_BYTES, blo = alo + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 8; ++k) {
                        const uint32_t ko = k * 32;  // bytes along K inside the 128-byte swizzle atom
                        const uint64_t dah = tc::smem_desc(a + ko, 16, 1024, 2);
                        const uint64_t dal = tc::smem_desc(alo + ko, 16, 1024, 2);
                        const uint64_t dbh = tc::smem_desc(bsm + ko, 16, 1024, 2);
                        const uint64_t dbl = tc::smem_desc(blo + ko, 16, 1024, 2);
                        tc::mma_tf32(dt, dah, dbh, idesc, (kc > 0 || k > 0) ? 1u : 0u);
                        tc::mma_tf32(dt, dah, dbl, idesc, 1);
                        tc::mma_tf32(dt, dal, dbh, idesc, 1);
                    }
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(&tfull[b]);
            }
        }
    } else if (MODE == 2 && warp >= 14 - epi) {
        // ------------------------------------------------------- epilogue (TMA stores)
        // warp e of `epi`: TMEM lanes of quarter (warp % 4); the quarter's
        // 256/BC column chunks go round-robin over its epi/4 warps
        constexpr int NCH = BN / BC, BOX = BC * 32 * 4;
        const int e = warp - (14 - epi), q = warp & 3, sub = e >> 2, nsub = epi >> 2;
        const int r = q * 32 + lane;
        const int nbuf = nbuf_of(nst);
        unsigned char* stg = smem + off_stg(nst) + e * stg_bytes(BC, nbuf);  // nbuf boxes, swizzle-atom aligned
        int64_t tcount = 0, nbox = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tcount) {
            int64_t rb, cb;
            cdtc_tile_of(t, nrb, ncb, rb, cb);
            const int64_t row0 = rb * BM, col0 = cb * BN;
            const int b = static_cast<int>(tcount & 1);
            tc::mbar_wait(&tfull[b], static_cast<uint32_t>((tcount / 2) & 1));
            tc::tc_fence_after();
            const int64_t gi = row0 + r;
            const float xni = gi < p.nx ? __ldg(p.xn + gi) : 0.f;
            const float xdi = (p.xd && gi < p.nx) ? __ldg(p.xd + gi) : 0.f;
            const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * BN;
            const bool diag = p.diag_offset >= 0 && col0 < row0 + p.diag_offset + BM &&
                              row0 + p.diag_offset < col0 + BN;
            // column norms of a chunk, fetched one chunk ahead
            auto load_yn = [&](int64_t gc, float4 (&y4)[BC / 4]) {
#pragma unroll
                for (int j = 0; j < BC; j += 4) {
                    float4 yv = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (gc + j + 3 < p.ny) {
                        yv = __ldg(reinterpret_cast<const float4*>(p.yn + gc + j));
                    } else {
                        if (gc + j < p.ny) yv.x = __ldg(p.yn + gc + j);
                        if (gc + j + 1 < p.ny) yv.y = __ldg(p.yn + gc + j + 1);
                        if (gc + j + 2 < p.ny) yv.z = __ldg(p.yn + gc + j + 2);
                    }
                    y4[j / 4] = yv;
                }
            };
            float4 ynext[BC / 4];
            load_yn(col0 + sub * BC, ynext);
#pragma unroll 1
            for (int cc = sub; cc < NCH; cc += nsub, ++nbox) {
                const int c0 = cc * BC;
                float v[BC];
#pragma unroll
#ifdef CDTC_EXP_STOREONLY
                for (int h = 0; h < BC; ++h) v[h] = 0.25f * static_cast<float>(h);  // timing experiment: stores only
#else
                for (int h = 0; h < BC / 16; ++h) tc::tmem_ld16(trow + c0 + 16 * h, *reinterpret_cast<float(*)[16]>(v + 16 * h));
#endif
                const int64_t gc = col0 + c0;
                float4 ycur[BC / 4];
#pragma unroll
                for (int u = 0; u < BC / 4; ++u) ycur[u] = ynext[u];
                if (cc + nsub < NCH) load_yn(gc + BC * nsub, ynext);
                float d[BC];
                if (p.xd) {
                    // norm-bias model (large d): s = a + b - 2g with the tensor-core
                    // norms a, b (so an exact duplicate gives s == 0), then
                    // s += (t - 1)(da + db), t = 2g / (a + b) clamped to [-1, 1],
                    // da, db = tensor-core minus f64-exact norms: the accumulation
                    // bias of g is modelled as t times the norms' (t = 1 for a
                    // duplicate, ~0 for unrelated centred rows -> exact norms)
#pragma unroll
                    for (int j = 0; j < BC; ++j) {
                        const int64_t cj = gc + j;
                        const float ynj = reinterpret_cast<const float*>(ycur)[j];
                        const float ydj = cj < p.ny ? __ldg(p.yd + cj) : 0.f;
                        const float ab = xni + ynj;
                        float sq = fmaf(-2.f, v[j], ab);
                        if (sq != 0.f) {
                            const float t = fminf(fmaxf(__fdividef(2.f * v[j], ab), -1.f), 1.f);
                            sq = fmaf(t - 1.f, xdi + ydj, sq);
                        }
                        d[j] = sqrt_approx(fmaxf(sq, 0.f));
                    }
                } else {
#pragma unroll
                for (int j = 0; j < BC; j += 4) {
                    const float4 yv = ycur[j / 4];
                    const float2 b0 = fadd2(make_float2(xni, xni), make_float2(yv.x, yv.y));
                    const float2 b1 = fadd2(make_float2(xni, xni), make_float2(yv.z, yv.w));
                    const float2 s0 = ffma2(make_float2(-2.f, -2.f), make_float2(v[j], v[j + 1]), b0);
                    const float2 s1 = ffma2(make_float2(-2.f, -2.f), make_float2(v[j + 2], v[j + 3]), b1);
                    d[j] = sqrt_approx(fmaxf(s0.x, 0.f));
                    d[j + 1] = sqrt_approx(fmaxf(s0.y, 0.f));
                    d[j + 2] = sqrt_approx(fmaxf(s1.x, 0.f));
                    d[j + 3] = sqrt_approx(fmaxf(s1.y, 0.f));
                }
                }
                if (diag) {
#pragma unroll
                    for (int j = 0; j < BC; ++j)
                        if (gc + j == gi + p.diag_offset) d[j] = 0.f;
                }
                // buffer nbox % nbuf: its previous box (nbuf stores ago) has been read
                unsigned char* box = stg + (nbox % nbuf) * BOX;
                if (lane == 0) {
                    if (nbuf == 3)
                        asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
                    else
                        tc::bulk_wait_read1();
                }
                __syncwarp();
                // 16-byte chunk j of row `lane` sits at chunk j ^ (the row's swizzle
                // phase): SWIZZLE_64B (lane >> 1) & 3, SWIZZLE_128B lane & 7
#pragma unroll
                for (int j = 0; j < BC / 4; ++j) {
                    const int phys = BC == 16 ? (j ^ ((lane >> 1) & 3)) : (j ^ (lane & 7));
                    *reinterpret_cast<float4*>(box + lane * (BC * 4) + (phys << 4)) =
                        make_float4(d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3]);
                }
                tc::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    // evict_first: the distance matrix is streamed out, never re-read
                    // here (cfg2: 42.9 -> 42.0 ms, tools/gpu_var_cdist.sh)
#ifndef CDTC_STORE_NO_HINT
                    tc::tma_store_2d_hint(&mapo, box, static_cast<int>(gc), static_cast<int>(row0 + q * 32),
                                          tc::l2_policy_evict_first());
#else
                    tc::tma_store_2d(&mapo, box, static_cast<int>(gc), static_cast<int>(row0 + q * 32));
#endif
                    tc::bulk_commit();
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[b]);
        }
        if (lane == 0) tc::bulk_wait0();
    } else if (MODE != 2 && warp >= 6 && warp < 10) {
        // ------------------------------------------------------- epilogue warps (MODE 0 / 1)
        const int q = warp & 3;             // TMEM lane quarter of this warp
        const int r = q * 32 + lane;        // accumulator row = TMEM lane
        int64_t tcount = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tcount) {
            int64_t rb, cb;
            if (NORM) { rb = t; cb = 0; } else cdtc_tile_of(t, nrb, ncb, rb, cb);
            const int64_t row0 = rb * BM, col0 = NORM ? row0 : cb * BN;
            const int b = static_cast<int>(tcount & 1);
            tc::mbar_wait(&tfull[b], static_cast<uint32_t>((tcount / 2) & 1));
            tc::tc_fence_after();
            const int64_t gi = row0 + r;
            const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * BN;
            if (NORM) {
                // the diagonal of the (X-block, X-block) tile: column r of row r
                float v[16];
#pragma unroll 1
                for (int c16 = 0; c16 < BM / 16; ++c16) {
                    tc::tmem_ld16(trow + c16 * 16, v);
                    if (c16 == r / 16 && gi < p.nx) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (i == r % 16) p.out[gi] = v[i];
                    }
                }
            } else {
                const float xni = gi < p.nx ? __ldg(p.xn + gi) : 0.f;
                const float xdi = (p.xd && gi < p.nx) ? __ldg(p.xd + gi) : 0.f;
                float* orow = p.out + gi * p.ld + p.col_off + col0;
                const bool full_cols = col0 + BN <= p.ny;
#pragma unroll 1
                for (int c16 = 0; c16 < BN / 16; ++c16) {
                    float v[16];
                    tc::tmem_ld16(trow + c16 * 16, v);
                    if (gi >= p.nx) continue;
                    const int64_t c0 = col0 + c16 * 16;
                    float d[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float ynj = (c0 + i < p.ny) ? __ldg(p.yn + c0 + i) : 0.f;
                        float sq = fmaf(-2.f, v[i], xni + ynj);
                        if (p.xd && sq != 0.f) {  // norm-bias model, as in MODE 2
                            const float ydj = (c0 + i < p.ny) ? __ldg(p.yd + c0 + i) : 0.f;
                            const float t = fminf(fmaxf(__fdividef(2.f * v[i], xni + ynj), -1.f), 1.f);
                            sq = fmaf(t - 1.f, xdi + ydj, sq);
                        }
                        d[i] = sqrt_approx(fmaxf(sq, 0.f));
                        if (p.diag_offset >= 0 && c0 + i == gi + p.diag_offset) d[i] = 0.f;
                    }
                    float* o = orow + c16 * 16;
                    if (p.vec && full_cols) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4) st_stream4(o + i, d[i], d[i + 1], d[i + 2], d[i + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c0 + i < p.ny) st_stream(o + i, d[i]);
                    }
                }
            }
            tc::tc_fence_before();
            tc::named_sync(2, 128);
            if (r == 0) tc::mbar_arrive(&tempty[b]);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// ------------------------------------------------------------------ host
constexpr int BK_SMALL = 32;  // one K chunk (cdtc::BK)

static int tc_min_m() {
    const char* v = std::getenv("DNDC_CDIST_TC_MIN_M");
    return v ? std::atoi(v) : 256;
}

// d >= 256: a real dense contraction (tensor-pipe bound).  d <= 32 on large
// blocks: one K chunk per tile, the output stream dominates and the
// tensor-core epilogue (12 warps, TMA bulk stores) writes it faster than the
// FFMA tile kernel (cfg2: 44.4 vs 48.7 ms).  DNDC_CDIST_TC_MIN_M overrides.
bool cdist_tc_eligible(int64_t nx, int64_t ny, int64_t m) {
    if (nx < 128 || ny < 128) return false;
    if (std::getenv("DNDC_CDIST_TC_MIN_M")) return m >= tc_min_m();
    return m >= 256 || (m <= BK_SMALL && nx * ny >= (int64_t{1} << 26));
}

// Centre of the operands: mu_f = (mean over <= 256 rows of x sampled evenly +
// the same over y) / 2, f64 sums rounded once to fp32.  Any mu gives the same
// distances in exact arithmetic (|x - y| = |(x - mu) - (y - mu)|); a mu near the
// data's centre keeps the norms and the dot products small, and with them the
// fp32 rounding of the tensor-core accumulation over K (cfg4: 1.6e-5 of
// relative error with raw [0,1) data at d = 1024, against BASELINE's 1e-5 gate).
__global__ void centre_sample_kernel(const float* __restrict__ x, int64_t nx, const float* __restrict__ y,
                                     int64_t ny, int64_t m, float* __restrict__ mu, int64_t pitch) {
    const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (f >= pitch) return;
    if (f >= m) {
        mu[f] = 0.f;
        return;
    }
    auto mean = [&](const float* a, int64_t n) {
        const int64_t ns = n < 256 ? n : 256;
        double acc = 0.0;
        for (int64_t s = 0; s < ns; ++s) acc += static_cast<double>(a[(s * n / ns) * m + f]);
        return ns > 0 ? acc / static_cast<double>(ns) : 0.0;
    };
    mu[f] = static_cast<float>(0.5 * (mean(x, nx) + mean(y, ny)));
}

// hi = fl(x - mu) into a 16-byte-pitched matrix (TMA needs 16-byte row
// pitches; pad columns 0) and lo = hi - trunc_tf32(hi): the 3xTF32 operands,
// made once per operand (the tensor core truncates hi to tf32 itself).
__global__ void centre_split_kernel(const float* __restrict__ src, int64_t rows, int64_t m,
                                    const float* __restrict__ mu, int64_t pitch, float* __restrict__ hi,
                                    float* __restrict__ lo) {
    const int64_t total = rows * pitch;
    if (m == pitch && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const int64_t total4 = total / 4, pitch4 = pitch / 4;
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total4;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
            const float4 c = __ldg(reinterpret_cast<const float4*>(mu) + i % pitch4);
            float4 h = make_float4(v.x - c.x, v.y - c.y, v.z - c.z, v.w - c.w);
            float4 l;
            l.x = h.x - __uint_as_float(__float_as_uint(h.x) & 0xFFFFE000u);
            l.y = h.y - __uint_as_float(__float_as_uint(h.y) & 0xFFFFE000u);
            l.z = h.z - __uint_as_float(__float_as_uint(h.z) & 0xFFFFE000u);
            l.w = h.w - __uint_as_float(__float_as_uint(h.w) & 0xFFFFE000u);
            reinterpret_cast<float4*>(hi)[i] = h;
            reinterpret_cast<float4*>(lo)[i] = l;
        }
        return;
    }
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / pitch, f = i % pitch;
        const float h = f < m ? src[r * m + f] - mu[f] : 0.f;
        hi[i] = h;
        lo[i] = h - __uint_as_float(__float_as_uint(h) & 0xFFFFE000u);
    }
}

// d[i] = a[i] - fl32(sum_f hi[i][f]^2 in f64): how far the tensor-core norm a
// (3xTF32, fp32 accumulation over K) sits from the exact norm of the same
// centred row; one warp per row.
__global__ void norm_bias_kernel(const float* __restrict__ hi, int64_t rows, int64_t m, int64_t pitch,
                                 const float* __restrict__ a, float* __restrict__ dout) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
        double acc = 0.0;
        for (int64_t f = lane; f < m; f += 32) {
            const double v = static_cast<double>(hi[r * pitch + f]);
            acc = fma(v, v, acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) dout[r] = a[r] - static_cast<float>(acc);
    }
}

// DNDC_CDTC_NORM=mma|model: the norm-bias model (see the epilogue) is on by
// default from d >= 128 (at small d the plain formula is already ~1e-6).
static bool use_norm_model(int64_t m) {
    const char* v = std::getenv("DNDC_CDTC_NORM");
    if (v && std::string(v) == "mma") return false;
    if (v && std::string(v) == "model") return true;
    return m >= 128;
}

struct TmaView {
    const float* p;
    int64_t pitch;  // elements
};

struct TcOperand {
    const float* hi;
    const float* lo;
    int64_t pitch;  // elements
};

static TcOperand tc_operand(dndc_ctx* ctx, const char* hname, const char* lname, const float* src, int64_t rows,
                            int64_t m, const float* mu, cudaStream_t s) {
    const int64_t pitch = (m + 3) / 4 * 4;
    const size_t bytes = sizeof(float) * std::max<int64_t>(rows, 1) * pitch;
    float* hi = static_cast<float*>(ctx->slot(hname, bytes));
    float* lo = static_cast<float*>(ctx->slot(lname, bytes));
    const int64_t work = rows * pitch / (pitch == m ? 4 : 1);
    if (work > 0) {
        const int grid = static_cast<int>(std::min<int64_t>(ceil_div(work, 256), ctx->num_sms * 8));
        centre_split_kernel<<<grid, 256, 0, s>>>(src, rows, m, mu, pitch, hi, lo);
        DNDC_LAUNCHED(ctx);
    }
    return {hi, lo, pitch};
}

void cdist_tile_tc_f32(dndc_ctx* ctx, const float* x, const float* xn_unused, int64_t nx, const float* y,
                       const float* yn_unused, int64_t ny, int64_t m, float* out, int64_t ld_out, int64_t col_off,
                       int64_t diag_offset, cudaStream_t stream) {
    using namespace cdtc;
    (void)xn_unused;
    (void)yn_unused;
    const bool same = y == x && ny == nx;
    const int64_t pitch = (m + 3) / 4 * 4;
    float* mu = static_cast<float*>(ctx->slot("cdtc_mu", sizeof(float) * pitch));
    centre_sample_kernel<<<static_cast<int>(ceil_div(pitch, 128)), 128, 0, stream>>>(x, nx, y, ny, m, mu, pitch);
    DNDC_LAUNCHED(ctx);
    const TcOperand xo = tc_operand(ctx, "cdtc_x", "cdtc_xlo", x, nx, m, mu, stream);
    const TcOperand yo = same ? xo : tc_operand(ctx, "cdtc_y", "cdtc_ylo", y, ny, m, mu, stream);
    const TmaView xv{xo.hi, pitch}, yv{yo.hi, pitch}, xl{xo.lo, pitch}, yl{yo.lo, pitch};
    const float* xa = xv.p;
    const float* ya = yv.p;
    static bool attr = false;
    if (!attr) {
        DNDC_CUDA(cudaFuncSetAttribute(cdist_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        DNDC_CUDA(cudaFuncSetAttribute(cdist_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        DNDC_CUDA(cudaFuncSetAttribute(cdist_tc_kernel<2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        DNDC_CUDA(cudaFuncSetAttribute(cdist_tc_kernel<2, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        attr = true;
    }
    // norms through the same tensor-core path (diagonal tiles)
    float* xn = static_cast<float*>(ctx->slot("cdtc_xn", sizeof(float) * std::max<int64_t>(nx, 1)));
    float* yn = static_cast<float*>(ctx->slot("cdtc_yn", sizeof(float) * std::max<int64_t>(ny, 1)));
    auto norms = [&](const float* a, const float* al, int64_t pitch, int64_t rows, float* dst) {
        const CUtensorMap ma = make_tmap_2d_f32(a, rows, m, pitch * 4, BK, BM, true);
        const CUtensorMap mb = make_tmap_2d_f32(a, rows, m, pitch * 4, BK, BN, true);
        const CUtensorMap mal = make_tmap_2d_f32(al, rows, m, pitch * 4, BK, BM, true);
        const CUtensorMap mbl = make_tmap_2d_f32(al, rows, m, pitch * 4, BK, BN, true);
        CdtcParams np{};
        np.nx = rows;
        np.ny = rows;
        np.m = static_cast<int>(m);
        np.nst = m <= BK ? 1 : 2;
        np.epi = 8;
        np.out = dst;
        const int grid = static_cast<int>(std::min<int64_t>(ceil_div(rows, BM), ctx->num_sms));
        cdist_tc_kernel<0><<<grid, THREADS, SMEM, stream>>>(ma, mb, mal, mbl, ma, np);
        DNDC_LAUNCHED(ctx);
    };
    norms(xa, xl.p, xv.pitch, nx, xn);
    if (same) DNDC_CUDA(cudaMemcpyAsync(yn, xn, sizeof(float) * nx, cudaMemcpyDeviceToDevice, stream));
    else norms(ya, yl.p, yv.pitch, ny, yn);
    float* xd = nullptr;
    float* yd = nullptr;
    if (use_norm_model(m)) {
        xd = static_cast<float*>(ctx->slot("cdtc_xd", sizeof(float) * std::max<int64_t>(nx, 1)));
        yd = same ? xd : static_cast<float*>(ctx->slot("cdtc_yd", sizeof(float) * std::max<int64_t>(ny, 1)));
        auto bias = [&](const float* hi, int64_t rows, const float* a, float* d) {
            if (rows <= 0) return;
            const int grid = static_cast<int>(std::min<int64_t>(ceil_div(rows * 32, 256), ctx->num_sms * 16));
            norm_bias_kernel<<<grid, 256, 0, stream>>>(hi, rows, m, pitch, a, d);
            DNDC_LAUNCHED(ctx);
        };
        bias(xa, nx, xn, xd);
        if (!same) bias(ya, ny, yn, yd);
    }

    const CUtensorMap mx = make_tmap_2d_f32(xa, nx, m, xv.pitch * 4, BK, BM, true);
    const CUtensorMap my = make_tmap_2d_f32(ya, ny, m, yv.pitch * 4, BK, BN, true);
    const CUtensorMap mxl = make_tmap_2d_f32(xl.p, nx, m, xl.pitch * 4, BK, BM, true);
    const CUtensorMap myl = make_tmap_2d_f32(yl.p, ny, m, yl.pitch * 4, BK, BN, true);
    CdtcParams pp{};
    pp.nx = nx;
    pp.ny = ny;
    pp.m = static_cast<int>(m);
    pp.xn = xn;
    pp.yn = yn;
    pp.xd = xd;
    pp.yd = yd;
    pp.out = out;
    pp.ld = ld_out;
    pp.col_off = col_off;
    pp.diag_offset = diag_offset;
    pp.vec = (ld_out % 4 == 0) && (col_off % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    // one K chunk per tile: one stage keeps the MMAs fed and frees room for 12
    // epilogue warps (the epilogue is then the long pole)
    pp.nst = m <= BK ? 1 : 2;
    pp.epi = pp.nst == 1 ? CDTC_EPI1 : 8;
    const int64_t tiles = ceil_div(nx, BM) * ceil_div(ny, BN);
    const int grid = static_cast<int>(std::min<int64_t>(tiles, ctx->num_sms));
    float* obase = out + col_off;
    if (pp.vec && (ld_out * 4) % 16 == 0 && ny >= 16) {
        // TMA stores: the window [nx x ny] of the ld-wide output at col_off
        if (pp.nst == 1 && ny >= 32 && CDTC_BC1 == 32) {
            // 128-byte box rows: half the TMA store transactions of 16-column boxes
            const CUtensorMap mo = make_tmap_2d_f32_swz(obase, nx, ny, ld_out * 4, 32, 32, 128);
            cdist_tc_kernel<2, 32><<<grid, THREADS, SMEM, stream>>>(mx, my, mxl, myl, mo, pp);
        } else {
            const CUtensorMap mo = make_tmap_2d_f32_swz(obase, nx, ny, ld_out * 4, 16, 32, 64);
            cdist_tc_kernel<2, 16><<<grid, THREADS, SMEM, stream>>>(mx, my, mxl, myl, mo, pp);
        }
    } else {
        cdist_tc_kernel<1><<<grid, THREADS, SMEM, stream>>>(mx, my, mxl, myl, mx, pp);
    }
    DNDC_LAUNCHED(ctx);
}

}  // namespace dndc
