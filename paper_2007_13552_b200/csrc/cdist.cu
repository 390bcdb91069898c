// cdist.cu -- A3-A7: row norms, the distance tile and the ring exchange.
//
// Reference: detail::row_norms / distance_block / cdist / cdist_xy
// (pairwise.cpp:10-100), matmul_local (ndarray.hpp:400-418), place_chunk
// (tile.hpp:90-107).
//
// f32 (the performance path, small feature counts): a register-blocked FFMA
// tile (128x128 per CTA, 8x8 per thread) computing
//     d = sqrt(max(xn_i + yn_j - 2 * x_i.y_j, 0))
// with the dot product accumulated by a sequential fmaf chain over k -- the
// same chain row_norms_f32 uses, so a row's distance to itself cancels to an
// exact 0 (test_pairwise.cpp:135-144 relies on that).  The epilogue writes the
// column window [col_off, col_off + ny) of an ld_out-wide row block directly
// (place_chunk without the temporary) with streaming (evict-first) vector
// stores.  The feature-rich case (d = 1024, BASELINE config 4) goes to the
// tcgen05 3xTF32 kernel in cdist_tc.cu.
//
// f64: the reference's arithmetic bit for bit (products rounded before adds,
// IEEE sqrt), used by the drop-in f64 API.
#include <algorithm>

#include "common.cuh"

namespace dndc {

bool cdist_tc_eligible(int64_t nx, int64_t ny, int64_t m);
void cdist_tile_tc_f32(dndc_ctx* ctx, const float* x, const float* xn, int64_t nx, const float* y,
                       const float* yn, int64_t ny, int64_t m, float* out, int64_t ld_out,
                       int64_t col_off, int64_t diag_offset, cudaStream_t stream);

// ------------------------------------------------------------- row norms
__global__ void row_norms_f32_kernel(const float* __restrict__ x, int64_t rows, int m,
                                     float* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const float* row = x + i * m;
    float acc = 0.f;
    for (int k = 0; k < m; ++k) acc = fmaf(row[k], row[k], acc);
    out[i] = acc;
}

__global__ void row_norms_f64_kernel(const double* __restrict__ x, int64_t rows, int m,
                                     double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const double* row = x + i * m;
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc = add_rn(acc, mul_rn(row[k], row[k]));
    out[i] = acc;
}

template <typename T>
void row_norms(dndc_ctx* ctx, const T* x, int64_t rows, int64_t m, T* out, cudaStream_t stream) {
    if (rows <= 0) return;
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>(ceil_div(rows, threads));
    if constexpr (sizeof(T) == 4)
        row_norms_f32_kernel<<<blocks, threads, 0, stream>>>(x, rows, static_cast<int>(m), out);
    else
        row_norms_f64_kernel<<<blocks, threads, 0, stream>>>(x, rows, static_cast<int>(m), out);
    DNDC_LAUNCHED(ctx);
}

template void row_norms<float>(dndc_ctx*, const float*, int64_t, int64_t, float*, cudaStream_t);
template void row_norms<double>(dndc_ctx*, const double*, int64_t, int64_t, double*, cudaStream_t);

// --------------------------------------------------------- f32 FFMA tile
namespace ffma {
constexpr int BM = 128, BN = 128, BK = 32, THREADS = 256;
}

// Loads a BK-deep slab of a 128-row operand tile into smem transposed
// ([kk][row], conflict-free stores).  FULL: every row is in bounds.
template <bool FULL>
__device__ __forceinline__ void load_slab(float (*dst)[ffma::BM], const float* __restrict__ src, int64_t rows_left,
                                          int m, int k0, int kc) {
    const int tid = threadIdx.x;
    for (int idx = tid; idx < ffma::BM * kc; idx += ffma::THREADS) {
        const int r = idx & (ffma::BM - 1), kk = idx >> 7;
        dst[kk][r] = (FULL || r < rows_left) ? __ldg(src + static_cast<int64_t>(r) * m + k0 + kk) : 0.f;
    }
}

// acc[i][jp] (column pairs) += x-slab . y-slab over kc features: one FFMA2 with
// x_i broadcast per two outputs.
__device__ __forceinline__ void tile_mainloop(float2 (&acc)[8][4], const float (*xs)[ffma::BM],
                                              const float (*ys)[ffma::BN], int kc) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll 2
    for (int kk = 0; kk < kc; ++kk) {
        const float4 a0 = *reinterpret_cast<const float4*>(&xs[kk][ty * 4]);
        const float4 a1 = *reinterpret_cast<const float4*>(&xs[kk][64 + ty * 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&ys[kk][tx * 4]);
        const float4 b1 = *reinterpret_cast<const float4*>(&ys[kk][64 + tx * 4]);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                             make_float2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(make_float2(a[i], a[i]), b[j], acc[i][j]);
    }
}

// d = sqrt(max(xn_i + yn_j - 2 g_ij, 0)) for the thread's 8x8 outputs, streaming
// stores; FULL = interior tile (no bounds checks), DIAG = the tile meets the
// self block's diagonal (entries j == i + diag_offset written as 0).
template <bool VEC, bool FULL, bool DIAG>
__device__ __forceinline__ void tile_epilogue(const float2 (&acc)[8][4], const float* __restrict__ xn, int64_t nx,
                                              const float* __restrict__ yn, int64_t ny, float* __restrict__ out,
                                              int64_t ld, int64_t row0, int64_t col0, int64_t diag_offset) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float ynv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int cj = j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4;
        ynv[j] = (FULL || col0 + cj < ny) ? __ldg(yn + col0 + cj) : 0.f;
    }
    float* obase = out + row0 * ld + col0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int ri = i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4;
        if (!FULL && row0 + ri >= nx) continue;
        const float xni = __ldg(xn + row0 + ri);
        float* orow = obase + static_cast<int64_t>(ri) * ld;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = h * 64 + tx * 4;
            float v[4];
#pragma unroll
            for (int jp = 0; jp < 2; ++jp) {
                const float2 base =
                    fadd2(make_float2(xni, xni), make_float2(ynv[h * 4 + 2 * jp], ynv[h * 4 + 2 * jp + 1]));
                const float2 sq = ffma2(make_float2(-2.f, -2.f), acc[i][h * 2 + jp], base);
                v[2 * jp] = sqrt_approx(fmaxf(sq.x, 0.f));
                v[2 * jp + 1] = sqrt_approx(fmaxf(sq.y, 0.f));
            }
            if (DIAG) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    if (col0 + c + jj == row0 + ri + diag_offset) v[jj] = 0.f;
            }
            if (VEC && (FULL || col0 + c + 3 < ny)) {
                st_stream4(orow + c, v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    if (FULL || col0 + c + jj < ny) st_stream(orow + c + jj, v[jj]);
            }
        }
    }
}

// One 128x128 output tile (any m: K slabs of BK through shared memory).
template <bool VEC, bool FULL, bool DIAG>
__device__ __forceinline__ void cdist_tile_body(const float* __restrict__ x, const float* __restrict__ xn,
                                                int64_t nx, const float* __restrict__ y,
                                                const float* __restrict__ yn, int64_t ny, int m,
                                                float* __restrict__ out, int64_t ld, int64_t row0, int64_t col0,
                                                int64_t diag_offset, float (*xs)[ffma::BM], float (*ys)[ffma::BN]) {
    using namespace ffma;
    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
    const float* xb = x + row0 * m;
    const float* yb = y + col0 * m;
    for (int k0 = 0; k0 < m; k0 += BK) {
        const int kc = min(BK, m - k0);
        load_slab<FULL>(xs, xb, nx - row0, m, k0, kc);
        load_slab<FULL>(ys, yb, ny - col0, m, k0, kc);
        __syncthreads();
        if (k0 == 0) {
            tile_mainloop(acc, xs, ys, kc);
        } else {
            // continue the same fma chain across slabs (the norms use one chain)
            const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll 2
            for (int kk = 0; kk < kc; ++kk) {
                const float4 a0 = *reinterpret_cast<const float4*>(&xs[kk][ty * 4]);
                const float4 a1 = *reinterpret_cast<const float4*>(&xs[kk][64 + ty * 4]);
                const float4 b0 = *reinterpret_cast<const float4*>(&ys[kk][tx * 4]);
                const float4 b1 = *reinterpret_cast<const float4*>(&ys[kk][64 + tx * 4]);
                const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                     make_float2(b1.z, b1.w)};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(make_float2(a[i], a[i]), b[j], acc[i][j]);
            }
        }
        __syncthreads();
    }
    tile_epilogue<VEC, FULL, DIAG>(acc, xn, nx, yn, ny, out, ld, row0, col0, diag_offset);
}

template <bool VEC>
__global__ void __launch_bounds__(ffma::THREADS)
    cdist_tile_f32_kernel(const float* __restrict__ x, const float* __restrict__ xn, int64_t nx,
                          const float* __restrict__ y, const float* __restrict__ yn, int64_t ny,
                          int m, float* __restrict__ out, int64_t ld, int64_t col_off,
                          int64_t diag_offset, int64_t row_block0) {
    using namespace ffma;
    __shared__ __align__(16) float xs[BK][BM];
    __shared__ __align__(16) float ys[BK][BN];
    const int64_t row0 = (row_block0 + blockIdx.y) * BM;
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * BN;
    const bool full = row0 + BM <= nx && col0 + BN <= ny;
    // does column j == row i + diag_offset occur inside this tile?
    const bool diag = diag_offset >= 0 && col0 < row0 + diag_offset + BM && row0 + diag_offset < col0 + BN;
    float* o = out + col_off;
    if (full && !diag)
        cdist_tile_body<VEC, true, false>(x, xn, nx, y, yn, ny, m, o, ld, row0, col0, diag_offset, xs, ys);
    else if (diag)
        cdist_tile_body<VEC, false, true>(x, xn, nx, y, yn, ny, m, o, ld, row0, col0, diag_offset, xs, ys);
    else
        cdist_tile_body<VEC, false, false>(x, xn, nx, y, yn, ny, m, o, ld, row0, col0, diag_offset, xs, ys);
}

// ------------------------------------------------ f32 persistent row panels
// For m <= 32 (one K slab; BASELINE cfg2 has m = 18) the one-shot tile kernel
// spends its time loading operands it never reuses.  Here a CTA keeps a
// 128-row X slab in shared memory and sweeps PANEL_TILES column tiles of Y,
// prefetching the next Y slab with cp.async while it computes and stores the
// current tile: the output stream (the roofline) never waits on operand loads.
constexpr int PANEL_TILES = 16;

__device__ __forceinline__ void issue_slab_async(float (*dst)[ffma::BM], const float* __restrict__ src, int64_t row0,
                                                 int64_t n, int m) {
    for (int idx = threadIdx.x; idx < ffma::BM * m; idx += ffma::THREADS) {
        const int r = idx & (ffma::BM - 1), kk = idx >> 7;
        const bool in = row0 + r < n;
        const float* g = in ? src + (row0 + r) * m + kk : src;
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&dst[kk][r]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(g), "r"(in ? 4 : 0) : "memory");
    }
}

#ifndef CDIST_PANEL_CTAS
#define CDIST_PANEL_CTAS 2
#endif
template <bool VEC>
__global__ void __launch_bounds__(ffma::THREADS, CDIST_PANEL_CTAS)
    cdist_panel_f32_kernel(const float* __restrict__ x, const float* __restrict__ xn, int64_t nx,
                           const float* __restrict__ y, const float* __restrict__ yn, int64_t ny, int m,
                           float* __restrict__ out, int64_t ld, int64_t col_off, int64_t diag_offset) {
    using namespace ffma;
    extern __shared__ __align__(16) float panel_smem[];
    float(*xs)[BM] = reinterpret_cast<float(*)[BM]>(panel_smem);
    // (no pointer array: indexing one with a runtime value makes the compiler
    // fall back to generic loads)
    auto ys = [&](int b) { return reinterpret_cast<float(*)[BN]>(panel_smem + BK * BM + b * BK * BN); };
    const int64_t nrb = ceil_div(nx, BM), ncb = ceil_div(ny, BN);
    const int64_t per_row = ceil_div(ncb, PANEL_TILES), units = nrb * per_row;
    float* o = out + col_off;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t rb = u / per_row, ct0 = (u % per_row) * PANEL_TILES;
        const int64_t ct1 = min(ct0 + PANEL_TILES, ncb), row0 = rb * BM;
        __syncthreads();  // the previous unit's readers are done with xs / ys
        issue_slab_async(xs, x, row0, nx, m);
        issue_slab_async(ys(0), y, ct0 * BN, ny, m);
        cp_async_commit();
        for (int64_t ct = ct0; ct < ct1; ++ct) {
            const int buf = static_cast<int>((ct - ct0) & 1);
            if (ct + 1 < ct1) {
                issue_slab_async(ys(buf ^ 1), y, (ct + 1) * BN, ny, m);
                cp_async_commit();
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            float2 acc[8][4];
            tile_mainloop(acc, xs, ys(buf), m);
            __syncthreads();  // ys[buf] is refilled at the top of the next tile
            const int64_t col0 = ct * BN;
            const bool full = row0 + BM <= nx && col0 + BN <= ny;
            const bool diag = diag_offset >= 0 && col0 < row0 + diag_offset + BM && row0 + diag_offset < col0 + BN;
            if (full && !diag)
                tile_epilogue<VEC, true, false>(acc, xn, nx, yn, ny, o, ld, row0, col0, diag_offset);
            else if (diag)
                tile_epilogue<VEC, false, true>(acc, xn, nx, yn, ny, o, ld, row0, col0, diag_offset);
            else
                tile_epilogue<VEC, false, false>(acc, xn, nx, yn, ny, o, ld, row0, col0, diag_offset);
        }
    }
}

// ------------------------------------------------------- f64 exact tile
namespace f64t {
constexpr int BM = 64, BN = 64, BK = 16;
}

__global__ void __launch_bounds__(256)
    cdist_tile_f64_kernel(const double* __restrict__ x, const double* __restrict__ xn, int64_t nx,
                          const double* __restrict__ y, const double* __restrict__ yn, int64_t ny,
                          int m, double* __restrict__ out, int64_t ld, int64_t col_off,
                          int64_t diag_offset, int64_t row_block0) {
    using namespace f64t;
    __shared__ double xs[BK][BM + 1];
    __shared__ double ys[BK][BN + 1];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (row_block0 + blockIdx.y) * BM;
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * BN;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < m; k0 += BK) {
        const int kc = min(BK, m - k0);
        for (int idx = tid; idx < BM * kc; idx += 256) {
            const int r = idx % BM, kk = idx / BM;
            const int64_t gr = row0 + r, gc = col0 + r;
            xs[kk][r] = gr < nx ? x[gr * m + k0 + kk] : 0.0;
            ys[kk][r] = gc < ny ? y[gc * m + k0 + kk] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[i][j] = add_rn(acc[i][j], mul_rn(xs[kk][ty + 16 * i], ys[kk][tx + 16 * j]));
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gi = row0 + ty + 16 * i;
        if (gi >= nx) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gj = col0 + tx + 16 * j;
            if (gj >= ny) continue;
            const double d = (diag_offset >= 0 && gj == gi + diag_offset) ? 0.0 : ref_distance(xn[gi], yn[gj], acc[i][j]);
            out[gi * ld + col_off + gj] = d;
        }
    }
}

// ---------------------------------------------------------------- driver
template <typename T>
void cdist_tile(dndc_ctx* ctx, const T* x, const T* xn, int64_t nx, const T* y, const T* yn,
                int64_t ny, int64_t m, T* out, int64_t ld_out, int64_t col_off,
                int64_t diag_offset, cudaStream_t stream) {
    if (nx <= 0 || ny <= 0) return;
    if (m > (1 << 30)) value_error("cdist: feature count too large");
    if constexpr (sizeof(T) == 4) {
        if (cdist_tc_eligible(nx, ny, m)) {
            cdist_tile_tc_f32(ctx, x, xn, nx, y, yn, ny, m, out, ld_out, col_off, diag_offset, stream);
            return;
        }
        const bool vec = (ld_out % 4 == 0) && (col_off % 4 == 0) &&
                         (reinterpret_cast<uintptr_t>(out) % 16 == 0);
        if (m <= ffma::BK) {
            const int64_t units = ceil_div(nx, ffma::BM) * ceil_div(ceil_div(ny, ffma::BN), PANEL_TILES);
            const int grid = static_cast<int>(std::min<int64_t>(units, static_cast<int64_t>(ctx->num_sms) * CDIST_PANEL_CTAS));
            const size_t smem = sizeof(float) * 3 * ffma::BK * ffma::BM;
            if (vec)
                cdist_panel_f32_kernel<true><<<grid, ffma::THREADS, smem, stream>>>(
                    x, xn, nx, y, yn, ny, static_cast<int>(m), out, ld_out, col_off, diag_offset);
            else
                cdist_panel_f32_kernel<false><<<grid, ffma::THREADS, smem, stream>>>(
                    x, xn, nx, y, yn, ny, static_cast<int>(m), out, ld_out, col_off, diag_offset);
            DNDC_LAUNCHED(ctx);
            return;
        }
        const int64_t row_blocks = ceil_div(nx, ffma::BM);
        const unsigned gx = static_cast<unsigned>(ceil_div(ny, ffma::BN));
        for (int64_t rb = 0; rb < row_blocks; rb += 65535) {
            dim3 grid(gx, static_cast<unsigned>(std::min<int64_t>(65535, row_blocks - rb)));
            if (vec)
                cdist_tile_f32_kernel<true><<<grid, ffma::THREADS, 0, stream>>>(
                    x, xn, nx, y, yn, ny, static_cast<int>(m), out, ld_out, col_off, diag_offset, rb);
            else
                cdist_tile_f32_kernel<false><<<grid, ffma::THREADS, 0, stream>>>(
                    x, xn, nx, y, yn, ny, static_cast<int>(m), out, ld_out, col_off, diag_offset, rb);
            DNDC_LAUNCHED(ctx);
        }
    } else {
        const int64_t row_blocks = ceil_div(nx, f64t::BM);
        const unsigned gx = static_cast<unsigned>(ceil_div(ny, f64t::BN));
        for (int64_t rb = 0; rb < row_blocks; rb += 65535) {
            dim3 grid(gx, static_cast<unsigned>(std::min<int64_t>(65535, row_blocks - rb)));
            cdist_tile_f64_kernel<<<grid, 256, 0, stream>>>(x, xn, nx, y, yn, ny, static_cast<int>(m),
                                                           out, ld_out, col_off, diag_offset, rb);
            DNDC_LAUNCHED(ctx);
        }
    }
}

// The ring (pairwise.cpp:54-83): round t computes against the block that
// originated at (rank - t) mod p and fills that origin's column window, while
// the same block is already travelling to rank+1 on the comm stream (double
// buffer: compute reads buf[cur], NCCL receives into buf[1-cur]).  The packet
// is the block's rows followed by their norms, as in pairwise.cpp:73-74.
template <typename T>
void cdist_ring(dndc_ctx* ctx, const T* x_local, int64_t nx_local, const T* y_local,
                int64_t ny_local, int64_t ny_global, int64_t m, T* out, bool self) {
    const int p = ctx->world, r = ctx->rank;
    std::vector<int64_t> yoff, yext;
    chunk_map(ny_global, p, yoff, yext);
    if (ny_local != yext[r])
        value_error("cdist: local block has " + std::to_string(ny_local) + " rows, chunk_map gives " +
                    std::to_string(yext[r]));
    cudaStream_t s = ctx->stream;
    T* xn = static_cast<T*>(ctx->slot("cd_xn", std::max<int64_t>(nx_local, 1) * sizeof(T)));
    row_norms<T>(ctx, x_local, nx_local, m, xn, s);
    if (p == 1) {
        const T* yn = xn;
        if (!self) {
            T* ynb = static_cast<T*>(ctx->slot("cd_yn", std::max<int64_t>(ny_local, 1) * sizeof(T)));
            row_norms<T>(ctx, y_local, ny_local, m, ynb, s);
            yn = ynb;
        }
        cdist_tile<T>(ctx, x_local, xn, nx_local, y_local, yn, ny_local, m, out, ny_global, 0,
                      self ? 0 : -1, s);
        return;
    }
    const int64_t maxext = *std::max_element(yext.begin(), yext.end());
    const size_t pkt = static_cast<size_t>(std::max<int64_t>(maxext, 1)) * (m + 1) * sizeof(T);
    T* buf[2] = {static_cast<T*>(ctx->slot("cd_ring0", pkt)), static_cast<T*>(ctx->slot("cd_ring1", pkt))};
    if (ny_local > 0) {
        DNDC_CUDA(cudaMemcpyAsync(buf[0], y_local, ny_local * m * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (self)
            DNDC_CUDA(cudaMemcpyAsync(buf[0] + ny_local * m, xn, ny_local * sizeof(T),
                                      cudaMemcpyDeviceToDevice, s));
        else
            row_norms<T>(ctx, y_local, ny_local, m, buf[0] + ny_local * m, s);
    }
    const ncclDataType_t dt = sizeof(T) == 4 ? ncclFloat32 : ncclFloat64;
    int origin = r, cur = 0;
    for (int round = 0; round < p; ++round) {
        const int64_t rows = yext[origin];
        const bool more = round + 1 < p;
        if (more) {
            const int src_origin = (origin + p - 1) % p;
            const int64_t in_rows = yext[src_origin];
            if (ctx->group) {
                // ranks sharing GPUs: the packet travels through host memory, before this round's tile
                std::vector<XSend> xs;
                std::vector<XRecv> xr;
                if (rows > 0) xs.push_back({(r + 1) % p, buf[cur], static_cast<size_t>(rows * (m + 1)) * sizeof(T)});
                if (in_rows > 0)
                    xr.push_back({(r + p - 1) % p, buf[1 - cur], static_cast<size_t>(in_rows * (m + 1)) * sizeof(T)});
                xport_exchange(ctx, xs, xr, s);
                DNDC_CUDA(cudaEventRecord(ctx->ev_b, s));
            } else {
            DNDC_CUDA(cudaEventRecord(ctx->ev_a, s));
            DNDC_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0));
            DNDC_NCCL(ncclGroupStart());
            if (rows > 0)
                DNDC_NCCL(ncclSend(buf[cur], rows * (m + 1), dt, (r + 1) % p, ctx->comm, ctx->comm_stream));
            if (in_rows > 0)
                DNDC_NCCL(ncclRecv(buf[1 - cur], in_rows * (m + 1), dt, (r + p - 1) % p, ctx->comm,
                                   ctx->comm_stream));
            DNDC_NCCL(ncclGroupEnd());
            DNDC_CUDA(cudaEventRecord(ctx->ev_b, ctx->comm_stream));
            }
            ctx->counters.sendrecvs++;
        }
        cdist_tile<T>(ctx, x_local, xn, nx_local, buf[cur], buf[cur] + rows * m, rows, m, out,
                      ny_global, yoff[origin], (self && origin == r) ? 0 : -1, s);
        if (more) {
            DNDC_CUDA(cudaStreamWaitEvent(s, ctx->ev_b, 0));
            cur = 1 - cur;
            origin = (origin + p - 1) % p;
        }
    }
}

template <typename T>
void cdist_xy_replicated(dndc_ctx* ctx, const T* x_local, int64_t n_local, const T* y, int64_t ny,
                         int64_t m, T* out) {
    cudaStream_t s = ctx->stream;
    T* xn = static_cast<T*>(ctx->slot("cd_xn", std::max<int64_t>(n_local, 1) * sizeof(T)));
    T* yn = static_cast<T*>(ctx->slot("cd_yn", std::max<int64_t>(ny, 1) * sizeof(T)));
    row_norms<T>(ctx, x_local, n_local, m, xn, s);
    row_norms<T>(ctx, y, ny, m, yn, s);
    cdist_tile<T>(ctx, x_local, xn, n_local, y, yn, ny, m, out, ny, 0, -1, s);
}

}  // namespace dndc

using dndc::guard;

extern "C" {

int dndc_row_norms_f32(dndc_ctx* ctx, const float* x, int64_t rows, int64_t m, float* out) {
    return guard([&] { dndc::row_norms<float>(ctx, x, rows, m, out, ctx->stream); });
}
int dndc_row_norms_f64(dndc_ctx* ctx, const double* x, int64_t rows, int64_t m, double* out) {
    return guard([&] { dndc::row_norms<double>(ctx, x, rows, m, out, ctx->stream); });
}

int dndc_cdist_tile_f32(dndc_ctx* ctx, const float* x, const float* xn, int64_t nx, const float* y,
                        const float* yn, int64_t ny, int64_t m, float* out, int64_t ld_out,
                        int64_t col_off, int64_t diag_offset) {
    return guard([&] {
        dndc::cdist_tile<float>(ctx, x, xn, nx, y, yn, ny, m, out, ld_out, col_off, diag_offset,
                                ctx->stream);
    });
}
int dndc_cdist_tile_f64(dndc_ctx* ctx, const double* x, const double* xn, int64_t nx,
                        const double* y, const double* yn, int64_t ny, int64_t m, double* out,
                        int64_t ld_out, int64_t col_off, int64_t diag_offset) {
    return guard([&] {
        dndc::cdist_tile<double>(ctx, x, xn, nx, y, yn, ny, m, out, ld_out, col_off, diag_offset,
                                 ctx->stream);
    });
}

int dndc_cdist_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, int64_t n_global,
                   int64_t m, float* out) {
    return guard([&] {
        if (n_global == 0) dndc::value_error("cdist: input has no rows");
        dndc::cdist_ring<float>(ctx, x_local, n_local, x_local, n_local, n_global, m, out, true);
    });
}
int dndc_cdist_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, int64_t n_global,
                   int64_t m, double* out) {
    return guard([&] {
        if (n_global == 0) dndc::value_error("cdist: input has no rows");
        dndc::cdist_ring<double>(ctx, x_local, n_local, x_local, n_local, n_global, m, out, true);
    });
}

int dndc_cdist_xy_f32(dndc_ctx* ctx, const float* x_local, int64_t n_local, const float* y,
                      int64_t ny, int64_t m, float* out) {
    return guard([&] { dndc::cdist_xy_replicated<float>(ctx, x_local, n_local, y, ny, m, out); });
}
int dndc_cdist_xy_f64(dndc_ctx* ctx, const double* x_local, int64_t n_local, const double* y,
                      int64_t ny, int64_t m, double* out) {
    return guard([&] { dndc::cdist_xy_replicated<double>(ctx, x_local, n_local, y, ny, m, out); });
}

int dndc_cdist_xy_ring_f32(dndc_ctx* ctx, const float* x_local, int64_t nx_local,
                           const float* y_local, int64_t ny_local, int64_t ny_global, int64_t m,
                           float* out) {
    return guard([&] {
        dndc::cdist_ring<float>(ctx, x_local, nx_local, y_local, ny_local, ny_global, m, out, false);
    });
}

int dndc_cdist_xy_ring_f64(dndc_ctx* ctx, const double* x_local, int64_t nx_local,
                           const double* y_local, int64_t ny_local, int64_t ny_global, int64_t m,
                           double* out) {
    return guard([&] {
        dndc::cdist_ring<double>(ctx, x_local, nx_local, y_local, ny_local, ny_global, m, out, false);
    });
}

}  // extern "C"
