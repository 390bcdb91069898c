// generate.cu -- A1: the synthetic-data generator, bit-identical to
// dnd::random_uniform<T> (ndarray.hpp:154-169 over generate :118-143, with
// detail::uniform01 / splitmix64 from common.hpp:14-27).
//
// Element (i, f) of the global array has flat index i*m + f; a shard starting
// at global row row0 therefore covers the contiguous flat range
// [row0*m, (row0+rows)*m), so each thread evaluates its element directly.
#include "common.cuh"

namespace dndc {

template <typename T>
__global__ void fill_uniform_kernel(uint64_t seed, uint64_t flat0, int64_t count, T* out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += stride) {
        const double u = uniform01(seed, flat0 + static_cast<uint64_t>(e));
        out[e] = static_cast<T>(u);  // static_cast<float>(double): round to nearest
    }
}

template <typename T>
static void fill_uniform(dndc_ctx* ctx, uint64_t seed, int64_t row0, int64_t rows, int64_t m,
                         T* out) {
    if (rows < 0 || m < 0 || row0 < 0) value_error("fill_uniform: negative extent");
    const int64_t count = rows * m;
    if (count == 0) return;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(count, threads), ctx->num_sms * 16);
    fill_uniform_kernel<T><<<static_cast<unsigned>(blocks), threads, 0, ctx->stream>>>(
        seed, static_cast<uint64_t>(row0) * static_cast<uint64_t>(m), count, out);
    DNDC_LAUNCHED(ctx);
}

}  // namespace dndc

extern "C" {

int dndc_fill_uniform_f32(dndc_ctx* ctx, uint64_t seed, int64_t row0, int64_t rows, int64_t m,
                          float* out) {
    return dndc::guard([&] { dndc::fill_uniform<float>(ctx, seed, row0, rows, m, out); });
}

int dndc_fill_uniform_f64(dndc_ctx* ctx, uint64_t seed, int64_t row0, int64_t rows, int64_t m,
                          double* out) {
    return dndc::guard([&] { dndc::fill_uniform<double>(ctx, seed, row0, rows, m, out); });
}

}  // extern "C"
