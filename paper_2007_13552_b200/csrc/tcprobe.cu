// tcprobe.cu -- self-test of the tcgen05 / TMA plumbing in tc.cuh (not part of
// the dndc.h API; driven by tests/test_gpu_tc.py).  Each mode runs one CTA of
// 128 threads and writes raw results for the host to compare with numpy.
//   mode 0: D[128x16] = A[128x8] . B[16x8]^T, both K-major (one MMA)
//   mode 1: D[128xN]  = A^T . B with A = [K=128 rows x M=128 cols] viewed
//           MN-major and B = [K=128 x N=16] MN-major (16 K-steps)
//   mode 2: TMA 2-D box {4, 128} loads of a [rows x cols] matrix -> raw smem bytes
//   mode 3: as mode 1 with M = 64 (TMEM half-subpartition layout)
#include "common.cuh"
#include "tc.cuh"

namespace dndc {

using namespace tc;

// Write a row-major [R x C] fp32 matrix into the canonical chunked layout.
__device__ void to_chunked(float* dst, const float* src, int R, int C) {
    for (int e = threadIdx.x; e < R * C; e += blockDim.x) {
        const int r = e / C, c = e % C;
        dst[(c / 4) * (R * 4) + r * 4 + (c % 4)] = src[e];
    }
}

__global__ void __launch_bounds__(128) tc_probe_kernel(int mode, const float* a, const float* b, float* d,
                                                      const __grid_constant__ CUtensorMap map, int rows) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    float* sa = reinterpret_cast<float*>(smem);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;

    if (mode == 2) {
        if (threadIdx.x == 0) {
            const int boxes = 10;
            mbar_expect_tx(&bar, boxes * 128 * 16);
            for (int c = 0; c < boxes; ++c) tma_load_2d(sa + c * 512, &map, &bar, c * 4, 0);
        }
        mbar_wait(&bar, 0);
        for (int e = threadIdx.x; e < 10 * 512; e += 128) d[e] = sa[e];
    } else if (mode == 0 || mode == 6 || mode == 7) {
        // mode 6: A stored MN-major ([K=8 rows x M=128] chunked), B K-major
        // mode 7: A K-major, B stored MN-major ([K=8 x N=16] chunked)
        float* sb = sa + 128 * 8;
        if (mode == 6) {
            for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {  // a is [128 x 8] row-major
                const int m = e / 8, k = e % 8;
                sa[(m / 4) * 32 + k * 4 + (m % 4)] = a[e];
            }
        } else {
            to_chunked(sa, a, 128, 8);
        }
        if (mode == 7) {
            for (int e = threadIdx.x; e < 16 * 8; e += blockDim.x) {  // b is [16 x 8] row-major
                const int n = e / 8, k = e % 8;
                sb[(n / 4) * 32 + k * 4 + (n % 4)] = b[e];
            }
        } else {
            to_chunked(sb, b, 16, 8);
        }
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            tc_fence_after();
            const uint64_t ad = mode == 6 ? smem_desc(smem_u32(sa), 128, 128) : smem_desc(smem_u32(sa), 128 * 16, 128);
            const uint64_t bd = mode == 7 ? smem_desc(smem_u32(sb), 128, 128) : smem_desc(smem_u32(sb), 16 * 16, 128);
            mma_tf32(tm, ad, bd, idesc_tf32(128, 16, mode == 6, mode == 7), 0);
            mma_commit(&bar);
        }
        mbar_wait(&bar, 0);
        tc_fence_after();
        float v[16];
        tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16), v);
        for (int j = 0; j < 16; ++j) d[threadIdx.x * 16 + j] = v[j];
    } else {
        // A: [K=128 rows x M cols] chunked (rows are K), B: [K=128 x N=16] chunked
        // mode 1/3: LBO = K-group stride, SBO = MN-group stride; mode 4/5: swapped
        const int M = (mode == 3 || mode == 5) ? 64 : 128;
        const bool swapped = mode >= 4;
        float* sb = sa + 128 * 128;
        to_chunked(sa, a, 128, 128);
        to_chunked(sb, b, 128, 16);
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            tc_fence_after();
            for (int ks = 0; ks < 16; ++ks) {
                const uint32_t kgrp = 128, mngrp = 128 * 16;
                const uint64_t ad = swapped ? smem_desc(smem_u32(sa + ks * 8 * 4), mngrp, kgrp)
                                            : smem_desc(smem_u32(sa + ks * 8 * 4), kgrp, mngrp);
                const uint64_t bd = swapped ? smem_desc(smem_u32(sb + ks * 8 * 4), mngrp, kgrp)
                                            : smem_desc(smem_u32(sb + ks * 8 * 4), kgrp, mngrp);
                mma_tf32(tm, ad, bd, idesc_tf32(M, 16, 1, 1), ks > 0);
            }
            mma_commit(&bar);
        }
        mbar_wait(&bar, 0);
        tc_fence_after();
        float v[16];
        tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16), v);
        for (int j = 0; j < 16; ++j) d[threadIdx.x * 16 + j] = v[j];  // raw lane-major dump
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 128);
}

CUtensorMap make_tmap_2d_f32(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_bytes, uint32_t box_cols,
                             uint32_t box_rows, bool swizzle128) {
    return make_tmap_2d_f32_swz(base, rows, cols, pitch_bytes, box_cols, box_rows, swizzle128 ? 128 : 0);
}

CUtensorMap make_tmap_2d_f32_swz(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_bytes,
                                 uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
    using encode_t = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static encode_t encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        DNDC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw Error(DNDC_ECUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<encode_t>(fn);
    }
    CUtensorMap map;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {pitch_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                              : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                    : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(DNDC_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return map;
}

}  // namespace dndc

extern "C" int dndc_internal_tc_probe(int mode, const float* a, const float* b, float* d, const float* x, int rows,
                                      int cols) {
    return dndc::guard([&] {
        CUtensorMap map{};
        if (mode == 2) map = dndc::make_tmap_2d_f32(x, rows, cols, cols * 4, 4, 128);
        const size_t smem = 160 * 1024;
        DNDC_CUDA(cudaFuncSetAttribute(dndc::tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        dndc::tc_probe_kernel<<<1, 128, smem>>>(mode, a, b, d, map, rows);
        DNDC_CUDA(cudaGetLastError());
        DNDC_CUDA(cudaDeviceSynchronize());
    });
}
