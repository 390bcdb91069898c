// hostio.cu -- device memory, copies and the generic collectives of the C-ABI,
// so a host layer (the C++ drop-in in cpp/, or any FFI) needs no CUDA headers.
//
// Reference: Tile ownership and gather/resplit (ndarray.hpp:340-393),
// Communicator::allreduce with its rank-order fold (transport.hpp:136-148).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace dndc {

// out[e] = sum over ranks r = 0..world-1 of all[r * count + e], in rank order
// from the zero identity: bit-identical on every rank (transport.hpp:140-146).
__global__ void fold_ranks_kernel(const double* __restrict__ all, int world, int64_t count, double* __restrict__ out) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        for (int r = 0; r < world; ++r) v += all[r * count + e];
        out[e] = v;
    }
}

}  // namespace dndc

using dndc::guard;

extern "C" {

int dndc_device_count(int* out) {
    return guard([&] { DNDC_CUDA(cudaGetDeviceCount(out)); });
}

int dndc_barrier(dndc_ctx* ctx) {
    return guard([&] {
        dndc::xport_barrier(ctx);
        ctx->counters.barriers++;
    });
}

int dndc_alloc(dndc_ctx* ctx, size_t bytes, void** out) {
    return guard([&] {
        DNDC_CUDA(cudaSetDevice(ctx->device));
        *out = nullptr;
        if (!bytes) return;
        if (!ctx->pool) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = ctx->device;
            DNDC_CUDA(cudaMemPoolCreate(&ctx->pool, &props));
            uint64_t keep = UINT64_MAX;  // never release on sync: reuse across calls
            DNDC_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
        cudaError_t e = cudaMallocFromPoolAsync(out, bytes, ctx->pool, ctx->stream);
        if (e == cudaErrorMemoryAllocation) {
            (void)cudaGetLastError();
            ctx->trim_pool();
            e = cudaMallocFromPoolAsync(out, bytes, ctx->pool, ctx->stream);
        }
        DNDC_CUDA(e);
        // usable from any stream and from the host layer's next call at once
        DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int dndc_free(dndc_ctx* ctx, void* p) {
    return guard([&] {
        if (!p) return;
        DNDC_CUDA(cudaSetDevice(ctx->device));
        // ring sends may still read the array on comm_stream
        DNDC_CUDA(cudaStreamSynchronize(ctx->comm_stream));
        DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
        DNDC_CUDA(cudaFreeAsync(p, ctx->stream));
    });
}

int dndc_memcpy(dndc_ctx* ctx, void* dst, const void* src, size_t bytes, int kind) {
    return guard([&] {
        if (kind < DNDC_COPY_H2D || kind > DNDC_COPY_D2D) dndc::value_error("dndc_memcpy: unknown copy kind");
        if (!bytes) return;
        const cudaMemcpyKind k = kind == DNDC_COPY_H2D   ? cudaMemcpyHostToDevice
                                 : kind == DNDC_COPY_D2H ? cudaMemcpyDeviceToHost
                                                         : cudaMemcpyDeviceToDevice;
        DNDC_CUDA(cudaMemcpyAsync(dst, src, bytes, k, ctx->stream));
        DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int dndc_allgather_rows(dndc_ctx* ctx, const void* local, int64_t rows, int64_t row_bytes, void* out_host,
                        int64_t* total_rows) {
    return guard([&] {
        if (rows < 0 || row_bytes < 0) dndc::value_error("dndc_allgather_rows: negative extent");
        const int W = ctx->world;
        cudaStream_t s = ctx->stream;
        if (W == 1) {
            if (rows * row_bytes)
                DNDC_CUDA(cudaMemcpyAsync(out_host, local, rows * row_bytes, cudaMemcpyDeviceToHost, s));
            DNDC_CUDA(cudaStreamSynchronize(s));
            *total_rows = rows;
            return;
        }
        // every rank's row count, then one padded allgather of the blocks
        int64_t* dcnt = static_cast<int64_t*>(ctx->slot("ag_counts", sizeof(int64_t) * (W + 1)));
        DNDC_CUDA(cudaMemcpyAsync(dcnt + W, &rows, sizeof(int64_t), cudaMemcpyHostToDevice, s));
        dndc::xport_allgather(ctx, dcnt + W, dcnt, sizeof(int64_t), s);
        std::vector<int64_t> cnt(W);
        DNDC_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, s));
        DNDC_CUDA(cudaStreamSynchronize(s));
        const int64_t maxr = *std::max_element(cnt.begin(), cnt.end());
        const size_t blk = static_cast<size_t>(std::max<int64_t>(maxr, 1) * row_bytes);
        char* send = static_cast<char*>(ctx->slot("ag_send", blk));
        char* recv = static_cast<char*>(ctx->slot("ag_recv", blk * W));
        if (rows * row_bytes) DNDC_CUDA(cudaMemcpyAsync(send, local, rows * row_bytes, cudaMemcpyDeviceToDevice, s));
        dndc::xport_allgather(ctx, send, recv, blk, s);
        ctx->counters.allgathers++;
        int64_t off = 0;
        for (int r = 0; r < W; ++r) {
            if (cnt[r] * row_bytes)
                DNDC_CUDA(cudaMemcpyAsync(static_cast<char*>(out_host) + off * row_bytes, recv + r * blk,
                                          cnt[r] * row_bytes, cudaMemcpyDeviceToHost, s));
            off += cnt[r];
        }
        DNDC_CUDA(cudaStreamSynchronize(s));
        *total_rows = off;
    });
}

int dndc_allreduce_f64(dndc_ctx* ctx, double* buf, int64_t count) {
    return guard([&] {
        if (count < 0) dndc::value_error("dndc_allreduce_f64: negative count");
        if (ctx->world == 1 || count == 0) return;
        double* all = static_cast<double*>(ctx->slot("ar_all", sizeof(double) * count * ctx->world));
        dndc::xport_allgather(ctx, buf, all, static_cast<size_t>(count) * sizeof(double), ctx->stream);
        const int blocks = static_cast<int>(std::min<int64_t>(dndc::ceil_div(count, 256), 1024));
        dndc::fold_ranks_kernel<<<blocks, 256, 0, ctx->stream>>>(all, ctx->world, count, buf);
        DNDC_LAUNCHED(ctx);
        ctx->counters.allreduces++;
        DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
