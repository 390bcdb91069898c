// runtime.cu -- rank contexts, errors, workspace and the NCCL transport.
//
// Replaces the reference's loopback world (transport.hpp:85-223,
// transport.cpp:14-193): one dndc_ctx per GPU; world > 1 owns an NCCL
// communicator (NVLink 5 through NVSwitch on an 8xB200 box).  Collectives keep
// the reference's semantics where they are observable:
//   - allreduce folds in rank order 0..p-1 (transport.hpp:136-148): done here
//     as an allgather followed by an explicit rank-order fold on every GPU, so
//     every rank holds bit-identical results (never NCCL's ring order);
//   - sendrecv is a grouped ncclSend/ncclRecv pair (transport.hpp:122-129);
//   - TransportCounters are kept per rank (transport.hpp:19-27).
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace dndc {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& what) { g_last_error = what; }

void chunk_map(int64_t n, int p, std::vector<int64_t>& off, std::vector<int64_t>& ext) {
    if (n < 0) value_error("chunk_map: negative extent " + std::to_string(n));
    if (p < 1) value_error("chunk_map: rank count must be positive, got " + std::to_string(p));
    off.assign(p, 0);
    ext.assign(p, 0);
    const int64_t base = n / p, rem = n % p;
    int64_t o = 0;
    for (int r = 0; r < p; ++r) {
        ext[r] = base + (r < rem ? 1 : 0);
        off[r] = o;
        o += ext[r];
    }
}

void allgather_f64(dndc_ctx* ctx, const double* send, double* recv, size_t count,
                   cudaStream_t stream) {
    if (ctx->world == 1) {
        if (recv != send)
            DNDC_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice,
                                      stream));
        return;
    }
    DNDC_NCCL(ncclAllGather(send, recv, count, ncclFloat64, ctx->comm, stream));
    ctx->counters.allgathers++;
}

void allreduce_sum_f64(dndc_ctx* ctx, double* buf, size_t count, cudaStream_t stream) {
    if (ctx->world == 1) return;
    // Only used where every addend but one is an exact zero (gather_rows,
    // cluster.cpp:27-42), so the sum is exact whatever NCCL's order.
    DNDC_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, ctx->comm, stream));
    ctx->counters.allreduces++;
}

}  // namespace dndc

void* dndc_ctx::slot(const std::string& name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    auto it = slots.find(name);
    if (it != slots.end() && it->second.second >= bytes) return it->second.first;
    if (it != slots.end()) {
        DNDC_CUDA(cudaStreamSynchronize(stream));
        DNDC_CUDA(cudaFree(it->second.first));
        slots.erase(it);
    }
    void* p = nullptr;
    DNDC_CUDA(cudaMalloc(&p, bytes));
    slots[name] = {p, bytes};
    return p;
}

void* dndc_ctx::host_staging(size_t bytes) {
    if (bytes > pinned_bytes) {
        if (pinned) DNDC_CUDA(cudaFreeHost(pinned));
        pinned = nullptr;
        DNDC_CUDA(cudaMallocHost(&pinned, bytes));
        pinned_bytes = bytes;
    }
    return pinned;
}

using dndc::guard;

extern "C" {

int dndc_version(void) { return 1; }

const char* dndc_last_error(void) { return dndc::g_last_error.c_str(); }

int dndc_unique_id(void* id_out) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == DNDC_UNIQUE_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        DNDC_NCCL(ncclGetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int dndc_create(int device, int rank, int world, const void* unique_id, dndc_ctx** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world)
            dndc::value_error("dndc_create: rank " + std::to_string(rank) +
                              " out of range for world size " + std::to_string(world));
        if (world > 1 && unique_id == nullptr)
            dndc::value_error("dndc_create: world > 1 needs a unique id");
        auto ctx = std::make_unique<dndc_ctx>();
        ctx->device = device;
        ctx->rank = rank;
        ctx->world = world;
        DNDC_CUDA(cudaSetDevice(device));
        DNDC_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        DNDC_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        DNDC_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
        DNDC_CUDA(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
        DNDC_CUDA(cudaEventCreateWithFlags(&ctx->ev_b, cudaEventDisableTiming));
        ctx->stream = ctx->own_stream;
        {
            // constant-bank centroid table slot (kmeans.cu), distinct per context
            // on a device for up to DNDC_KM_SLOTS concurrent contexts
            static std::mutex mu;
            static std::map<int, int> next_slot;
            std::lock_guard<std::mutex> lock(mu);
            ctx->km_slot = next_slot[device]++ % 4;
        }
        if (world > 1) {
            ncclUniqueId id;
            std::memcpy(&id, unique_id, sizeof(id));
            DNDC_NCCL(ncclCommInitRank(&ctx->comm, world, id, rank));
        }
        *out = ctx.release();
    });
}

int dndc_destroy(dndc_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        dndc::destroy_kmeans_state(ctx->km);
        for (auto& kv : ctx->slots) cudaFree(kv.second.first);
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        cudaEventDestroy(ctx->ev_a);
        cudaEventDestroy(ctx->ev_b);
        cudaStreamDestroy(ctx->comm_stream);
        cudaStreamDestroy(ctx->own_stream);
        delete ctx;
    });
}

int dndc_set_stream(dndc_ctx* ctx, void* cuda_stream) {
    return guard([&] {
        // NULL is the legacy default stream (torch's default), not our own stream
        ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    });
}

int dndc_rank(const dndc_ctx* ctx) { return ctx->rank; }
int dndc_world(const dndc_ctx* ctx) { return ctx->world; }

int dndc_synchronize(dndc_ctx* ctx) {
    return guard([&] { DNDC_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int dndc_get_counters(const dndc_ctx* ctx, dndc_counters* out) {
    *out = ctx->counters;
    return DNDC_OK;
}

uint64_t dndc_launch_count(const dndc_ctx* ctx) { return ctx->launches; }

int dndc_chunk_map(int64_t n, int world, int64_t* offsets_host, int64_t* extents_host) {
    return guard([&] {
        std::vector<int64_t> off, ext;
        dndc::chunk_map(n, world, off, ext);
        std::memcpy(offsets_host, off.data(), off.size() * sizeof(int64_t));
        std::memcpy(extents_host, ext.data(), ext.size() * sizeof(int64_t));
    });
}

}  // extern "C"
