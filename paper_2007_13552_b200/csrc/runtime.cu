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
#include <cstdlib>
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
    xport_allgather(ctx, send, recv, count * sizeof(double), stream);
    ctx->counters.allgathers++;
}

void allreduce_sum_f64(dndc_ctx* ctx, double* buf, size_t count, cudaStream_t stream) {
    if (ctx->world == 1) return;
    // Only used where every addend but one is an exact zero (gather_rows,
    // cluster.cpp:27-42), so the sum is exact whatever NCCL's order.
    xport_allreduce_sum_f64(ctx, buf, count, stream);
    ctx->counters.allreduces++;
}

// Maps every rank's exchange region into every rank (CUDA IPC handles
// allgathered over NCCL).  Any failure leaves ctx->p2p false and the k-means
// stats exchange on the NCCL allgather path; DNDC_P2P=0 forces that path.
static void setup_peer_exchange(dndc_ctx* ctx) {
    const char* env = std::getenv("DNDC_P2P");
    if (env && env[0] == '0') {
        ctx->p2p_status = "disabled by DNDC_P2P=0";
        return;
    }
    const int W = ctx->world;
    cudaStream_t s = ctx->own_stream;
    DNDC_CUDA(cudaMalloc(&ctx->xchg, xchg_bytes(W)));
    DNDC_CUDA(cudaMemsetAsync(ctx->xchg, 0, xchg_bytes(W), s));
    cudaIpcMemHandle_t mine;
    DNDC_CUDA(cudaIpcGetMemHandle(&mine, ctx->xchg));
    char* dh = nullptr;
    DNDC_CUDA(cudaMalloc(&dh, sizeof(cudaIpcMemHandle_t) * W));
    DNDC_CUDA(cudaMemcpyAsync(dh + sizeof(cudaIpcMemHandle_t) * ctx->rank, &mine, sizeof(mine),
                              cudaMemcpyHostToDevice, s));
    // the allgather also orders every rank's zeroing before any peer write
    DNDC_NCCL(ncclAllGather(dh + sizeof(cudaIpcMemHandle_t) * ctx->rank, dh, sizeof(cudaIpcMemHandle_t), ncclChar,
                            ctx->comm, s));
    std::vector<cudaIpcMemHandle_t> all(W);
    DNDC_CUDA(cudaMemcpyAsync(all.data(), dh, sizeof(cudaIpcMemHandle_t) * W, cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    cudaFree(dh);
    ctx->peer_bases.assign(W, nullptr);
    bool ok = true;
    std::string why;
    for (int r = 0; r < W; ++r) {
        if (r == ctx->rank) {
            ctx->peer_bases[r] = ctx->xchg;
            continue;
        }
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            ok = false;
            why = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
            break;
        }
        ctx->peer_bases[r] = p;
    }
    // every rank must agree on the path: AND of the local outcomes
    int* flag = nullptr;
    DNDC_CUDA(cudaMalloc(&flag, sizeof(int)));
    const int v = ok ? 1 : 0;
    DNDC_CUDA(cudaMemcpyAsync(flag, &v, sizeof(int), cudaMemcpyHostToDevice, s));
    DNDC_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, ctx->comm, s));
    int all_ok = 0;
    DNDC_CUDA(cudaMemcpyAsync(&all_ok, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    DNDC_CUDA(cudaStreamSynchronize(s));
    cudaFree(flag);
    if (!all_ok) {
        for (int r = 0; r < W; ++r)
            if (r != ctx->rank && ctx->peer_bases[r]) cudaIpcCloseMemHandle(ctx->peer_bases[r]);
        ctx->peer_bases.clear();
        ctx->p2p_status = ok ? "a peer could not map the exchange regions" : why;
        return;
    }
    DNDC_CUDA(cudaMalloc(&ctx->peer_bases_dev, sizeof(void*) * W));
    DNDC_CUDA(cudaMemcpy(ctx->peer_bases_dev, ctx->peer_bases.data(), sizeof(void*) * W, cudaMemcpyHostToDevice));
    ctx->p2p = true;
    ctx->p2p_status = "nvlink peer exchange";
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
        ++slot_gen;  // a captured graph may hold the old address; a new name cannot be in one
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation && pool) {  // the array pool may hold the memory
        (void)cudaGetLastError();
        trim_pool();
        e = cudaMalloc(&p, bytes);
    }
    DNDC_CUDA(e);
    slots[name] = {p, bytes};
    return p;
}

void dndc_ctx::trim_pool() {
    if (!pool) return;
    DNDC_CUDA(cudaStreamSynchronize(stream));
    DNDC_CUDA(cudaMemPoolTrimTo(pool, 0));
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
            dndc::setup_peer_exchange(ctx.get());
        }
        *out = ctx.release();
    });
}

int dndc_create_in_group(int device, int rank, dndc_group* group, int world, dndc_ctx** out) {
    return guard([&] {
        if (!group) dndc::value_error("dndc_create_in_group: no group");
        if (world < 1 || rank < 0 || rank >= world)
            dndc::value_error("dndc_create_in_group: rank " + std::to_string(rank) + " out of range for world size " +
                              std::to_string(world));
        dndc_ctx* c = nullptr;
        const int rc = dndc_create(device, 0, 1, nullptr, &c);  // a one-rank context on `device` ...
        if (rc != DNDC_OK) throw dndc::Error(rc, dndc_last_error());
        c->rank = rank;  // ... that joins the group's world
        c->world = world;
        c->group = group;
        c->p2p_status = "host loopback (ranks share GPUs)";
        *out = c;
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
        if (ctx->ls_exec) cudaGraphExecDestroy(ctx->ls_exec);
        for (void* b : ctx->io_buf) cudaFreeHost(b);
        for (cudaEvent_t e : ctx->io_ev) cudaEventDestroy(e);
        for (int r = 0; r < static_cast<int>(ctx->peer_bases.size()); ++r)
            if (r != ctx->rank && ctx->peer_bases[r]) cudaIpcCloseMemHandle(ctx->peer_bases[r]);
        if (ctx->peer_bases_dev) cudaFree(ctx->peer_bases_dev);
        if (ctx->xchg) cudaFree(ctx->xchg);
        if (ctx->pool) cudaMemPoolDestroy(ctx->pool);  // released once outstanding arrays are freed
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

const char* dndc_transport_status(const dndc_ctx* ctx) { return ctx->p2p_status.c_str(); }
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
