// loopback.cu -- the transport for ranks that share GPUs, and the transport
// primitives every collective of the library goes through.
//
// A world whose ranks each own a GPU talks NCCL over NVLink (runtime.cu).  A
// world with more ranks than visible GPUs -- the reference's own tests run
// run_world(3..5) (test_pairwise.cpp:17-101, test_moments.cpp:195) -- cannot:
// NCCL refuses two ranks on one device, and kernels of different ranks that
// wait on each other must not share a GPU.  Such ranks are threads of one
// process (dnd::run_world), so their device collectives are staged through
// host memory in a `dndc_group`: the semantics of the reference's loopback
// world (transport.cpp:64-150): per-rank call indices, a collective completes
// when every rank contributed to the same index, mismatched kinds at one index
// are an OrderingError, every blocking wait is bounded by the world's timeout
// (TimeoutError, transport.cpp:76-93, :123-140), and a failing rank aborts the
// world so blocked peers wake with a TransportError (transport.cpp:174-192).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>

#include "common.cuh"

struct dndc_group {
    int world = 1;
    std::chrono::milliseconds timeout{30000};
    std::mutex mu;
    std::condition_variable cv;
    bool aborted = false;
    struct Slot {
        int kind = -1;
        int arrived = 0;
        int taken = 0;
        bool mismatch = false;
        std::vector<std::vector<char>> parts;
    };
    std::map<uint64_t, Slot> slots;
    std::vector<uint64_t> calls;  // per rank: index of its next collective
    std::map<std::pair<int, int>, std::deque<std::vector<char>>> mail;  // (src, dst) FIFO

    static const char* kind_name(int k) {
        switch (k) {
            case dndc::XK_ALLGATHER: return "allgather";
            case dndc::XK_ALLREDUCE: return "allreduce";
            case dndc::XK_BARRIER: return "barrier";
            default: return "collective";
        }
    }

    template <typename Pred>
    void wait(std::unique_lock<std::mutex>& lock, Pred ready, const char* what, int rank) {
        const auto deadline = std::chrono::steady_clock::now() + timeout;
        while (!ready() && !aborted) {
            if (cv.wait_until(lock, deadline) == std::cv_status::timeout && !ready() && !aborted)
                throw dndc::Error(DNDC_ETIMEOUT, std::string(what) + ": rank " + std::to_string(rank) +
                                                     " timed out after " + std::to_string(timeout.count()) +
                                                     " ms waiting for its peers (deadlock?)");
        }
        if (aborted && !ready())
            throw dndc::Error(DNDC_ETRANSPORT, std::string(what) + ": the world was aborted by a failing rank");
    }

    // Every rank's contribution to this rank's next collective, in rank order.
    std::vector<std::vector<char>> collect(int rank, int kind, const void* data, size_t bytes) {
        std::unique_lock<std::mutex> lock(mu);
        if (aborted) throw dndc::Error(DNDC_ETRANSPORT, "collective on an aborted world");
        const uint64_t idx = calls[rank]++;
        Slot& s = slots[idx];
        if (s.arrived == 0) {
            s.kind = kind;
            s.parts.assign(world, {});
        } else if (s.kind != kind) {
            s.mismatch = true;
        }
        s.parts[rank].assign(static_cast<const char*>(data), static_cast<const char*>(data) + bytes);
        ++s.arrived;
        cv.notify_all();
        wait(lock, [&] { return s.arrived == world || s.mismatch; }, kind_name(kind), rank);
        if (s.mismatch)
            throw dndc::Error(DNDC_EORDERING, std::string("collective #") + std::to_string(idx) + ": rank " +
                                                  std::to_string(rank) + " entered " + kind_name(kind) +
                                                  " while another rank entered " + kind_name(s.kind) +
                                                  " (ranks must call collectives in the same order)");
        std::vector<std::vector<char>> out = s.parts;
        if (++s.taken == world) slots.erase(idx);
        return out;
    }

    void send(int src, int dst, const void* data, size_t bytes) {
        std::lock_guard<std::mutex> lock(mu);
        if (aborted) throw dndc::Error(DNDC_ETRANSPORT, "send on an aborted world");
        mail[{src, dst}].emplace_back(static_cast<const char*>(data), static_cast<const char*>(data) + bytes);
        cv.notify_all();
    }

    std::vector<char> recv(int dst, int src) {
        std::unique_lock<std::mutex> lock(mu);
        auto& q = mail[{src, dst}];
        wait(lock, [&] { return !q.empty(); }, "recv", dst);
        std::vector<char> v = std::move(q.front());
        q.pop_front();
        return v;
    }

    void abort() {
        std::lock_guard<std::mutex> lock(mu);
        aborted = true;
        cv.notify_all();
    }
};

namespace dndc {

static int nccl_kind_ok(dndc_ctx* ctx) { return ctx->world > 1 && ctx->comm != nullptr; }

// ---- the transport primitives (device buffers, ordered on stream s)

void xport_allgather(dndc_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    if (ctx->world == 1) {
        if (recv != send && bytes) DNDC_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (ctx->group) {
        std::vector<char> h(bytes);
        DNDC_CUDA(cudaStreamSynchronize(s));
        if (bytes) DNDC_CUDA(cudaMemcpy(h.data(), send, bytes, cudaMemcpyDeviceToHost));
        const auto all = ctx->group->collect(ctx->rank, XK_ALLGATHER, h.data(), bytes);
        for (int r = 0; r < ctx->world; ++r) {
            if (all[r].size() != bytes)
                throw Error(DNDC_EORDERING, "allgather: ranks contributed different sizes");
            if (bytes)
                DNDC_CUDA(cudaMemcpy(static_cast<char*>(recv) + r * bytes, all[r].data(), bytes, cudaMemcpyHostToDevice));
        }
        return;
    }
    if (!nccl_kind_ok(ctx)) throw Error(DNDC_ETRANSPORT, "allgather: no transport");
    DNDC_NCCL(ncclAllGather(send, recv, bytes, ncclChar, ctx->comm, s));
}

void xport_allreduce_sum_f64(dndc_ctx* ctx, double* buf, size_t count, cudaStream_t s) {
    if (ctx->world == 1) return;
    if (ctx->group) {
        std::vector<double> h(count);
        DNDC_CUDA(cudaStreamSynchronize(s));
        if (count) DNDC_CUDA(cudaMemcpy(h.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost));
        const auto all = ctx->group->collect(ctx->rank, XK_ALLREDUCE, h.data(), count * sizeof(double));
        // rank-order fold from the zero identity (transport.hpp:136-148)
        std::vector<double> acc(count, 0.0);
        for (int r = 0; r < ctx->world; ++r) {
            if (all[r].size() != count * sizeof(double))
                throw Error(DNDC_EORDERING, "allreduce: ranks contributed different sizes");
            const double* v = reinterpret_cast<const double*>(all[r].data());
            for (size_t e = 0; e < count; ++e) acc[e] += v[e];
        }
        if (count) DNDC_CUDA(cudaMemcpy(buf, acc.data(), count * sizeof(double), cudaMemcpyHostToDevice));
        return;
    }
    if (!nccl_kind_ok(ctx)) throw Error(DNDC_ETRANSPORT, "allreduce: no transport");
    DNDC_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, ctx->comm, s));
}

void xport_exchange(dndc_ctx* ctx, const std::vector<XSend>& sends, const std::vector<XRecv>& recvs, cudaStream_t s) {
    if (ctx->group) {
        DNDC_CUDA(cudaStreamSynchronize(s));
        std::vector<char> h;
        for (const XSend& x : sends) {
            h.resize(x.bytes);
            if (x.bytes) DNDC_CUDA(cudaMemcpy(h.data(), x.buf, x.bytes, cudaMemcpyDeviceToHost));
            ctx->group->send(ctx->rank, x.peer, h.data(), x.bytes);
        }
        for (const XRecv& x : recvs) {
            const std::vector<char> v = ctx->group->recv(ctx->rank, x.peer);
            if (v.size() != x.bytes)
                throw Error(DNDC_EORDERING, "recv: " + std::to_string(v.size()) + " bytes from rank " +
                                                std::to_string(x.peer) + ", expected " + std::to_string(x.bytes));
            if (x.bytes) DNDC_CUDA(cudaMemcpy(x.buf, v.data(), x.bytes, cudaMemcpyHostToDevice));
        }
        return;
    }
    if (!nccl_kind_ok(ctx)) throw Error(DNDC_ETRANSPORT, "send/recv: no transport");
    DNDC_NCCL(ncclGroupStart());
    for (const XSend& x : sends)
        if (x.bytes) DNDC_NCCL(ncclSend(x.buf, x.bytes, ncclChar, x.peer, ctx->comm, s));
    for (const XRecv& x : recvs)
        if (x.bytes) DNDC_NCCL(ncclRecv(x.buf, x.bytes, ncclChar, x.peer, ctx->comm, s));
    DNDC_NCCL(ncclGroupEnd());
}

void xport_barrier(dndc_ctx* ctx) {
    DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->world == 1) return;
    if (ctx->group) {
        ctx->group->collect(ctx->rank, XK_BARRIER, nullptr, 0);
        return;
    }
    double* d = static_cast<double*>(ctx->slot("barrier", sizeof(double)));
    DNDC_NCCL(ncclAllReduce(d, d, 1, ncclFloat64, ncclSum, ctx->comm, ctx->stream));
    DNDC_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace dndc

using dndc::guard;

extern "C" {

int dndc_group_create(int world, int64_t timeout_ms, dndc_group** out) {
    return guard([&] {
        if (world < 1) dndc::value_error("dndc_group_create: world must be positive");
        auto g = std::make_unique<dndc_group>();
        g->world = world;
        g->timeout = std::chrono::milliseconds(timeout_ms > 0 ? timeout_ms : 30000);
        g->calls.assign(world, 0);
        *out = g.release();
    });
}

int dndc_group_destroy(dndc_group* g) {
    delete g;
    return DNDC_OK;
}

int dndc_group_abort(dndc_group* g) {
    if (g) g->abort();
    return DNDC_OK;
}

}  // extern "C"
