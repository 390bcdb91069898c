// dnd/transport.hpp -- B200 drop-in for proj/include/dnd/transport.hpp.
//
// A rank is a GPU.  run_world(p, body) starts one host thread per rank (rank r
// on device r % #GPUs), each owning a dndc_ctx; `body` runs SPMD exactly as in
// the reference and the first exception of any rank aborts the world and is
// rethrown after join (transport.cpp:166-193).
//   * p <= #GPUs: the device data path (cdist ring, k-means stats, moments,
//     resplit) is NCCL over NVLink plus the NVLink peer exchange of the fused
//     kernels.
//   * p >  #GPUs (the reference's own tests run run_world(3..5)): ranks share
//     GPUs, so their device collectives go through a host loopback group of
//     libdndc (dndc_create_in_group) with the same semantics.
// The reference's host-typed collectives -- send/recv/sendrecv, allreduce with
// a user combiner, allgather_varying, alltoall_varying, barrier
// (transport.hpp:105-194) -- run on an in-process rendezvous of the rank
// threads (detail::HostWorld below): per-rank call indices, kind checks
// (OrderingError), a bounded wait (TimeoutError, WorldOptions::timeout /
// DND_TIMEOUT_SECS) and abort-on-failure.
#pragma once

#include <any>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "dnd/errors.hpp"

namespace dnd {

enum class BackendKind { loopback, external };

/// Per-rank tally of transport calls (transport.hpp:19-27): the device data
/// path's (libdndc) plus the host-typed collectives'.
struct TransportCounters {
    std::uint64_t sends = 0, recvs = 0, sendrecvs = 0, allreduces = 0, allgathers = 0, alltoalls = 0,
                  barriers = 0;
};

struct WorldOptions {
    /// Deadlock-detection timeout for blocking operations.
    std::chrono::milliseconds timeout{30000};

    /// Defaults; DND_TIMEOUT_SECS overrides the timeout (transport.cpp:14-23).
    static WorldOptions from_env() {
        WorldOptions o;
        if (const char* v = std::getenv("DND_TIMEOUT_SECS")) {
            char* end = nullptr;
            const double secs = std::strtod(v, &end);
            if (end != v && secs > 0) o.timeout = std::chrono::milliseconds(static_cast<std::int64_t>(secs * 1000.0));
        }
        return o;
    }
};

namespace detail {

enum class CollectiveKind : std::uint8_t { allreduce, allgather, alltoall, barrier };

inline const char* collective_name(CollectiveKind k) {
    switch (k) {
        case CollectiveKind::allreduce: return "allreduce";
        case CollectiveKind::allgather: return "allgather";
        case CollectiveKind::alltoall: return "alltoall";
        case CollectiveKind::barrier: return "barrier";
    }
    return "collective";
}

/// In-process rendezvous of the rank threads for host-typed payloads.
class HostWorld {
public:
    HostWorld(int size, WorldOptions options)
        : size_(size), timeout_(options.timeout), calls_(static_cast<std::size_t>(size), 0),
          counters_(static_cast<std::size_t>(size)) {}

    int size() const { return size_; }
    TransportCounters& counters(int rank) { return counters_[static_cast<std::size_t>(rank)]; }

    /// Every rank's contribution to this rank's next collective, by rank.
    std::shared_ptr<const std::vector<std::any>> collect(int rank, CollectiveKind kind, std::any mine) {
        std::unique_lock<std::mutex> lock(mu_);
        if (aborted_) throw TransportError("collective on an aborted world");
        const std::uint64_t idx = calls_[static_cast<std::size_t>(rank)]++;
        Round& r = rounds_[idx];
        if (r.arrived == 0) {
            r.kind = kind;
            r.parts = std::make_shared<std::vector<std::any>>(static_cast<std::size_t>(size_));
        } else if (r.kind != kind) {
            r.mismatch = true;
        }
        (*r.parts)[static_cast<std::size_t>(rank)] = std::move(mine);
        ++r.arrived;
        cv_.notify_all();
        wait(lock, [&] { return r.arrived == size_ || r.mismatch; }, collective_name(kind), rank);
        if (r.mismatch) {
            const std::string msg = std::string("collective #") + std::to_string(idx) + ": rank " +
                                    std::to_string(rank) + " entered " + collective_name(kind) +
                                    " but another rank entered " + collective_name(r.kind);
            throw OrderingError(msg);
        }
        auto out = r.parts;
        if (++r.taken == size_) rounds_.erase(idx);
        return out;
    }

    void send(int src, int dst, std::any payload) {
        std::lock_guard<std::mutex> lock(mu_);
        if (aborted_) throw TransportError("send on an aborted world");
        mail_[{src, dst}].push_back(std::move(payload));
        cv_.notify_all();
    }

    std::any recv(int dst, int src) {
        std::unique_lock<std::mutex> lock(mu_);
        auto& q = mail_[{src, dst}];
        wait(lock, [&] { return !q.empty(); }, "recv", dst);
        std::any v = std::move(q.front());
        q.pop_front();
        return v;
    }

    void abort() noexcept {
        std::lock_guard<std::mutex> lock(mu_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    struct Round {
        CollectiveKind kind{};
        int arrived = 0, taken = 0;
        bool mismatch = false;
        std::shared_ptr<std::vector<std::any>> parts;
    };

    template <typename Ready>
    void wait(std::unique_lock<std::mutex>& lock, Ready ready, const char* what, int rank) {
        const auto deadline = std::chrono::steady_clock::now() + timeout_;
        while (!ready() && !aborted_)
            if (cv_.wait_until(lock, deadline) == std::cv_status::timeout && !ready() && !aborted_)
                throw TimeoutError(std::string(what) + ": rank " + std::to_string(rank) + " waited " +
                                   std::to_string(timeout_.count()) + " ms for its peers (deadlock?)");
        if (!ready()) throw TransportError(std::string(what) + ": the world was aborted by a failing rank");
    }

    int size_;
    std::chrono::milliseconds timeout_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool aborted_ = false;
    std::vector<std::uint64_t> calls_;
    std::map<std::uint64_t, Round> rounds_;
    std::map<std::pair<int, int>, std::deque<std::any>> mail_;
    std::vector<TransportCounters> counters_;
};

}  // namespace detail

/// Rank-local handle (transport.hpp:85-217): the rank's GPU context plus the
/// world's host rendezvous.  Copies share both.
class Communicator {
public:
    Communicator(dndc_ctx* ctx, std::shared_ptr<detail::HostWorld> world, int rank)
        : h_(ctx, [](dndc_ctx* c) {
              if (c) dndc_destroy(c);
          }),
          world_(std::move(world)), rank_(rank) {}

    int rank() const { return rank_; }
    int size() const { return world_->size(); }
    dndc_ctx* handle() const { return h_.get(); }
    BackendKind backend() const { return BackendKind::external; }

    /// True when both handles refer to the same rank of the same world.
    bool congruent(const Communicator& other) const { return world_ == other.world_ && rank_ == other.rank_; }

    TransportCounters counters() const {
        dndc_counters c{};
        detail::check(dndc_get_counters(h_.get(), &c));
        const TransportCounters& hc = world_->counters(rank_);
        return TransportCounters{c.sends + hc.sends,           c.recvs + hc.recvs,
                                 c.sendrecvs + hc.sendrecvs,   c.allreduces + hc.allreduces,
                                 c.allgathers + hc.allgathers, c.alltoalls + hc.alltoalls,
                                 c.barriers + hc.barriers};
    }

    /// How the device stats exchange travels (NVLink peer stores, NCCL, or the
    /// host loopback of ranks that share GPUs).
    std::string transport() const { return dndc_transport_status(h_.get()); }

    /// Delivers `payload` to `dest`; FIFO per (source, destination) pair.
    template <typename T>
    void send(int dest, std::vector<T> payload) const {
        check_peer(dest, false, "send");
        world_->counters(rank_).sends++;
        world_->send(rank_, dest, std::any(std::move(payload)));
    }

    /// The next buffer from `src`; TimeoutError on deadlock.
    template <typename T>
    std::vector<T> recv(int src) const {
        check_peer(src, false, "recv");
        world_->counters(rank_).recvs++;
        return take<std::vector<T>>(world_->recv(rank_, src), src);
    }

    /// Ships `payload` to `dest` and returns the buffer `src` sent here; safe
    /// for ring shifts and dest == src == self.
    template <typename T>
    std::vector<T> sendrecv(int dest, std::vector<T> payload, int src) const {
        check_peer(dest, true, "sendrecv");
        check_peer(src, true, "sendrecv");
        world_->counters(rank_).sendrecvs++;
        world_->send(rank_, dest, std::any(std::move(payload)));
        return take<std::vector<T>>(world_->recv(rank_, src), src);
    }

    /// combine(acc, value_r) folded over r = 0..size-1 from `identity`: the
    /// same bits on every rank (transport.hpp:130-148).
    template <typename T, typename Combine>
    T allreduce(const T& local, Combine combine, T identity) const {
        world_->counters(rank_).allreduces++;
        auto all = world_->collect(rank_, detail::CollectiveKind::allreduce, std::any(local));
        T acc = std::move(identity);
        for (int r = 0; r < size(); ++r) {
            const T* v = std::any_cast<T>(&(*all)[static_cast<std::size_t>(r)]);
            if (!v) throw OrderingError("allreduce: payload type mismatch between ranks");
            acc = combine(std::move(acc), *v);
        }
        return acc;
    }

    /// Every rank's buffer (lengths may differ), indexed by source rank.
    template <typename T>
    std::vector<std::vector<T>> allgather_varying(std::vector<T> local) const {
        world_->counters(rank_).allgathers++;
        auto all = world_->collect(rank_, detail::CollectiveKind::allgather, std::any(std::move(local)));
        std::vector<std::vector<T>> out;
        out.reserve(static_cast<std::size_t>(size()));
        for (int r = 0; r < size(); ++r) {
            const auto* v = std::any_cast<std::vector<T>>(&(*all)[static_cast<std::size_t>(r)]);
            if (!v) throw OrderingError("allgather_varying: payload type mismatch between ranks");
            out.push_back(*v);
        }
        return out;
    }

    /// parts[d] goes to rank d; returned[s] is what rank s addressed here.
    template <typename T>
    std::vector<std::vector<T>> alltoall_varying(std::vector<std::vector<T>> parts) const {
        if (static_cast<int>(parts.size()) != size())
            throw ValueError("alltoall_varying: expected " + std::to_string(size()) + " parts, got " +
                             std::to_string(parts.size()));
        world_->counters(rank_).alltoalls++;
        auto all = world_->collect(rank_, detail::CollectiveKind::alltoall, std::any(std::move(parts)));
        std::vector<std::vector<T>> out;
        out.reserve(static_cast<std::size_t>(size()));
        for (int r = 0; r < size(); ++r) {
            const auto* sent = std::any_cast<std::vector<std::vector<T>>>(&(*all)[static_cast<std::size_t>(r)]);
            if (!sent) throw OrderingError("alltoall_varying: payload type mismatch between ranks");
            out.push_back((*sent)[static_cast<std::size_t>(rank_)]);
        }
        return out;
    }

    /// Returns once every rank entered (and this rank's GPU work is done).
    void barrier() const {
        detail::check(dndc_synchronize(h_.get()));
        world_->counters(rank_).barriers++;
        world_->collect(rank_, detail::CollectiveKind::barrier, std::any());
    }

private:
    void check_peer(int peer, bool allow_self, const char* who) const {
        if (peer < 0 || peer >= size())
            throw ValueError(std::string(who) + ": rank " + std::to_string(peer) + " out of range for world size " +
                             std::to_string(size()));
        if (!allow_self && peer == rank_)
            throw ValueError(std::string(who) + ": rank " + std::to_string(peer) + " may not address itself");
    }
    template <typename T>
    T take(std::any m, int src) const {
        T* v = std::any_cast<T>(&m);
        if (!v)
            throw OrderingError("recv: payload from rank " + std::to_string(src) +
                                " does not match the receiver's element type");
        return std::move(*v);
    }

    std::shared_ptr<dndc_ctx> h_;
    std::shared_ptr<detail::HostWorld> world_;
    int rank_;
};

namespace detail {
/// The calling rank thread's communicator (set by run_world): lets the
/// reference's context-free helpers (detail::row_norms, distance_block, the
/// host-tile moments) find the GPU of the rank that calls them.
inline const Communicator*& current_comm() {
    thread_local const Communicator* c = nullptr;
    return c;
}
inline const Communicator& require_current_comm(const char* who) {
    if (!detail::current_comm())
        throw ValueError(std::string(who) + ": call from inside run_world (needs the rank's GPU)");
    return *detail::current_comm();
}

/// Destroys a libdndc loopback group after its contexts.
struct GroupHolder {
    dndc_group* g = nullptr;
    ~GroupHolder() {
        if (g) dndc_group_destroy(g);
    }
};
}  // namespace detail

/// Runs `size` ranks SPMD and joins them (transport.hpp:222-223).  Rank r uses
/// GPU r % #GPUs; with more ranks than GPUs the ranks share GPUs through a
/// host loopback group.  The first failing rank aborts the world; its
/// exception is rethrown after every rank finished.
inline void run_world(int size, const std::function<void(const Communicator&)>& body,
                      WorldOptions options = WorldOptions::from_env()) {
    if (size < 1) throw ValueError("run_world: size must be positive");
    int ndev = 0;
    detail::check(dndc_device_count(&ndev));
    if (ndev < 1) throw DeviceError("run_world: no CUDA device visible");
    const bool shared = size > ndev;
    std::vector<unsigned char> uid(DNDC_UNIQUE_ID_BYTES, 0);
    if (size > 1 && !shared) detail::check(dndc_unique_id(uid.data()));
    detail::GroupHolder group;
    if (shared) detail::check(dndc_group_create(size, options.timeout.count(), &group.g));
    auto world = std::make_shared<detail::HostWorld>(size, options);
    std::exception_ptr first;
    std::mutex mu;
    {
        std::vector<std::thread> ranks;
        for (int r = 0; r < size; ++r) {
            ranks.emplace_back([&, r] {
                try {
                    dndc_ctx* c = nullptr;
                    if (shared)
                        detail::check(dndc_create_in_group(r % ndev, r, group.g, size, &c));
                    else
                        detail::check(dndc_create(r, r, size, size > 1 ? uid.data() : nullptr, &c));
                    Communicator comm(c, world, r);
                    detail::current_comm() = &comm;
                    body(comm);
                    detail::check(dndc_synchronize(comm.handle()));
                    detail::current_comm() = nullptr;
                } catch (...) {
                    detail::current_comm() = nullptr;
                    {
                        std::lock_guard<std::mutex> lock(mu);
                        if (!first) first = std::current_exception();
                    }
                    world->abort();  // wake blocked peers (transport.cpp:181-192)
                    if (group.g) dndc_group_abort(group.g);
                }
            });
        }
        for (auto& t : ranks) t.join();
    }
    if (first) std::rethrow_exception(first);
}

}  // namespace dnd
