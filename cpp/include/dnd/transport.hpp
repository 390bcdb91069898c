// dnd/transport.hpp -- B200 drop-in for proj/include/dnd/transport.hpp.
//
// The reference's Communicator is a rank handle into an in-process loopback
// world of rank threads (transport.hpp:85-217, transport.cpp:166-193).  Here
// a rank is a GPU: run_world(p, body) starts one host thread per GPU (device
// r for rank r), each owning a dndc_ctx with its NCCL communicator over
// NVLink and the peer-mapped exchange region; `body` runs SPMD exactly as in
// the reference, and the first exception of any rank is rethrown after join.
#pragma once

#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dnd/errors.hpp"

namespace dnd {

/// Per-rank tally of transport calls (transport.hpp:19-27).
struct TransportCounters {
    std::uint64_t sends = 0, recvs = 0, sendrecvs = 0, allreduces = 0, allgathers = 0, alltoalls = 0,
                  barriers = 0;
};

class Communicator {
public:
    /// Adopts a rank handle (normally made by run_world).
    explicit Communicator(dndc_ctx* ctx)
        : h_(ctx, [](dndc_ctx* c) {
              if (c) dndc_destroy(c);
          }) {}

    int rank() const { return dndc_rank(h_.get()); }
    int size() const { return dndc_world(h_.get()); }
    dndc_ctx* handle() const { return h_.get(); }

    TransportCounters counters() const {
        dndc_counters c{};
        detail::check(dndc_get_counters(h_.get(), &c));
        return TransportCounters{c.sends, c.recvs, c.sendrecvs, c.allreduces, c.allgathers, c.alltoalls,
                                 c.barriers};
    }
    void barrier() const { detail::check(dndc_barrier(h_.get())); }
    /// How the k-means stats exchange travels (NVLink peer stores or NCCL).
    std::string transport() const { return dndc_transport_status(h_.get()); }

private:
    std::shared_ptr<dndc_ctx> h_;
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
}  // namespace detail

/// One rank per GPU, SPMD (transport.hpp:222-223).  size must not exceed the
/// number of visible GPUs (one NCCL rank per device).
inline void run_world(int size, const std::function<void(const Communicator&)>& body) {
    if (size < 1) throw ValueError("run_world: size must be positive");
    int ndev = 0;
    detail::check(dndc_device_count(&ndev));
    if (size > ndev)
        throw ValueError("run_world: " + std::to_string(size) + " ranks but " + std::to_string(ndev) +
                         " visible GPU(s) (one rank per GPU)");
    std::vector<unsigned char> uid(DNDC_UNIQUE_ID_BYTES, 0);
    if (size > 1) detail::check(dndc_unique_id(uid.data()));
    std::exception_ptr first;
    std::mutex mu;
    std::vector<std::thread> ranks;
    for (int r = 0; r < size; ++r) {
        ranks.emplace_back([&, r] {
            try {
                dndc_ctx* c = nullptr;
                detail::check(dndc_create(r, r, size, size > 1 ? uid.data() : nullptr, &c));
                Communicator comm(c);
                detail::current_comm() = &comm;
                body(comm);
                dndc_synchronize(comm.handle());
                detail::current_comm() = nullptr;
            } catch (...) {
                detail::current_comm() = nullptr;
                std::lock_guard<std::mutex> lock(mu);
                if (!first) first = std::current_exception();
            }
        });
    }
    for (auto& t : ranks) t.join();
    if (first) std::rethrow_exception(first);
}

}  // namespace dnd
