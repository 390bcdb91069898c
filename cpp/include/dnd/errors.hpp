// dnd/errors.hpp -- B200 drop-in for proj/include/dnd/errors.hpp: the same
// exception types, raised from the C-ABI status codes of include/dndc.h.
#pragma once

#include <stdexcept>
#include <string>

#include "dndc.h"

namespace dnd {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// Invalid shapes/arguments (errors.hpp:14-18 of the reference).
struct ValueError : Error {
    using Error::Error;
};
/// Collective/transport failures (errors.hpp:21-25): NCCL or the NVLink exchange.
struct TransportError : Error {
    using Error::Error;
};
/// A blocking transport operation exceeded the deadlock-detection timeout
/// (errors.hpp:27-31; DND_TIMEOUT_SECS, transport.cpp:14-23).
struct TimeoutError : TransportError {
    using TransportError::TransportError;
};
/// Ranks diverged in their sequence of collective calls, or a payload did not
/// match the receiver's type (errors.hpp:33-37).
struct OrderingError : TransportError {
    using TransportError::TransportError;
};
/// Malformed containers and file I/O failures (errors.hpp:40).
struct DataError : Error {
    using Error::Error;
};
/// A CUDA failure inside libdndc (no reference counterpart: the CPU path has none).
struct DeviceError : Error {
    using Error::Error;
};

namespace detail {
inline void check(int rc) {
    if (rc == DNDC_OK) return;
    const std::string msg = dndc_last_error();
    switch (rc) {
        case DNDC_EVALUE: throw ValueError(msg);
        case DNDC_ETRANSPORT: throw TransportError(msg);
        case DNDC_ETIMEOUT: throw TimeoutError(msg);
        case DNDC_EORDERING: throw OrderingError(msg);
        case DNDC_ECUDA: throw DeviceError(msg);
        case DNDC_EDATA: throw DataError(msg);
        default: throw Error(msg);
    }
}
}  // namespace detail
}  // namespace dnd
