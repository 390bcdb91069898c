// dnd/chunking.hpp -- B200 drop-in for proj/include/dnd/chunking.hpp
// (chunking.cpp:9-30): the balanced chunk map, computed by dndc_chunk_map.
#pragma once

#include <cstdint>
#include <vector>

#include "dnd/common.hpp"
#include "dnd/errors.hpp"

namespace dnd {

struct ChunkMap {
    std::vector<index_t> offsets;
    std::vector<index_t> extents;
    index_t offset(int r) const { return offsets[static_cast<std::size_t>(r)]; }
    index_t extent(int r) const { return extents[static_cast<std::size_t>(r)]; }
    index_t end(int r) const { return offset(r) + extent(r); }
    int size() const { return static_cast<int>(offsets.size()); }
};

/// n / p + (r < n % p) rows per rank, larger chunks on lower ranks.
inline ChunkMap chunk_map(index_t n, int p) {
    if (p < 1) throw ValueError("chunk_map: rank count must be positive");
    ChunkMap m{std::vector<index_t>(static_cast<std::size_t>(p)), std::vector<index_t>(static_cast<std::size_t>(p))};
    detail::check(dndc_chunk_map(n, p, m.offsets.data(), m.extents.data()));
    return m;
}

}  // namespace dnd
