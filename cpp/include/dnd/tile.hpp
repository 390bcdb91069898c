// dnd/tile.hpp -- host tiles (proj/include/dnd/tile.hpp:16-40): what the
// reference keeps per rank; here a host staging type next to the HBM shard.
#pragma once

#include <cstdint>
#include <vector>

#include "dnd/common.hpp"

namespace dnd {

template <typename T>
struct Tile {
    std::vector<index_t> extents;
    std::vector<T> data;
    int ndim() const { return static_cast<int>(extents.size()); }
    index_t numel() const { return detail::product(extents); }
};

}  // namespace dnd
