// dnd/pairwise.hpp -- B200 drop-in for proj/include/dnd/pairwise.hpp
// (pairwise.cpp:10-100): cdist through the NCCL ring, cdist_xy, and the two
// detail kernels, on the shards in HBM.  float overloads next to the double
// ones (the hot path computes in fp32; f64 reproduces the reference bitwise).
#pragma once

#include <type_traits>
#include <vector>

#include "dnd/ndarray.hpp"

namespace dnd {

namespace detail {
template <typename T>
void require_2d(const DndArray<T>& a, const char* who) {
    if (a.ndim() != 2) throw ValueError(std::string(who) + ": expects a 2-D array, got " + shape_string(a.shape()));
}
/// This rank's rows of x: its shard (split=0) or its chunk of a replicated x
/// (the reference redistributes such inputs to split=0 first, pairwise.cpp:41).
template <typename T>
const T* rank_rows(const DndArray<T>& x, index_t& rows) {
    if (x.split()) {
        rows = x.lshape()[0];
        return x.device_data();
    }
    const ChunkMap map = chunk_map(x.shape()[0], x.comm().size());
    rows = map.extent(x.comm().rank());
    return x.device_data() + map.offset(x.comm().rank()) * x.shape()[1];
}
}  // namespace detail

/// Pairwise Euclidean distances of the rows of x (pairwise.cpp:37-85): n x n,
/// split=0, exactly p-1 ring exchanges per rank.
template <typename T>
DndArray<T> cdist(const DndArray<T>& x) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "cdist: float or double");
    detail::require_2d(x, "cdist");
    const index_t n = x.shape()[0], m = x.shape()[1];
    if (n == 0) throw ValueError("cdist: empty input");
    if (x.split() && *x.split() != 0) return cdist(resplit(x, 0));  // pairwise.cpp:41
    index_t rows = 0;
    const T* xl = detail::rank_rows(x, rows);
    auto out = detail::empty_like_shape<T>({n, n}, 0, x.comm());
    if constexpr (std::is_same_v<T, float>)
        detail::check(dndc_cdist_f32(x.comm().handle(), xl, rows, n, m, out.device_data()));
    else
        detail::check(dndc_cdist_f64(x.comm().handle(), xl, rows, n, m, out.device_data()));
    detail::check(dndc_synchronize(x.comm().handle()));
    return out;
}

/// Distances between the rows of x (split=0) and y (pairwise.cpp:87-100).
/// y replicated: communication-free.  y split=0: its shards travel the ring
/// (device to device) instead of the reference's allgather.
template <typename T>
DndArray<T> cdist_xy(const DndArray<T>& x, const DndArray<T>& y) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "cdist_xy: float or double");
    detail::require_2d(x, "cdist_xy");
    detail::require_2d(y, "cdist_xy");
    if (x.shape()[1] != y.shape()[1])
        throw ValueError("cdist_xy: feature counts differ (" + std::to_string(x.shape()[1]) + " vs " +
                         std::to_string(y.shape()[1]) + ")");
    // pairwise.cpp:93-94: x to row shards; y other than row shards replicated
    if (x.split() && *x.split() != 0) return cdist_xy(resplit(x, 0), y);
    if (y.split() && *y.split() != 0) return cdist_xy(x, resplit(y, std::nullopt));
    const index_t n = x.shape()[0], ny = y.shape()[0], m = x.shape()[1];
    index_t rows = 0;
    const T* xl = detail::rank_rows(x, rows);
    auto out = detail::empty_like_shape<T>({n, ny}, 0, x.comm());
    dndc_ctx* h = x.comm().handle();
    if (!y.split() || y.comm().size() == 1) {
        if constexpr (std::is_same_v<T, float>)
            detail::check(dndc_cdist_xy_f32(h, xl, rows, y.device_data(), ny, m, out.device_data()));
        else
            detail::check(dndc_cdist_xy_f64(h, xl, rows, y.device_data(), ny, m, out.device_data()));
    } else if constexpr (std::is_same_v<T, float>) {
        detail::check(dndc_cdist_xy_ring_f32(h, xl, rows, y.device_data(), y.lshape()[0], ny, m, out.device_data()));
    } else {
        detail::check(dndc_cdist_xy_ring_f64(h, xl, rows, y.device_data(), y.lshape()[0], ny, m, out.device_data()));
    }
    detail::check(dndc_synchronize(h));
    return out;
}

namespace detail {

/// Squared row norms of a host tile (pairwise.cpp:10-20), computed on the GPU
/// of the calling rank's default context.
inline std::vector<double> row_norms(const Tile<double>& t, const Communicator& comm) {
    if (t.ndim() != 2) throw ValueError("row_norms: expects a 2-D tile");
    const index_t rows = t.extents[0], m = t.extents[1];
    std::vector<double> out(static_cast<std::size_t>(rows));
    if (rows == 0) return out;
    auto dx = device_alloc<double>(comm, rows * m);
    auto dn = device_alloc<double>(comm, rows);
    check(dndc_memcpy(comm.handle(), dx.get(), t.data.data(), t.data.size() * sizeof(double), DNDC_COPY_H2D));
    check(dndc_row_norms_f64(comm.handle(), dx.get(), rows, m, dn.get()));
    check(dndc_memcpy(comm.handle(), out.data(), dn.get(), out.size() * sizeof(double), DNDC_COPY_D2H));
    return out;
}

/// block[i][j] = sqrt(max(na[i] + nb[j] - 2 a_i.b_j, 0)) (pairwise.cpp:22-33).
inline Tile<double> distance_block(const Tile<double>& a, const std::vector<double>& na, const Tile<double>& b,
                                   const std::vector<double>& nb, const Communicator& comm) {
    if (a.ndim() != 2 || b.ndim() != 2 || a.extents[1] != b.extents[1])
        throw ValueError("distance_block: expects 2-D tiles with equal feature counts");
    const index_t nx = a.extents[0], ny = b.extents[0], m = a.extents[1];
    if (static_cast<index_t>(na.size()) != nx || static_cast<index_t>(nb.size()) != ny)
        throw ValueError("distance_block: norm vectors do not match the tiles");
    Tile<double> out{{nx, ny}, std::vector<double>(static_cast<std::size_t>(nx * ny))};
    if (nx * ny == 0) return out;
    auto da = device_alloc<double>(comm, nx * m + nx);
    auto db = device_alloc<double>(comm, ny * m + ny);
    auto dd = device_alloc<double>(comm, nx * ny);
    check(dndc_memcpy(comm.handle(), da.get(), a.data.data(), nx * m * sizeof(double), DNDC_COPY_H2D));
    check(dndc_memcpy(comm.handle(), da.get() + nx * m, na.data(), nx * sizeof(double), DNDC_COPY_H2D));
    check(dndc_memcpy(comm.handle(), db.get(), b.data.data(), ny * m * sizeof(double), DNDC_COPY_H2D));
    check(dndc_memcpy(comm.handle(), db.get() + ny * m, nb.data(), ny * sizeof(double), DNDC_COPY_H2D));
    check(dndc_cdist_tile_f64(comm.handle(), da.get(), da.get() + nx * m, nx, db.get(), db.get() + ny * m, ny, m,
                              dd.get(), ny, 0, -1));
    check(dndc_memcpy(comm.handle(), out.data.data(), dd.get(), out.data.size() * sizeof(double), DNDC_COPY_D2H));
    return out;
}

inline std::vector<double> row_norms(const Tile<double>& t) {
    return row_norms(t, require_current_comm("row_norms"));
}
inline Tile<double> distance_block(const Tile<double>& a, const std::vector<double>& na, const Tile<double>& b,
                                   const std::vector<double>& nb) {
    return distance_block(a, na, b, nb, require_current_comm("distance_block"));
}

}  // namespace detail
}  // namespace dnd
