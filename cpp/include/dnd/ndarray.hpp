// dnd/ndarray.hpp -- B200 drop-in for proj/include/dnd/ndarray.hpp: the
// distributed array whose rank shard lives in HBM.
//
// Same class name, accessors and factories as the reference (ndarray.hpp:58-96,
// :154-193, :389-393).  Differences a user sees:
//  * the shard is device memory owned by the array (allocated through the
//    C-ABI, freed with the last copy); device_data() exposes it;
//  * tile() returns a HOST copy of the shard by value (the reference returns a
//    reference to its host tile); code that reads tile().data keeps working;
//  * any split axis (or none); the hot-path kernels take row shards, so
//    cdist / kmeans_fit / moments resplit other layouts to split=0 first, as
//    the reference does (pairwise.cpp:41, cluster.cpp:79) -- resplit runs on
//    the GPUs (dndc_resplit: one grouped NCCL exchange);
//  * element types with device kernels: float and double (int32 for labels).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <type_traits>
#include <vector>

#include "dnd/chunking.hpp"
#include "dnd/errors.hpp"
#include "dnd/tile.hpp"
#include "dnd/transport.hpp"

namespace dnd {

namespace detail {

inline std::string shape_string(const std::vector<index_t>& shape) {
    std::string s = "(";
    for (std::size_t i = 0; i < shape.size(); ++i) s += (i ? ", " : "") + std::to_string(shape[i]);
    return s + ")";
}

inline void validate_shape_split(const std::vector<index_t>& shape, std::optional<int> split) {
    for (index_t e : shape)
        if (e < 0) throw ValueError("negative extent in shape " + shape_string(shape));
    if (split && (*split < 0 || *split >= static_cast<int>(shape.size())))
        throw ValueError("split axis " + std::to_string(*split) + " out of range for shape " + shape_string(shape));
}

/// Local extents of this rank's shard (ndarray.hpp local_extents).
inline std::vector<index_t> local_extents(const std::vector<index_t>& shape, std::optional<int> split,
                                         const Communicator& comm) {
    std::vector<index_t> l = shape;
    if (split) l[static_cast<std::size_t>(*split)] = chunk_map(shape[static_cast<std::size_t>(*split)], comm.size())
                                                         .extent(comm.rank());
    return l;
}

/// Rows of this rank and elements per row (product of the trailing extents),
/// for split 0 or none.
inline void local_rows(const std::vector<index_t>& shape, std::optional<int> split, const Communicator& comm,
                       index_t& row0, index_t& rows, index_t& row_elems) {
    const index_t n = shape.empty() ? 1 : shape[0];
    row_elems = 1;
    for (std::size_t i = 1; i < shape.size(); ++i) row_elems *= shape[i];
    if (split) {
        const ChunkMap map = chunk_map(n, comm.size());
        row0 = map.offset(comm.rank());
        rows = map.extent(comm.rank());
    } else {
        row0 = 0;
        rows = n;
    }
}

template <typename T>
std::shared_ptr<T> device_alloc(const Communicator& comm, index_t count) {
    void* p = nullptr;
    check(dndc_alloc(comm.handle(), static_cast<std::size_t>(count) * sizeof(T), &p));
    dndc_ctx* ctx = comm.handle();
    return std::shared_ptr<T>(static_cast<T*>(p), [ctx](T* q) {
        if (q) dndc_free(ctx, q);
    });
}

}  // namespace detail

template <typename T>
class DndArray {
public:
    using value_type = T;

    DndArray(std::vector<index_t> shape, std::optional<int> split, Communicator comm, std::vector<index_t> lshape,
             std::shared_ptr<T> device)
        : shape_(std::move(shape)), split_(split), comm_(std::move(comm)), lshape_(std::move(lshape)),
          dev_(std::move(device)) {}

    const std::vector<index_t>& shape() const { return shape_; }
    std::optional<int> split() const { return split_; }
    const Communicator& comm() const { return comm_; }
    int ndim() const { return static_cast<int>(shape_.size()); }
    const std::vector<index_t>& lshape() const { return lshape_; }
    index_t numel_global() const { return detail::product(shape_); }
    index_t numel_local() const { return detail::product(lshape_); }

    /// The rank's shard in HBM, row-major lshape().
    T* device_data() const { return dev_.get(); }

    /// Host copy of the shard (the reference's tile(), by value).
    Tile<T> tile() const {
        Tile<T> t{lshape_, std::vector<T>(static_cast<std::size_t>(numel_local()))};
        if (!t.data.empty())
            detail::check(dndc_memcpy(comm_.handle(), t.data.data(), dev_.get(), t.data.size() * sizeof(T),
                                      DNDC_COPY_D2H));
        return t;
    }

    ChunkMap split_chunks() const {
        if (!split_) throw ValueError("split_chunks: array is not split");
        return chunk_map(shape_[static_cast<std::size_t>(*split_)], comm_.size());
    }

    /// Row offset of this rank's shard in the global array (0 unless split=0).
    index_t row_offset() const { return split_ == 0 ? split_chunks().offset(comm_.rank()) : 0; }

private:
    std::vector<index_t> shape_;
    std::optional<int> split_;
    Communicator comm_;
    std::vector<index_t> lshape_;
    std::shared_ptr<T> dev_;
};

namespace detail {
template <typename T>
DndArray<T> empty_like_shape(std::vector<index_t> shape, std::optional<int> split, const Communicator& comm) {
    validate_shape_split(shape, split);
    std::vector<index_t> lshape = local_extents(shape, split, comm);
    auto dev = device_alloc<T>(comm, product(lshape));
    return DndArray<T>(std::move(shape), split, comm, std::move(lshape), std::move(dev));
}
}  // namespace detail

/// Same global content on another split axis, or replicated (ndarray.hpp:340-386),
/// moved between the HBM shards by dndc_resplit.
template <typename T>
DndArray<T> resplit(const DndArray<T>& a, std::optional<int> new_split) {
    detail::validate_shape_split(a.shape(), new_split);
    if (a.split() == new_split) return a;
    auto b = detail::empty_like_shape<T>(a.shape(), new_split, a.comm());
    if (a.numel_global() > 0)
        detail::check(dndc_resplit(a.comm().handle(), a.device_data(), a.ndim(), a.shape().data(),
                                   static_cast<std::int64_t>(sizeof(T)), a.split() ? *a.split() : -1,
                                   new_split ? *new_split : -1, b.device_data()));
    return b;
}

// ---------------------------------------------------------------- factories

/// Seed-deterministic uniform values in [0, 1) (ndarray.hpp:154-169): element
/// i*m + f of the global array is static_cast<T>(uniform01(seed, i*m + f)),
/// generated in HBM, bit-identical to the reference for any split / rank count.
template <typename T>
DndArray<T> random_uniform(std::vector<index_t> shape, std::optional<int> split, std::uint64_t seed,
                           const Communicator& comm) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "random_uniform: float or double");
    detail::validate_shape_split(shape, split);
    if (split && *split != 0 && shape.size() > 1)  // generated as row shards, then moved
        return resplit(random_uniform<T>(shape, 0, seed, comm), split);
    auto a = detail::empty_like_shape<T>(shape, split, comm);
    index_t row0, rows, row_elems;
    detail::local_rows(shape, split, comm, row0, rows, row_elems);
    if (rows * row_elems > 0) {
        if constexpr (std::is_same_v<T, float>)
            detail::check(dndc_fill_uniform_f32(comm.handle(), seed, row0, rows, row_elems, a.device_data()));
        else
            detail::check(dndc_fill_uniform_f64(comm.handle(), seed, row0, rows, row_elems, a.device_data()));
        detail::check(dndc_synchronize(comm.handle()));
    }
    return a;
}

/// Every rank passes the same row-major global data and keeps its rows
/// (ndarray.hpp:173-189).
template <typename T>
DndArray<T> from_global(const std::vector<T>& data, std::vector<index_t> shape, std::optional<int> split,
                        const Communicator& comm) {
    detail::validate_shape_split(shape, split);
    if (static_cast<index_t>(data.size()) != detail::product(shape))
        throw ValueError("from_global: data holds " + std::to_string(data.size()) + " elements, shape " +
                         detail::shape_string(shape) + " needs " + std::to_string(detail::product(shape)));
    auto a = detail::empty_like_shape<T>(shape, split, comm);
    if (split && *split != 0) {
        // (outer, extent, inner) view of the split axis: copy this rank's slab
        const std::size_t s = static_cast<std::size_t>(*split);
        index_t outer = 1, inner = 1;
        for (std::size_t i = 0; i < s; ++i) outer *= shape[i];
        for (std::size_t i = s + 1; i < shape.size(); ++i) inner *= shape[i];
        const ChunkMap map = chunk_map(shape[s], comm.size());
        const index_t off = map.offset(comm.rank()), ext = map.extent(comm.rank());
        std::vector<T> local(static_cast<std::size_t>(outer * ext * inner));
        for (index_t o = 0; o < outer; ++o)
            std::copy_n(data.begin() + (o * shape[s] + off) * inner, ext * inner, local.begin() + o * ext * inner);
        if (!local.empty())
            detail::check(dndc_memcpy(comm.handle(), a.device_data(), local.data(), local.size() * sizeof(T),
                                      DNDC_COPY_H2D));
        return a;
    }
    index_t row0, rows, row_elems;
    detail::local_rows(shape, split, comm, row0, rows, row_elems);
    if (rows * row_elems > 0)
        detail::check(dndc_memcpy(comm.handle(), a.device_data(), data.data() + row0 * row_elems,
                                  static_cast<std::size_t>(rows * row_elems) * sizeof(T), DNDC_COPY_H2D));
    return a;
}

/// Array whose element at global index idx is fn(idx) (ndarray.hpp:118-144):
/// evaluated on the host for this rank's slab only, then copied to its shard.
/// (Elementwise ops are outside the GPU hot path.)
template <typename T, typename F>
DndArray<T> generate(std::vector<index_t> shape, std::optional<int> split, const Communicator& comm, F fn) {
    auto a = detail::empty_like_shape<T>(shape, split, comm);
    const std::vector<index_t>& lshape = a.lshape();
    const index_t count = detail::product(lshape);
    if (count == 0) return a;
    index_t off = 0;
    if (split) off = chunk_map(shape[static_cast<std::size_t>(*split)], comm.size()).offset(comm.rank());
    std::vector<T> local(static_cast<std::size_t>(count));
    std::vector<index_t> idx(shape.size(), 0);
    for (index_t e = 0; e < count; ++e) {
        index_t rem = e;
        for (std::size_t d = shape.size(); d-- > 0;) {
            idx[d] = rem % lshape[d];
            rem /= lshape[d];
        }
        if (split) idx[static_cast<std::size_t>(*split)] += off;
        local[static_cast<std::size_t>(e)] = fn(static_cast<const std::vector<index_t>&>(idx));
    }
    detail::check(dndc_memcpy(comm.handle(), a.device_data(), local.data(), local.size() * sizeof(T), DNDC_COPY_H2D));
    return a;
}

/// Constant array (ndarray.hpp:97-112).
template <typename T>
DndArray<T> full(std::vector<index_t> shape, T value, std::optional<int> split, const Communicator& comm) {
    return generate<T>(std::move(shape), split, comm, [value](const std::vector<index_t>&) { return value; });
}
template <typename T>
DndArray<T> zeros(std::vector<index_t> shape, std::optional<int> split, const Communicator& comm) {
    return full<T>(std::move(shape), T(0), split, comm);
}
template <typename T>
DndArray<T> ones(std::vector<index_t> shape, std::optional<int> split, const Communicator& comm) {
    return full<T>(std::move(shape), T(1), split, comm);
}

/// 0, 1, ..., n-1 (ndarray.hpp:146-151).
template <typename T>
DndArray<T> arange(index_t n, std::optional<int> split, const Communicator& comm) {
    return generate<T>({n}, split, comm, [](const std::vector<index_t>& idx) { return static_cast<T>(idx[0]); });
}

/// (rows, m) array whose every row equals `row` (ndarray.hpp:191-200).
template <typename T>
DndArray<T> broadcast_row(const std::vector<T>& row, index_t rows, std::optional<int> split,
                          const Communicator& comm) {
    return generate<T>({rows, static_cast<index_t>(row.size())}, split, comm,
                       [&row](const std::vector<index_t>& idx) { return row[static_cast<std::size_t>(idx[1])]; });
}

/// fn applied to every element (ndarray.hpp:204-209), through the host.
template <typename T, typename F>
DndArray<T> map_elementwise(const DndArray<T>& a, F fn) {
    Tile<T> t = a.tile();
    for (auto& v : t.data) v = fn(v);
    auto b = detail::empty_like_shape<T>(a.shape(), a.split(), a.comm());
    if (!t.data.empty())
        detail::check(dndc_memcpy(a.comm().handle(), b.device_data(), t.data.data(), t.data.size() * sizeof(T),
                                  DNDC_COPY_H2D));
    return b;
}

/// fn of two equally shaped and split arrays (ndarray.hpp:211-225).
template <typename T, typename F>
DndArray<T> zip_elementwise(const DndArray<T>& a, const DndArray<T>& b, F fn) {
    if (a.shape() != b.shape())
        throw ValueError("zip_elementwise: shape mismatch " + detail::shape_string(a.shape()) + " vs " +
                         detail::shape_string(b.shape()));
    if (a.split() != b.split()) throw ValueError("zip_elementwise: split mismatch");
    if (!a.comm().congruent(b.comm()))
        throw ValueError("zip_elementwise: operands live on different communicators");
    Tile<T> t = a.tile();
    const Tile<T> u = b.tile();
    for (std::size_t i = 0; i < t.data.size(); ++i) t.data[i] = fn(t.data[i], u.data[i]);
    auto c = detail::empty_like_shape<T>(a.shape(), a.split(), a.comm());
    if (!t.data.empty())
        detail::check(dndc_memcpy(a.comm().handle(), c.device_data(), t.data.data(), t.data.size() * sizeof(T),
                                  DNDC_COPY_H2D));
    return c;
}

/// Full global content, identical on every rank (ndarray.hpp:389-393).
template <typename T>
std::vector<T> gather(const DndArray<T>& a) {
    if (!a.split()) return a.tile().data;
    if (*a.split() != 0) return resplit(a, std::nullopt).tile().data;
    std::vector<T> out(static_cast<std::size_t>(a.numel_global()));
    index_t row_elems = 1;
    for (std::size_t i = 1; i < a.shape().size(); ++i) row_elems *= a.shape()[i];
    const index_t rows = a.lshape().empty() ? 0 : a.lshape()[0];
    index_t total = 0;
    detail::check(dndc_allgather_rows(a.comm().handle(), a.device_data(), rows,
                                      row_elems * static_cast<index_t>(sizeof(T)), out.data(), &total));
    return out;
}

/// Element type conversion (ndarray.hpp:227-242), through the host.
template <typename To, typename From>
DndArray<To> astype(const DndArray<From>& a) {
    const Tile<From> t = a.tile();
    std::vector<To> conv(t.data.begin(), t.data.end());
    auto b = detail::empty_like_shape<To>(a.shape(), a.split(), a.comm());
    if (!conv.empty())
        detail::check(dndc_memcpy(a.comm().handle(), b.device_data(), conv.data(), conv.size() * sizeof(To),
                                  DNDC_COPY_H2D));
    return b;
}

}  // namespace dnd
