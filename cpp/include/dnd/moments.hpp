// dnd/moments.hpp -- B200 drop-in for proj/include/dnd/moments.hpp
// (moments.cpp:10-140): single-pass count/mean/M2, Chan merge in rank order.
#pragma once

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <vector>

#include "dnd/ndarray.hpp"

namespace dnd {

struct MomentState {
    std::int64_t count = 0;
    std::vector<double> mean;
    std::vector<double> m2;
    std::size_t arity() const { return mean.size(); }
    static MomentState identity(std::size_t arity) {
        return MomentState{0, std::vector<double>(arity, 0.0), std::vector<double>(arity, 0.0)};
    }
};

/// Chan et al. merge (moments.cpp:69-89); the identity returns the other operand.
inline MomentState combine(const MomentState& a, const MomentState& b) {
    if (a.arity() != b.arity()) throw ValueError("combine: arity mismatch");
    if (a.count == 0) return b;
    if (b.count == 0) return a;
    MomentState o = MomentState::identity(a.arity());
    o.count = a.count + b.count;
    const double na = static_cast<double>(a.count), nb = static_cast<double>(b.count), n = na + nb;
    for (std::size_t i = 0; i < a.arity(); ++i) {
        const double delta = b.mean[i] - a.mean[i];
        o.mean[i] = a.mean[i] + delta * nb / n;
        o.m2[i] = a.m2[i] + b.m2[i] + delta * delta * na * nb / n;
    }
    return o;
}

/// Welford over a host tile, flattened (moments.cpp:91-98).
inline MomentState local_moments(const Tile<double>& t) {
    MomentState s = MomentState::identity(1);
    for (double v : t.data) {
        ++s.count;
        const double d = v - s.mean[0];
        s.mean[0] += d / static_cast<double>(s.count);
        s.m2[0] += d * (v - s.mean[0]);
    }
    return s;
}

/// Welford along `axis` of a 2-D host tile (moments.cpp:100-114): axis 0 gives
/// one state slot per column, axis 1 one per row; count = the axis extent.
inline MomentState local_moments_axis(const Tile<double>& t, int axis) {
    if (t.ndim() != 2 || (axis != 0 && axis != 1)) throw ValueError("local_moments_axis: 2-D tiles, axis 0 or 1");
    const index_t rows = t.extents[0], m = t.extents[1];
    const index_t slots = axis == 0 ? m : rows, extent = axis == 0 ? rows : m;
    MomentState s = MomentState::identity(static_cast<std::size_t>(slots));
    s.count = extent;
    for (index_t c = 0; c < slots; ++c) {
        double mu = 0.0, m2 = 0.0;
        for (index_t r = 0; r < extent; ++r) {
            const double v = axis == 0 ? t.data[static_cast<std::size_t>(r * m + c)]
                                       : t.data[static_cast<std::size_t>(c * m + r)];
            const double d = v - mu;
            mu += d / static_cast<double>(r + 1);
            m2 += d * (v - mu);
        }
        s.mean[static_cast<std::size_t>(c)] = mu;
        s.m2[static_cast<std::size_t>(c)] = m2;
    }
    return s;
}

namespace detail {
inline double variance_from(const MomentState& s, std::size_t i, std::int64_t ddof, const char* who) {
    if (s.count <= ddof) throw ValueError(std::string(who) + ": count must exceed ddof");
    return s.m2[i] / static_cast<double>(s.count - ddof);
}

/// Global state of the array: flattened (axis < 0) or per column (axis 0).
/// Row shards use the device pass + rank-order fold (dndc_moments_axis0_*);
/// replicated arrays are reduced locally like the reference.
template <typename T>
MomentState global_state(const DndArray<T>& a, int axis) {
    if (a.split() && *a.split() != 0) return global_state(resplit(a, 0), axis);
    if (!a.split()) {
        Tile<double> t{a.lshape(), {}};
        const Tile<T> h = a.tile();
        t.data.assign(h.data.begin(), h.data.end());
        if (axis < 0) return local_moments(t);
        return local_moments_axis(t, 0);
    }
    const index_t rows = a.lshape().empty() ? 0 : a.lshape()[0];
    index_t m = 1;
    for (std::size_t i = 1; i < a.shape().size(); ++i) m *= a.shape()[i];
    // flattened: the shard as one column of rows*m values (row-major order)
    const index_t n_arg = axis < 0 ? rows * m : rows, m_arg = axis < 0 ? 1 : m;
    MomentState s = MomentState::identity(static_cast<std::size_t>(m_arg));
    if constexpr (std::is_same_v<T, float>)
        check(dndc_moments_axis0_f32(a.comm().handle(), a.device_data(), n_arg, m_arg, &s.count, s.mean.data(),
                                     s.m2.data()));
    else
        check(dndc_moments_axis0_f64(a.comm().handle(), a.device_data(), n_arg, m_arg, &s.count, s.mean.data(),
                                     s.m2.data()));
    return s;
}

template <typename T>
DndArray<double> replicated_vector(const std::vector<double>& v, const DndArray<T>& like) {
    return from_global(v, {static_cast<index_t>(v.size())}, std::nullopt, like.comm());
}
}  // namespace detail

template <typename T>
double mean(const DndArray<T>& a) {
    return detail::global_state(a, -1).mean[0];
}
template <typename T>
double var(const DndArray<T>& a, std::int64_t ddof = 0) {
    return detail::variance_from(detail::global_state(a, -1), 0, ddof, "var");
}
template <typename T>
double stddev(const DndArray<T>& a, std::int64_t ddof = 0) {
    return std::sqrt(var(a, ddof));
}

namespace detail {
/// The per-row statistic of a 2-D array (axis 1, off the GPU hot path: the
/// reference's axis_statistic, moments.cpp:33-52): each rank reduces its
/// tile's rows; a column split combines the rank states in rank order into a
/// replicated result, a row split keeps the rows split (1-D, split 0).
template <typename T, typename F>
DndArray<double> axis1_statistic(const DndArray<T>& a, F value) {
    const Tile<T> h = a.tile();
    Tile<double> t{h.extents, std::vector<double>(h.data.begin(), h.data.end())};
    MomentState s = local_moments_axis(t, 1);
    if (a.split() == std::optional<int>(1)) {
        s = a.comm().allreduce(
            s, [](MomentState acc, const MomentState& v) { return combine(acc, v); },
            MomentState::identity(s.arity()));
    }
    std::vector<double> out(s.arity());
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = value(s, i);
    const index_t n = a.shape()[0];
    if (a.split() == std::optional<int>(0)) {
        auto r = empty_like_shape<double>({n}, 0, a.comm());
        if (!out.empty())
            check(dndc_memcpy(a.comm().handle(), r.device_data(), out.data(), out.size() * sizeof(double),
                              DNDC_COPY_H2D));
        return r;
    }
    return from_global(out, {n}, std::nullopt, a.comm());
}
}  // namespace detail

/// Along the split axis (axis 0): combined across ranks by the device pass and
/// the rank-order fold, result replicated (moments.cpp:41-52).  Axis 1 of a
/// 2-D array is reduced per row (detail::axis1_statistic).
template <typename T>
DndArray<double> mean_axis(const DndArray<T>& a, int axis) {
    if (a.ndim() != 2 || (axis != 0 && axis != 1)) throw ValueError("mean_axis: axis 0 or 1 of a 2-D array");
    if (axis == 1) return detail::axis1_statistic(a, [](const MomentState& s, std::size_t i) { return s.mean[i]; });
    return detail::replicated_vector(detail::global_state(a, 0).mean, a);
}
template <typename T>
DndArray<double> var_axis(const DndArray<T>& a, int axis, std::int64_t ddof = 0) {
    if (a.ndim() != 2 || (axis != 0 && axis != 1)) throw ValueError("var_axis: axis 0 or 1 of a 2-D array");
    if (axis == 1)
        return detail::axis1_statistic(
            a, [ddof](const MomentState& s, std::size_t i) { return detail::variance_from(s, i, ddof, "var_axis"); });
    const MomentState s = detail::global_state(a, 0);
    std::vector<double> v(s.arity());
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = detail::variance_from(s, i, ddof, "var_axis");
    return detail::replicated_vector(v, a);
}
template <typename T>
DndArray<double> stddev_axis(const DndArray<T>& a, int axis, std::int64_t ddof = 0) {
    if (a.ndim() != 2 || (axis != 0 && axis != 1)) throw ValueError("stddev_axis: axis 0 or 1 of a 2-D array");
    if (axis == 1)
        return detail::axis1_statistic(a, [ddof](const MomentState& s, std::size_t i) {
            return std::sqrt(detail::variance_from(s, i, ddof, "stddev_axis"));
        });
    const MomentState s = detail::global_state(a, 0);
    std::vector<double> v(s.arity());
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sqrt(detail::variance_from(s, i, ddof, "stddev_axis"));
    return detail::replicated_vector(v, a);
}

}  // namespace dnd
