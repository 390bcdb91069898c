// dnd/dataio.hpp -- B200 drop-in for proj/include/dnd/dataio.hpp (dataio.cpp):
// the DNB container ("DNB1", dtype byte, ndim byte, little-endian u64
// extents, row-major payload), loaded straight into the HBM shards.
//
// Same names and contract as the reference (dataio.hpp:18-150): dnb_save /
// dnb_load are collective, split=0 ranks touch only their own byte range
// `header + offset(r) * row_bytes`, other splits go through split=0 and
// resplit, malformed files raise DataError naming the field.  The payload
// moves file <-> HBM through libdndc's pinned double-buffered streamer
// (dndc_file_read_to_device / dndc_file_write_from_device); only the header
// is handled here.
#pragma once

#include <bit>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "dnd/ndarray.hpp"

namespace dnd {

static_assert(std::endian::native == std::endian::little, "DNB containers are little-endian");
static_assert(std::numeric_limits<float>::is_iec559 && std::numeric_limits<double>::is_iec559);

enum class DnbDtype : std::uint8_t { f32 = 1, f64 = 2 };

struct DnbHeader {
    DnbDtype dtype = DnbDtype::f64;
    std::vector<std::uint64_t> extents;

    std::size_t header_bytes() const { return 6 + 8 * extents.size(); }
    std::size_t element_size() const { return dtype == DnbDtype::f32 ? 4 : 8; }
    std::uint64_t payload_elements() const {
        std::uint64_t n = 1;
        for (auto e : extents) n *= e;
        return n;
    }
};

namespace detail {

template <typename T>
constexpr DnbDtype dnb_dtype_of() {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "DNB holds f32 or f64");
    return std::is_same_v<T, float> ? DnbDtype::f32 : DnbDtype::f64;
}

inline const char* dnb_dtype_name(DnbDtype d) { return d == DnbDtype::f32 ? "f32" : "f64"; }

inline std::vector<std::uint8_t> encode_header(const DnbHeader& h) {
    std::vector<std::uint8_t> out{'D', 'N', 'B', '1', static_cast<std::uint8_t>(h.dtype),
                                  static_cast<std::uint8_t>(h.extents.size())};
    for (std::uint64_t e : h.extents)
        for (int b = 0; b < 8; ++b) out.push_back(static_cast<std::uint8_t>(e >> (8 * b)));
    return out;
}

}  // namespace detail

/// Parses and validates the header (dataio.cpp:57-88): DataError on a
/// missing file, bad magic, unknown dtype_code, ndim 0 or truncated extents.
inline DnbHeader dnb_read_header(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw DataError("dnb_read_header: cannot open " + path);
    std::uint8_t fixed[6] = {};
    in.read(reinterpret_cast<char*>(fixed), 6);
    if (in.gcount() != 6) throw DataError("dnb_read_header: " + path + " is shorter than the fixed header");
    if (fixed[0] != 'D' || fixed[1] != 'N' || fixed[2] != 'B' || fixed[3] != '1')
        throw DataError("dnb_read_header: bad magic in " + path + ", expected \"DNB1\"");
    if (fixed[4] != static_cast<std::uint8_t>(DnbDtype::f32) && fixed[4] != static_cast<std::uint8_t>(DnbDtype::f64))
        throw DataError("dnb_read_header: unknown dtype_code " + std::to_string(fixed[4]) + " in " + path);
    if (fixed[5] == 0) throw DataError("dnb_read_header: ndim must be at least 1 in " + path);
    DnbHeader h;
    h.dtype = static_cast<DnbDtype>(fixed[4]);
    std::vector<std::uint8_t> raw(8 * static_cast<std::size_t>(fixed[5]));
    in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
    if (in.gcount() != static_cast<std::streamsize>(raw.size()))
        throw DataError("dnb_read_header: truncated extents in " + path);
    for (std::size_t d = 0; d < fixed[5]; ++d) {
        std::uint64_t e = 0;
        for (int b = 0; b < 8; ++b) e |= static_cast<std::uint64_t>(raw[8 * d + static_cast<std::size_t>(b)]) << (8 * b);
        h.extents.push_back(e);
    }
    return h;
}

/// Collective save (dataio.hpp:61-100): rank 0 writes the header (and the
/// payload of a replicated array), then every split=0 rank writes its rows
/// at its byte offset from HBM; other splits are resplit to 0 first.
template <typename T>
void dnb_save(const DndArray<T>& a, const std::string& path) {
    if (a.split() && *a.split() != 0) return dnb_save(resplit(a, 0), path);
    DnbHeader h;
    h.dtype = detail::dnb_dtype_of<T>();
    h.extents.assign(a.shape().begin(), a.shape().end());
    const Communicator& comm = a.comm();
    if (comm.rank() == 0) {
        const auto bytes = detail::encode_header(h);
        {
            std::ofstream out(path, std::ios::binary | std::ios::trunc);
            if (!out) throw DataError("dnb_save: cannot create " + path);
            out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
            if (!out) throw DataError("dnb_save: write to " + path + " failed");
        }
        if (!a.split() && a.numel_local() > 0)
            detail::check(dndc_file_write_from_device(comm.handle(), path.c_str(), h.header_bytes(), a.device_data(),
                                                      static_cast<std::size_t>(a.numel_local()) * sizeof(T)));
    }
    comm.barrier();
    if (a.split() && a.numel_local() > 0) {
        const index_t row_elems = a.numel_local() / a.lshape()[0];
        const std::uint64_t off =
            h.header_bytes() + static_cast<std::uint64_t>(a.row_offset() * row_elems) * sizeof(T);
        detail::check(dndc_file_write_from_device(comm.handle(), path.c_str(), off, a.device_data(),
                                                  static_cast<std::size_t>(a.numel_local()) * sizeof(T)));
    }
    comm.barrier();
}

/// Collective load (dataio.hpp:102-142): split=0 ranks read only their byte
/// range, straight into HBM; replicated loads read the whole payload; other
/// splits load as split=0 and resplit.
template <typename T>
DndArray<T> dnb_load(const std::string& path, std::optional<int> split, const Communicator& comm) {
    const DnbHeader h = dnb_read_header(path);
    if (h.dtype != detail::dnb_dtype_of<T>())
        throw DataError("dnb_load: dtype_code mismatch: " + path + " holds " + detail::dnb_dtype_name(h.dtype) +
                        ", caller requested " + detail::dnb_dtype_name(detail::dnb_dtype_of<T>()));
    const std::uint64_t want = h.header_bytes() + h.payload_elements() * sizeof(T);
    const std::uint64_t have = std::filesystem::file_size(path);
    if (have != want)
        throw DataError("dnb_load: truncated payload in " + path + ": expected " + std::to_string(want) +
                        " bytes, file has " + std::to_string(have));
    std::vector<index_t> shape(h.extents.begin(), h.extents.end());
    detail::validate_shape_split(shape, split);
    if (split && *split != 0) return resplit(dnb_load<T>(path, 0, comm), split);
    auto a = detail::empty_like_shape<T>(shape, split, comm);
    if (a.numel_local() > 0) {
        const index_t row_elems = a.numel_local() / a.lshape()[0];
        const std::uint64_t off =
            h.header_bytes() + static_cast<std::uint64_t>(a.row_offset() * row_elems) * sizeof(T);
        detail::check(dndc_file_read_to_device(comm.handle(), path.c_str(), off,
                                               static_cast<std::size_t>(a.numel_local()) * sizeof(T),
                                               a.device_data()));
    }
    return a;
}

/// Serial CSV -> 2-D DNB conversion (dataio.cpp:120-166): comma separated,
/// blanks around fields ignored, blank lines skipped, optional header line;
/// parse errors and ragged rows raise DataError with the line number.
inline void csv_to_dnb(const std::string& src_path, const std::string& dst_path, DnbDtype dtype = DnbDtype::f64,
                       bool skip_header = false) {
    std::ifstream in(src_path);
    if (!in) throw DataError("csv_to_dnb: cannot open " + src_path);
    auto is_blank = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
    std::vector<double> values;
    std::uint64_t rows = 0, cols = 0;
    std::string line;
    for (std::size_t line_no = 1; std::getline(in, line); ++line_no) {
        if (skip_header && line_no == 1) continue;
        if (std::all_of(line.begin(), line.end(), is_blank)) continue;
        std::uint64_t fields = 0;
        for (std::size_t start = 0;;) {
            std::size_t end = line.find(',', start);
            const bool last = end == std::string::npos;
            if (last) end = line.size();
            std::size_t lo = start, hi = end;
            while (lo < hi && is_blank(line[lo])) ++lo;
            while (hi > lo && is_blank(line[hi - 1])) --hi;
            double v = 0.0;
            const auto res = std::from_chars(line.data() + lo, line.data() + hi, v);
            if (res.ec != std::errc{} || res.ptr != line.data() + hi)
                throw DataError("csv_to_dnb: line " + std::to_string(line_no) + ", column " +
                                std::to_string(fields + 1) + ": cannot parse \"" + line.substr(lo, hi - lo) +
                                "\" as a number");
            values.push_back(v);
            ++fields;
            if (last) break;
            start = end + 1;
        }
        if (rows == 0) cols = fields;
        else if (fields != cols)
            throw DataError("csv_to_dnb: line " + std::to_string(line_no) + ": expected " + std::to_string(cols) +
                            " columns, got " + std::to_string(fields));
        ++rows;
    }
    if (rows == 0) throw DataError("csv_to_dnb: " + src_path + " holds no data rows");
    DnbHeader h;
    h.dtype = dtype;
    h.extents = {rows, cols};
    const auto head = detail::encode_header(h);
    std::ofstream out(dst_path, std::ios::binary | std::ios::trunc);
    if (!out) throw DataError("csv_to_dnb: cannot create " + dst_path);
    out.write(reinterpret_cast<const char*>(head.data()), static_cast<std::streamsize>(head.size()));
    if (dtype == DnbDtype::f64) {
        out.write(reinterpret_cast<const char*>(values.data()), static_cast<std::streamsize>(values.size() * 8));
    } else {
        const std::vector<float> narrow(values.begin(), values.end());
        out.write(reinterpret_cast<const char*>(narrow.data()), static_cast<std::streamsize>(narrow.size() * 4));
    }
    if (!out) throw DataError("csv_to_dnb: write to " + dst_path + " failed");
}

}  // namespace dnd
