#pragma once

// aidw/io.hpp — source-compatible restatement of proj/include/aidw/io.hpp
// (CSV point sets, per-query result CSV, ASCII-grid rasters, grid debug
// dump).  The bulk readers and writers call the
// library's parallel implementations (csrc/io.cpp through the C-ABI): same
// bytes ("%.17g" fields), same headers, same "<path>:<line>: ..." parse
// diagnostics and exception types as the reference.

#include <charconv>
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "aidw/grid.hpp"
#include "aidw/interpolate.hpp"
#include "aidw/types.hpp"
#include "aidw_capi.h"

namespace aidw {

namespace detail {

/// "%.17g": 17 significant digits, so a value survives a write/read round trip.
inline std::string format_double(double value) {
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof(buf), value, std::chars_format::general, 17);
    return std::string(buf, r.ptr);
}

inline std::ofstream open_for_write(const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(path + ": cannot open for writing");
    return out;
}

inline std::ifstream open_for_read(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error(path + ": cannot open for reading");
    return in;
}

inline PointSet read_points(const std::string& path, bool with_values) {
    aidw_points_buffer buf{};
    aidw_error err{};
    raise_if(aidw_read_points_csv(path.c_str(), with_values ? 1 : 0, &buf, &err), err);
    PointSet set;
    set.xs.assign(buf.xs, buf.xs + buf.count);
    set.ys.assign(buf.ys, buf.ys + buf.count);
    if (with_values) set.zs.assign(buf.zs, buf.zs + buf.count);
    aidw_free_points(&buf);
    return set;
}

inline void write_columns(const std::string& path, const char* header, std::size_t rows,
                          std::initializer_list<const double*> cols) {
    std::vector<const double*> c(cols);
    aidw_error err{};
    raise_if(aidw_write_columns_csv(path.c_str(), header, rows, static_cast<int32_t>(c.size()),
                                    c.data(), &err),
             err);
}

}  // namespace detail

/// Data points: header `x,y,z`, one point per line (io.hpp:103-124).
inline PointSet read_data_csv(const std::string& path) { return detail::read_points(path, true); }

/// Query points: header `x,y` (io.hpp:126-145).
inline PointSet read_query_csv(const std::string& path) {
    return detail::read_points(path, false);
}

inline void write_data_csv(const std::string& path, const PointSet& set) {
    if (set.zs.size() != set.xs.size())
        throw std::invalid_argument("write_data_csv: point set carries no values");
    detail::write_columns(path, "x,y,z", set.count(), {set.xs.data(), set.ys.data(), set.zs.data()});
}

inline void write_query_csv(const std::string& path, const PointSet& set) {
    detail::write_columns(path, "x,y", set.count(), {set.xs.data(), set.ys.data()});
}

/// Per-query output: `x,y,alpha,z_pred`, input order (io.hpp:169-188).
inline void write_result_csv(const std::string& path, const PointSet& queries,
                             const InterpolationResult& result) {
    if (result.predicted.size() != queries.count() || result.alphas.size() != queries.count())
        throw std::invalid_argument("write_result_csv: result length does not match queries");
    detail::write_columns(path, "x,y,alpha,z_pred", queries.count(),
                          {queries.xs.data(), queries.ys.data(), result.alphas.data(),
                           result.predicted.data()});
}

/// A regular lattice of interpolated values: row-major, NORTHERNMOST row
/// first (the ASCII-grid convention); cellsize is the spacing along x.
struct Raster {
    std::size_t ncols = 0;
    std::size_t nrows = 0;
    double xllcorner = 0.0;
    double yllcorner = 0.0;
    double cellsize = 0.0;
    std::vector<double> values;
};

inline void write_raster_asc(const std::string& path, const Raster& raster) {
    if (raster.values.size() != raster.ncols * raster.nrows)
        throw std::invalid_argument("write_raster_asc: value count does not match dimensions");
    aidw_error err{};
    detail::raise_if(aidw_write_raster_asc(path.c_str(), raster.ncols, raster.nrows,
                                           raster.xllcorner, raster.yllcorner, raster.cellsize,
                                           raster.values.data(), &err),
                     err);
}

inline Raster parse_raster_asc(const std::string& path) {
    aidw_raster_buffer buf{};
    aidw_error err{};
    detail::raise_if(aidw_read_raster_asc(path.c_str(), &buf, &err), err);
    Raster r;
    r.ncols = buf.ncols;
    r.nrows = buf.nrows;
    r.xllcorner = buf.xllcorner;
    r.yllcorner = buf.yllcorner;
    r.cellsize = buf.cellsize;
    r.values.assign(buf.values, buf.values + buf.count);
    aidw_free_raster(&buf);
    return r;
}

/// Debug dump of the cell layout: `cellId,count,head`, head -1 for empty
/// cells (io.hpp:255-272).  Inspection aid only.
inline void write_grid_debug_csv(const std::string& path, const GridIndex& index) {
    std::string text = "cellId,count,head\n";
    char buf[64];
    for (std::size_t c = 0; c < index.config.cell_total(); ++c) {
        const std::uint32_t count = index.cell_count(c);
        const long long head = count == 0 ? -1 : static_cast<long long>(index.cell_head(c));
        const int len = std::snprintf(buf, sizeof buf, "%zu,%u,%lld\n", c, count, head);
        text.append(buf, static_cast<std::size_t>(len));
    }
    auto out = detail::open_for_write(path);
    out << text;
    if (!out) throw std::runtime_error(path + ": write failed");
}

}  // namespace aidw
