// raster_io.cpp — write_raster_asc (proj/include/aidw/io.hpp:199-221) for
// the rasters aidw_run_raster produces (writing 16.8M
// "%.17g" values through an ostream is a multi-second host cost).
//
// Same bytes as the reference writer: the five header lines, then one line
// per raster row, values separated by single spaces.  std::to_chars with
// chars_format::general and precision 17 is specified "as if by printf
// %.17g" in the C locale; rows are formatted in parallel on all host
// threads and written in order.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "aidw_capi.h"

namespace {

int fail(aidw_error* err, int code, const std::string& msg) {
    if (err) {
        err->code = code;
        err->index = -1;
        std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
    }
    return code;
}

void put_double(std::string& out, double v) {
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
    out.append(buf, r.ptr);
}

void format_rows(const double* values, size_t ncols, size_t r0, size_t r1, std::string& out) {
    out.clear();
    out.reserve((r1 - r0) * ncols * 24);
    for (size_t r = r0; r < r1; ++r) {
        const double* row = values + r * ncols;
        for (size_t c = 0; c < ncols; ++c) {
            if (c != 0) out.push_back(' ');
            put_double(out, row[c]);
        }
        out.push_back('\n');
    }
}

}  // namespace

extern "C" int aidw_write_raster_asc(const char* path, size_t ncols, size_t nrows,
                                     double xllcorner, double yllcorner, double cellsize,
                                     const double* values, aidw_error* err) {
    try {
        if (!path) return fail(err, AIDW_ERR_INVALID_ARGUMENT, "write_raster_asc: path missing");
        if (ncols * nrows && !values)
            return fail(err, AIDW_ERR_INVALID_ARGUMENT,
                        "write_raster_asc: value count does not match dimensions");
        FILE* f = std::fopen(path, "wb");
        if (!f) return fail(err, AIDW_ERR_RUNTIME, std::string(path) + ": cannot open for writing");
        std::string head = "ncols " + std::to_string(ncols) + "\nnrows " + std::to_string(nrows) +
                           "\nxllcorner ";
        put_double(head, xllcorner);
        head += "\nyllcorner ";
        put_double(head, yllcorner);
        head += "\ncellsize ";
        put_double(head, cellsize);
        head += "\n";
        bool good = std::fwrite(head.data(), 1, head.size(), f) == head.size();
        const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
        const size_t rows_per = std::max<size_t>(1, (1u << 16) / std::max<size_t>(1, ncols));
        std::vector<std::string> bufs(threads);
        for (size_t base = 0; good && base < nrows; base += rows_per * threads) {
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < threads; ++t) {
                const size_t r0 = std::min(nrows, base + t * rows_per);
                const size_t r1 = std::min(nrows, r0 + rows_per);
                pool.emplace_back(format_rows, values, ncols, r0, r1, std::ref(bufs[t]));
            }
            for (auto& th : pool) th.join();
            for (unsigned t = 0; t < threads && good; ++t)
                good = std::fwrite(bufs[t].data(), 1, bufs[t].size(), f) == bufs[t].size();
        }
        good = (std::fclose(f) == 0) && good;
        if (!good) return fail(err, AIDW_ERR_RUNTIME, std::string(path) + ": write failed");
        if (err) {
            err->code = AIDW_OK;
            err->index = -1;
            err->message[0] = '\0';
        }
        return AIDW_OK;
    } catch (const std::exception& e) {
        return fail(err, AIDW_ERR_RUNTIME, e.what());
    }
}
