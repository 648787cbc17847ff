// io.cpp — the file formats either side of the AIDW path (SURVEY §8f ranks 2
// and 4), restating proj/include/aidw/io.hpp with the same bytes and the
// same diagnostics, but built for inputs the GPU path digests in
// milliseconds: 1M-16.8M rows.
//
//   CSV point sets   read_data_csv / read_query_csv (io.hpp:103-145): the file
//                    is read once, split at line boundaries into one chunk per
//                    host thread, each chunk parsed with std::from_chars into
//                    its slice of the output (a first pass counts the non-blank
//                    rows of every chunk); the first failing line (smallest
//                    line number) reports exactly the reference's message.
//   CSV writers      write_data_csv / write_query_csv / write_result_csv
//                    (:146-188) and write_raster_asc (:199-221): rows are
//                    formatted in parallel with std::to_chars(general, 17) —
//                    specified as printf("%.17g") — and written in order.
//   raster reader    parse_raster_asc (:223-253): stream-extraction semantics
//                    (whitespace tokens, no inf/nan literals, stop at the first
//                    non-number) over an in-memory buffer.
//
// Host code only; errors map to the C-ABI codes of the reference's exception
// types (runtime_error for I/O and parse failures, invalid_argument for
// non-finite values, io.hpp / types.hpp:146-159).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <system_error>
#include <thread>
#include <vector>

#include "aidw_capi.h"

namespace {

struct IoError {
    int code;
    std::string msg;
};

int fail(aidw_error* err, int code, const std::string& msg) {
    if (err) {
        err->code = code;
        err->index = -1;
        std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
    }
    return code;
}

int ok(aidw_error* err) {
    if (err) {
        err->code = AIDW_OK;
        err->index = -1;
        err->message[0] = '\0';
    }
    return AIDW_OK;
}

unsigned host_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

// ------------------------------------------------------------------ formatting
void put_double(std::string& out, double v) {
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
    out.append(buf, r.ptr);
}

// Rows [0, rows) formatted by `fmt(row, out)` on all host threads, written in
// order after `head`.
template <class RowFmt>
void write_rows(const std::string& path, const std::string& head, size_t rows,
                size_t bytes_per_row, RowFmt fmt) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError{AIDW_ERR_RUNTIME, path + ": cannot open for writing"};
    bool good = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    const unsigned threads = host_threads();
    const size_t per = std::max<size_t>(1, (size_t{1} << 20) / std::max<size_t>(1, bytes_per_row));
    std::vector<std::string> bufs(threads);
    for (size_t base = 0; good && base < rows; base += per * threads) {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < threads; ++t) {
            const size_t r0 = std::min(rows, base + t * per), r1 = std::min(rows, r0 + per);
            pool.emplace_back([&, r0, r1, t] {
                std::string& out = bufs[t];
                out.clear();
                out.reserve((r1 - r0) * bytes_per_row);
                for (size_t r = r0; r < r1; ++r) fmt(r, out);
            });
        }
        for (auto& th : pool) th.join();
        for (unsigned t = 0; t < threads && good; ++t)
            good = std::fwrite(bufs[t].data(), 1, bufs[t].size(), f) == bufs[t].size();
    }
    good = (std::fclose(f) == 0) && good;
    if (!good) throw IoError{AIDW_ERR_RUNTIME, path + ": write failed"};
}

// ------------------------------------------------------------------ parsing
std::string slurp(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError{AIDW_ERR_RUNTIME, path + ": cannot open for reading"};
    std::string s;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, got);
    std::fclose(f);
    return s;
}

bool blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

std::string_view trim(std::string_view t) {  // io.hpp:36-44
    while (!t.empty() && blank(t.front())) t.remove_prefix(1);
    while (!t.empty() && blank(t.back())) t.remove_suffix(1);
    return t;
}

std::string located(const std::string& path, size_t line, const std::string& what) {
    return path + ":" + std::to_string(line) + ": " + what;
}

// One CSV row into exactly `expected` numbers (io.hpp:46-75): fields are
// parsed left to right, so an unparsable field is reported before a wrong
// field count.  Returns an empty string on success, else the message.
std::string parse_row(std::string_view row, int expected, double* out, const std::string& path,
                      size_t line) {
    int found = 0;
    while (true) {
        const size_t comma = row.find(',');
        const std::string_view tok = trim(row.substr(0, comma));
        double v = 0.0;
        const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (tok.empty() || r.ec != std::errc{} || r.ptr != tok.data() + tok.size())
            return located(path, line, "cannot parse number from '" + std::string(tok) + "'");
        if (found < expected) out[found] = v;
        ++found;
        if (comma == std::string_view::npos) break;
        row.remove_prefix(comma + 1);
    }
    if (found != expected)
        return located(path, line, "expected " + std::to_string(expected) + " fields, found " +
                                       std::to_string(found));
    return {};
}

struct Chunk {
    size_t begin = 0, end = 0;  // byte range, starts at a line start
    size_t lines = 0, rows = 0;  // lines / non-blank lines in the range
    size_t first_line = 0, first_row = 0;
    size_t err_line = 0;
    std::string err;
};

// read_data_csv / read_query_csv (io.hpp:103-145) + validate_finite
// (types.hpp:146-159).
void read_points(const std::string& path, int columns, std::vector<double>& xs,
                 std::vector<double>& ys, std::vector<double>& zs) {
    const std::string wanted = columns == 3 ? "x,y,z" : "x,y";
    const std::string text = slurp(path);
    if (text.empty())
        throw IoError{AIDW_ERR_RUNTIME,
                      located(path, 1, "empty file, expected header '" + wanted + "'")};
    const size_t nl = text.find('\n');
    const std::string header = text.substr(0, nl);
    if (std::string(trim(header)) != wanted)
        throw IoError{AIDW_ERR_RUNTIME, located(path, 1, "expected header '" + wanted +
                                                             "', found '" + header + "'")};
    const size_t body = nl == std::string::npos ? text.size() : nl + 1;
    const size_t size = text.size();
    // chunks at line starts
    const unsigned threads = host_threads();
    std::vector<Chunk> ch;
    size_t pos = body;
    const size_t step = std::max<size_t>(1 << 16, (size - body) / threads + 1);
    while (pos < size) {
        size_t e = std::min(size, pos + step);
        if (e < size) {
            const size_t k = text.find('\n', e);
            e = k == std::string::npos ? size : k + 1;
        }
        Chunk c;
        c.begin = pos;
        c.end = e;
        ch.push_back(c);
        pos = e;
    }
    auto each_line = [&](const Chunk& c, auto&& fn) {
        size_t p = c.begin;
        while (p < c.end) {
            size_t q = text.find('\n', p);
            if (q == std::string::npos || q >= c.end) q = c.end;
            const std::string_view line(text.data() + p, (q < c.end && text[q] == '\n') ? q - p : q - p);
            if (!fn(line)) return;
            p = q + 1;
        }
    };
    auto run = [&](auto&& body_fn) {
        std::vector<std::thread> pool;
        for (size_t i = 0; i < ch.size(); ++i) pool.emplace_back(body_fn, i);
        for (auto& t : pool) t.join();
    };
    run([&](size_t i) {
        Chunk& c = ch[i];
        each_line(c, [&](std::string_view line) {
            ++c.lines;
            if (!trim(line).empty()) ++c.rows;
            return true;
        });
    });
    size_t line_no = 2, row_no = 0;
    for (Chunk& c : ch) {
        c.first_line = line_no;
        c.first_row = row_no;
        line_no += c.lines;
        row_no += c.rows;
    }
    xs.assign(row_no, 0.0);
    ys.assign(row_no, 0.0);
    zs.assign(columns == 3 ? row_no : 0, 0.0);
    run([&](size_t i) {
        Chunk& c = ch[i];
        size_t ln = c.first_line, r = c.first_row;
        each_line(c, [&](std::string_view line) {
            const size_t this_line = ln++;
            if (trim(line).empty()) return true;
            double v[3] = {0.0, 0.0, 0.0};
            std::string e = parse_row(line, columns, v, path, this_line);
            if (!e.empty()) {
                c.err_line = this_line;
                c.err = std::move(e);
                return false;
            }
            xs[r] = v[0];
            ys[r] = v[1];
            if (columns == 3) zs[r] = v[2];
            ++r;
            return true;
        });
    });
    for (const Chunk& c : ch)
        if (!c.err.empty()) throw IoError{AIDW_ERR_RUNTIME, c.err};
    for (size_t i = 0; i < xs.size(); ++i)
        if (!std::isfinite(xs[i]) || !std::isfinite(ys[i]))
            throw IoError{AIDW_ERR_INVALID_ARGUMENT,
                          path + ": non-finite coordinate at point " + std::to_string(i)};
    for (size_t i = 0; i < zs.size(); ++i)
        if (!std::isfinite(zs[i]))
            throw IoError{AIDW_ERR_INVALID_ARGUMENT,
                          path + ": non-finite value at point " + std::to_string(i)};
}

// `in >> value` over a buffer: whitespace-separated, optional sign, no
// inf / nan literals, out-of-range fails; a token's trailing non-number text
// is left for the next extraction.  Returns false at EOF or failure.
bool extract_double(const char*& p, const char* end, double& v) {
    while (p < end && std::isspace(static_cast<unsigned char>(*p))) ++p;
    if (p >= end) return false;
    const char* s = p;
    bool neg = false;
    if (*s == '+' || *s == '-') neg = *s++ == '-';
    if (s >= end || !(std::isdigit(static_cast<unsigned char>(*s)) || *s == '.')) return false;
    double x = 0.0;
    const auto r = std::from_chars(s, end, x);
    if (r.ec != std::errc{}) return false;
    v = neg ? -x : x;
    p = r.ptr;
    return true;
}

bool extract_token(const char*& p, const char* end, std::string& tok) {
    while (p < end && std::isspace(static_cast<unsigned char>(*p))) ++p;
    const char* s = p;
    while (p < end && !std::isspace(static_cast<unsigned char>(*p))) ++p;
    tok.assign(s, p);
    return p > s;
}

}  // namespace

extern "C" {

int aidw_read_points_csv(const char* path, int32_t with_values, aidw_points_buffer* out,
                         aidw_error* err) {
    try {
        if (!path || !out) return fail(err, AIDW_ERR_INVALID_ARGUMENT, "read_points_csv: null argument");
        std::vector<double> xs, ys, zs;
        read_points(path, with_values ? 3 : 2, xs, ys, zs);
        out->count = xs.size();
        auto dup = [](const std::vector<double>& v) -> double* {
            double* p = static_cast<double*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(double)));
            if (!p) throw std::bad_alloc();
            if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(double));
            return p;
        };
        out->xs = dup(xs);
        out->ys = dup(ys);
        out->zs = with_values ? dup(zs) : nullptr;
        return ok(err);
    } catch (const IoError& e) {
        return fail(err, e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(err, AIDW_ERR_RUNTIME, e.what());
    }
}

void aidw_free_points(aidw_points_buffer* buf) {
    if (!buf) return;
    std::free(buf->xs);
    std::free(buf->ys);
    std::free(buf->zs);
    buf->xs = buf->ys = buf->zs = nullptr;
    buf->count = 0;
}

int aidw_write_columns_csv(const char* path, const char* header, size_t rows, int32_t ncols,
                           const double* const* cols, aidw_error* err) {
    try {
        if (!path || !header || ncols < 1 || ncols > 8 || (rows && !cols))
            return fail(err, AIDW_ERR_INVALID_ARGUMENT, "write_columns_csv: bad arguments");
        write_rows(path, std::string(header) + "\n", rows, 24 * static_cast<size_t>(ncols),
                   [&](size_t r, std::string& out) {
                       for (int c = 0; c < ncols; ++c) {
                           if (c) out.push_back(',');
                           put_double(out, cols[c][r]);
                       }
                       out.push_back('\n');
                   });
        return ok(err);
    } catch (const IoError& e) {
        return fail(err, e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(err, AIDW_ERR_RUNTIME, e.what());
    }
}

int aidw_write_raster_asc(const char* path, size_t ncols, size_t nrows, double xllcorner,
                          double yllcorner, double cellsize, const double* values,
                          aidw_error* err) {
    try {
        if (!path) return fail(err, AIDW_ERR_INVALID_ARGUMENT, "write_raster_asc: path missing");
        if (ncols * nrows && !values)
            return fail(err, AIDW_ERR_INVALID_ARGUMENT,
                        "write_raster_asc: value count does not match dimensions");
        std::string head = "ncols " + std::to_string(ncols) + "\nnrows " + std::to_string(nrows) +
                           "\nxllcorner ";
        put_double(head, xllcorner);
        head += "\nyllcorner ";
        put_double(head, yllcorner);
        head += "\ncellsize ";
        put_double(head, cellsize);
        head += "\n";
        write_rows(path, head, nrows, 24 * std::max<size_t>(1, ncols),
                   [&](size_t r, std::string& out) {
                       const double* row = values + r * ncols;
                       for (size_t c = 0; c < ncols; ++c) {
                           if (c) out.push_back(' ');
                           put_double(out, row[c]);
                       }
                       out.push_back('\n');
                   });
        return ok(err);
    } catch (const IoError& e) {
        return fail(err, e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(err, AIDW_ERR_RUNTIME, e.what());
    }
}

int aidw_read_raster_asc(const char* path, aidw_raster_buffer* out, aidw_error* err) {
    try {
        if (!path || !out) return fail(err, AIDW_ERR_INVALID_ARGUMENT, "read_raster_asc: null argument");
        const std::string p(path);
        const std::string text = slurp(p);
        const char* c = text.data();
        const char* end = c + text.size();
        size_t line = 0;
        std::string key;
        auto header = [&](const char* wanted) {
            ++line;
            double v = 0.0;
            if (!extract_token(c, end, key) || !extract_double(c, end, v) || key != wanted)
                throw IoError{AIDW_ERR_RUNTIME, located(p, line, std::string("expected header line '") +
                                                                     wanted + " <value>'")};
            return v;
        };
        const size_t ncols = static_cast<size_t>(header("ncols"));
        const size_t nrows = static_cast<size_t>(header("nrows"));
        const double xll = header("xllcorner"), yll = header("yllcorner"), cell = header("cellsize");
        std::vector<double> vals;
        vals.reserve(ncols * nrows);
        double v = 0.0;
        while (extract_double(c, end, v)) vals.push_back(v);
        if (vals.size() != ncols * nrows)
            throw IoError{AIDW_ERR_RUNTIME,
                          located(p, line, "expected " + std::to_string(ncols * nrows) +
                                               " values, found " + std::to_string(vals.size()))};
        out->ncols = ncols;
        out->nrows = nrows;
        out->xllcorner = xll;
        out->yllcorner = yll;
        out->cellsize = cell;
        out->count = vals.size();
        out->values = static_cast<double*>(std::malloc(std::max<size_t>(1, vals.size()) * sizeof(double)));
        if (!out->values) throw std::bad_alloc();
        if (!vals.empty()) std::memcpy(out->values, vals.data(), vals.size() * sizeof(double));
        return ok(err);
    } catch (const IoError& e) {
        return fail(err, e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(err, AIDW_ERR_RUNTIME, e.what());
    }
}

void aidw_free_raster(aidw_raster_buffer* buf) {
    if (!buf) return;
    std::free(buf->values);
    buf->values = nullptr;
    buf->count = 0;
}

}  // extern "C"
