// generate.cpp — deterministic synthetic inputs (host).
//
// generate_random_points / generate_random_queries restate
// proj/include/aidw/generate.hpp:45-95 (mt19937_64; one double in [0, 1)
// from the top 53 bits of a draw; three draws per data point whatever the
// value rule).  The clustered generator is the harness addition of SURVEY
// §8d (config 4; the reference has none).  The raster lattice restates
// cmd_raster's query lattice (cli.hpp:496-507).  Compiled with
// -ffp-contract=off so every coordinate is bit-identical to the reference's.
// Input synthesis only — not part of the accelerated path.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "aidw_capi.h"

namespace {

double unit_draw(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

bool box_ok(const double* b) {
    const double w = b[2] - b[0], h = b[3] - b[1];
    return b[0] <= b[2] && b[1] <= b[3] && (w * h > 0.0);
}

int fail(aidw_error* err, int code, const char* msg) {
    if (err) {
        err->code = code;
        err->index = -1;
        std::strncpy(err->message, msg, sizeof(err->message) - 1);
        err->message[sizeof(err->message) - 1] = '\0';
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

}  // namespace

extern "C" {

int aidw_generate_points(size_t count, const double* bbox, uint64_t seed, int32_t rule,
                         double* xs, double* ys, double* zs, aidw_error* err) {
    if (count == 0)
        return fail(err, AIDW_ERR_INVALID_ARGUMENT, "generate_random_points: count must be >= 1");
    if (!box_ok(bbox))
        return fail(err, AIDW_ERR_INVALID_ARGUMENT,
                    "generate_random_points: bbox must have positive area");
    std::mt19937_64 g(seed);
    const double w = bbox[2] - bbox[0], h = bbox[3] - bbox[1];
    const double cx = bbox[0] + 0.5 * w, cy = bbox[1] + 0.5 * h;
    for (size_t i = 0; i < count; ++i) {
        const double x = bbox[0] + unit_draw(g) * w;
        const double y = bbox[1] + unit_draw(g) * h;
        const double noise = unit_draw(g);
        double z = noise;
        if (rule == 1) {
            z = 1.5 * x + -2.5 * y + 4.0;  // planar_field, generate.hpp:23-30
        } else if (rule == 2) {
            z = std::hypot(x - cx, y - cy);
        }
        xs[i] = x;
        ys[i] = y;
        if (zs) zs[i] = z;
    }
    return ok(err);
}

int aidw_generate_queries(size_t count, const double* bbox, uint64_t seed, double* xs,
                          double* ys, aidw_error* err) {
    if (count == 0)
        return fail(err, AIDW_ERR_INVALID_ARGUMENT, "generate_random_queries: count must be >= 1");
    if (!box_ok(bbox))
        return fail(err, AIDW_ERR_INVALID_ARGUMENT,
                    "generate_random_queries: bbox must have positive area");
    std::mt19937_64 g(seed);
    const double w = bbox[2] - bbox[0], h = bbox[3] - bbox[1];
    for (size_t i = 0; i < count; ++i) {
        xs[i] = bbox[0] + unit_draw(g) * w;
        ys[i] = bbox[1] + unit_draw(g) * h;
    }
    return ok(err);
}

int aidw_generate_clustered(size_t count, int32_t blobs, double sigma, uint64_t center_seed,
                            uint64_t seed, double* xs, double* ys, double* zs, aidw_error* err) {
    if (count == 0 || blobs < 1 || !(sigma > 0.0))
        return fail(err, AIDW_ERR_INVALID_ARGUMENT, "generate_clustered: bad arguments");
    std::mt19937_64 cg(center_seed), g(seed);
    std::vector<double> cx(static_cast<size_t>(blobs)), cy(static_cast<size_t>(blobs));
    for (int b = 0; b < blobs; ++b) {
        cx[static_cast<size_t>(b)] = 0.1 + 0.8 * unit_draw(cg);
        cy[static_cast<size_t>(b)] = 0.1 + 0.8 * unit_draw(cg);
    }
    const double two_pi = 2.0 * std::numbers::pi;
    size_t i = 0;
    while (i < count) {
        const size_t b = static_cast<size_t>(g() % static_cast<uint64_t>(blobs));
        const double u1 = unit_draw(g), u2 = unit_draw(g);
        const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
        const double t = two_pi * u2;
        const double x = cx[b] + sigma * (r * std::cos(t));
        const double y = cy[b] + sigma * (r * std::sin(t));
        if (!(x >= 0.0 && x <= 1.0 && y >= 0.0 && y <= 1.0)) continue;
        xs[i] = x;
        ys[i] = y;
        if (zs) zs[i] = unit_draw(g);
        ++i;
    }
    return ok(err);
}

int aidw_raster_lattice(size_t nx, size_t ny, const double* bbox, double* xs, double* ys,
                        aidw_error* err) {
    if (nx < 1 || ny < 1)
        return fail(err, AIDW_ERR_INVALID_ARGUMENT, "cmd_raster: nx and ny must be >= 1");
    const double sx = (bbox[2] - bbox[0]) / static_cast<double>(nx);
    const double sy = (bbox[3] - bbox[1]) / static_cast<double>(ny);
    size_t i = 0;
    for (size_t r = 0; r < ny; ++r) {
        const double y = bbox[1] + (static_cast<double>(ny - 1 - r) + 0.5) * sy;
        for (size_t c = 0; c < nx; ++c, ++i) {
            xs[i] = bbox[0] + (static_cast<double>(c) + 0.5) * sx;
            ys[i] = y;
        }
    }
    return ok(err);
}

}  // extern "C"
