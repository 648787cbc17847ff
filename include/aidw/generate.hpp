#pragma once

// aidw/generate.hpp — deterministic synthetic inputs (drop-in for
// proj/include/aidw/generate.hpp: ValueRule :16-20, planar_field :23-30,
// generate_random_points :45-74, generate_random_queries :77-95).
// Implemented in libaidw_b200.so (csrc/generate.cpp, mt19937_64), bit-equal
// to the reference's output for every (count, bbox, seed, rule).

#include <cstdint>
#include <stdexcept>

#include "aidw/types.hpp"

namespace aidw {

enum class ValueRule { uniform, planar, radial };

inline constexpr double kPlanarA = 1.5;
inline constexpr double kPlanarB = -2.5;
inline constexpr double kPlanarC = 4.0;

inline double planar_field(double x, double y) noexcept {
    return kPlanarA * x + kPlanarB * y + kPlanarC;
}

inline PointSet generate_random_points(std::size_t count, const BoundingBox& bbox,
                                       std::uint64_t seed, ValueRule rule) {
    PointSet set;
    set.xs.resize(count);
    set.ys.resize(count);
    set.zs.resize(count);
    const double box[4] = {bbox.min_x, bbox.min_y, bbox.max_x, bbox.max_y};
    aidw_error err{};
    detail::raise_if(aidw_generate_points(count, box, seed, static_cast<int32_t>(rule),
                                          set.xs.data(), set.ys.data(), set.zs.data(), &err),
                     err);
    return set;
}

inline PointSet generate_random_queries(std::size_t count, const BoundingBox& bbox,
                                        std::uint64_t seed) {
    PointSet set;
    set.xs.resize(count);
    set.ys.resize(count);
    const double box[4] = {bbox.min_x, bbox.min_y, bbox.max_x, bbox.max_y};
    aidw_error err{};
    detail::raise_if(
        aidw_generate_queries(count, box, seed, set.xs.data(), set.ys.data(), &err), err);
    return set;
}

}  // namespace aidw
