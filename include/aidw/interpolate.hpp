#pragma once

// aidw/interpolate.hpp — weighted interpolation over all m data points
// (drop-in for proj/include/aidw/interpolate.hpp).
//
// Every entry point runs on the GPU:
//   aidw_predict_all (:453-489) -> aidw_aidw_predict_all (K3 alpha + K4)
//   idw_predict_all  (:426-448) -> aidw_idw_predict_all  (K4, constant alpha)
//   idw_predict      (:412-422) -> the same, one query, Variant::naive
// Precision contract: Variant::blocked uses the FP32 MUFU kernel
// (|err| <= 1e-5 * max(|ref|, 1e-3 * value span) against the FP64
// reference); Variant::naive and pinned_order use the FP64 kernel
// (<= 2e-11 relative): index-order running sums inside each data chunk of
// the m-only chunking (up to 64 chunks), the chunk sums then added in chunk
// order; w = 1 / pow(sqrt(d2), alpha), or 1 / (d2 d2) for alpha == 4 —
// not the reference's single index-order loop, but within its contract.
// Setting AIDW_WEIGHT_FP64=1 (or aidw_set_weight_precision) routes
// Variant::blocked to the FP64 kernel too.  Snap, nearest-value fallback
// and hull clamp follow the reference exactly (see csrc/weight.cu).

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "aidw/adaptive.hpp"
#include "aidw/executor.hpp"
#include "aidw/knn.hpp"
#include "aidw/types.hpp"

namespace aidw {

enum class Variant { naive, blocked };

/// The reference's CPU staging chunk (kept for source compatibility; the
/// GPU kernel stages 256-point tiles through shared memory).
inline constexpr std::size_t kStageSize = 256;

struct InterpolationResult {
    std::vector<double> predicted;
    std::vector<double> alphas;
};

namespace detail {
inline void validate_interpolation_inputs(const PointSet& data) {
    if (data.count() == 0) throw std::invalid_argument("interpolation: data set is empty");
    if (!data.has_values()) throw std::invalid_argument("interpolation: data set carries no values");
}
inline int32_t variant_c(Variant v) {
    return v == Variant::naive ? AIDW_VARIANT_NAIVE : AIDW_VARIANT_BLOCKED;
}
}  // namespace detail

/// Constant-alpha IDW over a query set on the GPU.
inline InterpolationResult idw_predict_all(const PointSet& queries, const PointSet& data,
                                           double alpha, Variant variant, int workers = 1,
                                           bool pinned_order = false) {
    (void)workers;
    detail::validate_interpolation_inputs(data);
    if (!(alpha > 0.0) || !std::isfinite(alpha)) {
        throw std::invalid_argument("idw_predict_all: alpha must be positive finite");
    }
    InterpolationResult r;
    r.predicted.resize(queries.count());
    r.alphas.resize(queries.count());
    aidw_error err{};
    detail::raise_if(aidw_idw_predict_all(queries.xs.data(), queries.ys.data(), queries.count(),
                                          data.xs.data(), data.ys.data(), data.zs.data(),
                                          data.count(), alpha, detail::variant_c(variant),
                                          pinned_order ? 1 : 0, r.predicted.data(),
                                          r.alphas.data(), &err),
                     err);
    return r;
}

/// One constant-alpha prediction (naive variant, FP64 kernel).
inline double idw_predict(const QueryPoint& q, const PointSet& data, double alpha) {
    detail::validate_interpolation_inputs(data);
    if (!(alpha > 0.0) || !std::isfinite(alpha)) {
        throw std::invalid_argument("idw_predict: alpha must be positive finite");
    }
    PointSet one;
    one.add(q.x, q.y);
    return idw_predict_all(one, data, alpha, Variant::naive).predicted.front();
}

/// AIDW over a query set: per-query alpha from its kNN average distance,
/// then the full-data weighting, both on the GPU.
inline InterpolationResult aidw_predict_all(const PointSet& queries, const PointSet& data,
                                            const std::vector<KnnResult>& knn,
                                            const AidwParams& params, Variant variant,
                                            int workers = 1, bool pinned_order = false) {
    (void)workers;
    detail::validate_interpolation_inputs(data);
    params.validate();
    const std::size_t n = queries.count();
    if (knn.size() != n) {
        throw std::invalid_argument("aidw_predict_all: " + std::to_string(knn.size()) +
                                    " kNN results for " + std::to_string(n) + " queries");
    }
    std::vector<double> r_obs(n);
    std::vector<int64_t> lens(n);
    std::vector<uint8_t> exhausted(n);
    for (std::size_t i = 0; i < n; ++i) {
        r_obs[i] = knn[i].average_distance;
        lens[i] = static_cast<int64_t>(knn[i].size());
        exhausted[i] = knn[i].exhausted ? 1 : 0;
    }
    InterpolationResult r;
    r.predicted.resize(n);
    r.alphas.resize(n);
    const aidw_params p = params.to_c();
    aidw_error err{};
    detail::raise_if(aidw_aidw_predict_all(queries.xs.data(), queries.ys.data(), n, data.xs.data(),
                                           data.ys.data(), data.zs.data(), data.count(),
                                           r_obs.data(), lens.data(), exhausted.data(), &p,
                                           detail::variant_c(variant), pinned_order ? 1 : 0,
                                           r.predicted.data(), r.alphas.data(), &err),
                     err);
    return r;
}

}  // namespace aidw
