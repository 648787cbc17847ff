#pragma once

// aidw/cli.hpp — the pipeline orchestrator of the reference's cli.hpp
// (RunConfig :30-43, the enum parsers :49-73, PipelineOutcome :207-211,
// run_pipeline :217-268).  run_pipeline is the fused, device-resident path
// (aidw_run_pipeline): bbox -> grid build (K1) -> cell-sorted kNN + alpha
// (K2 + K3) -> weighting (K4) with no per-query KnnResult materialisation;
// StageTimings come from CUDA events.  The file commands, JSON/CSV reports
// and CLI11 front end of the reference are out of scope (SURVEY §2 rows 9,
// 11) and not provided.

#include <cstdint>
#include <stdexcept>
#include <string>

#include "aidw/executor.hpp"
#include "aidw/interpolate.hpp"
#include "aidw/knn.hpp"
#include "aidw/types.hpp"

namespace aidw::cli {

inline constexpr const char* kVersion = "1.0.0";

enum class Mode { idw, aidw };

struct RunConfig {
    Mode mode = Mode::aidw;
    KnnEngine knn_engine = KnnEngine::grid;
    Variant variant = Variant::blocked;
    AidwParams params;
    double alpha = 2.0;
    double cell_factor = 4.0;
    int workers = 1;
    std::uint64_t seed = 42;
    std::string data_path;
    std::string queries_path;
    std::string out_path;
    std::string report_path;
};

inline Mode parse_mode(const std::string& text) {
    if (text == "idw") return Mode::idw;
    if (text == "aidw") return Mode::aidw;
    throw std::invalid_argument("unknown mode '" + text + "' (expected idw|aidw)");
}
inline KnnEngine parse_engine(const std::string& text) {
    if (text == "grid") return KnnEngine::grid;
    if (text == "brute") return KnnEngine::brute;
    throw std::invalid_argument("unknown knn engine '" + text + "' (expected grid|brute)");
}
inline Variant parse_variant(const std::string& text) {
    if (text == "naive") return Variant::naive;
    if (text == "blocked") return Variant::blocked;
    throw std::invalid_argument("unknown variant '" + text + "' (expected naive|blocked)");
}
inline const char* mode_name(Mode m) { return m == Mode::idw ? "idw" : "aidw"; }
inline const char* engine_name(KnnEngine e) { return e == KnnEngine::grid ? "grid" : "brute"; }
inline const char* variant_name(Variant v) { return v == Variant::naive ? "naive" : "blocked"; }

struct PipelineOutcome {
    InterpolationResult result;
    StageTimings timings;
    int k_effective = 0;
};

/// (grid build ->) kNN -> weighting, fused on the GPU.  k is clamped to m;
/// idw mode has no kNN stage (build / knn report 0 ms).
inline PipelineOutcome run_pipeline(const PointSet& data, const PointSet& queries,
                                    const RunConfig& cfg) {
    const int workers = resolve_workers(cfg.workers);
    aidw_run_config c{};
    c.mode = cfg.mode == Mode::idw ? AIDW_MODE_IDW : AIDW_MODE_AIDW;
    c.engine = cfg.knn_engine == KnnEngine::grid ? AIDW_ENGINE_GRID : AIDW_ENGINE_BRUTE;
    c.variant = detail::variant_c(cfg.variant);
    c.params = cfg.params.to_c();
    c.alpha = cfg.alpha;
    c.cell_factor = cfg.cell_factor;
    c.workers = workers;
    const std::size_t n = queries.count();
    PipelineOutcome out;
    out.result.predicted.resize(n);
    out.result.alphas.resize(n);
    aidw_run_stats st{};
    aidw_error err{};
    detail::raise_if(aidw_run_pipeline(data.xs.data(), data.ys.data(),
                                       data.has_values() ? data.zs.data() : nullptr, data.count(),
                                       queries.xs.data(), queries.ys.data(), n, &c,
                                       out.result.predicted.data(), out.result.alphas.data(), &st,
                                       &err),
                     err);
    out.k_effective = st.k_effective;
    out.timings.m = data.count();
    out.timings.n = n;
    out.timings.k = st.k_effective;
    out.timings.worker_count = workers;
    out.timings.build_millis = st.build_ms;
    out.timings.knn_millis = st.knn_ms;
    out.timings.interp_millis = st.interp_ms;
    out.timings.total_millis = st.total_ms;
    return out;
}

}  // namespace aidw::cli
