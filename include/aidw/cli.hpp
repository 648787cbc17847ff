#pragma once

// aidw/cli.hpp — source-compatible restatement of proj/include/aidw/cli.hpp:
// the run configuration and its parsers (:30-143), the reports (:144-205),
// run_pipeline (:217-268) and the file commands that drive it
// (cmd_generate :278-291, cmd_interpolate :293-331, cmd_bench :333-474,
// cmd_raster :476-524).  run_pipeline is the fused, device-resident path
// (aidw_run_pipeline): bbox -> grid build (K1) -> cell-sorted kNN + alpha
// (K2 + K3) -> weighting (K4) with no per-query KnnResult materialisation;
// StageTimings come from CUDA events.  cmd_raster generates its lattice in
// HBM (aidw_run_raster).  The CLI11 front end (tools/aidw_cli.cpp) is out of
// scope.  Reports use nlohmann::json like the reference (<json.hpp>).

#include <algorithm>
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <json.hpp>

#include "aidw/executor.hpp"
#include "aidw/generate.hpp"
#include "aidw/grid.hpp"
#include "aidw/interpolate.hpp"
#include "aidw/io.hpp"
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

/// Point-count spec (cli.hpp:74-99): an integer, optionally with a K / k
/// suffix meaning exactly 1024 ("10K" = 10240).
inline std::size_t parse_size_spec(const std::string& text) {
    if (text.empty()) throw std::invalid_argument("empty size spec");
    const bool kilo = text.back() == 'K' || text.back() == 'k';
    const std::string digits = kilo ? text.substr(0, text.size() - 1) : text;
    unsigned long long value = 0;
    std::size_t used = 0;
    try {
        value = std::stoull(digits, &used);
    } catch (const std::exception&) {
        throw std::invalid_argument("bad size spec '" + text + "'");
    }
    if (used != digits.size() || value == 0) throw std::invalid_argument("bad size spec '" + text + "'");
    return static_cast<std::size_t>(value) * (kilo ? 1024 : 1);
}

/// Comma-separated size ladder, e.g. "10K,50K,100K" (cli.hpp:101-118).
inline std::vector<std::size_t> parse_size_ladder(const std::string& text) {
    std::vector<std::size_t> out;
    std::size_t start = 0;
    for (;;) {
        const std::size_t comma = text.find(',', start);
        out.push_back(parse_size_spec(text.substr(start, comma == std::string::npos
                                                             ? std::string::npos
                                                             : comma - start)));
        if (comma == std::string::npos) break;
        start = comma + 1;
    }
    return out;
}

/// Exactly five comma-separated alpha levels (cli.hpp:120-141).
inline std::array<double, 5> parse_alpha_levels(const std::string& text) {
    std::array<double, 5> out{};
    std::size_t start = 0;
    for (std::size_t i = 0; i < out.size(); ++i) {
        const std::size_t comma = text.find(',', start);
        if ((comma == std::string::npos) != (i + 1 == out.size()))
            throw std::invalid_argument("alpha levels need exactly 5 comma-separated values");
        try {
            out[i] = std::stod(text.substr(start, comma == std::string::npos ? std::string::npos
                                                                             : comma - start));
        } catch (const std::exception&) {
            throw std::invalid_argument("bad alpha level in '" + text + "'");
        }
        start = comma + 1;
    }
    return out;
}

/// The configuration echo of every report (cli.hpp:144-161).
inline nlohmann::json config_to_json(const RunConfig& cfg) {
    nlohmann::json j;
    j["mode"] = mode_name(cfg.mode);
    j["knn"] = engine_name(cfg.knn_engine);
    j["variant"] = variant_name(cfg.variant);
    j["k"] = cfg.params.k;
    j["alpha_levels"] = cfg.params.alpha_levels;
    j["alpha"] = cfg.alpha;
    j["rmin"] = cfg.params.r_min;
    j["rmax"] = cfg.params.r_max;
    j["area"] = cfg.params.area;
    j["cell_factor"] = cfg.cell_factor;
    j["workers"] = cfg.workers;
    j["seed"] = cfg.seed;
    j["data"] = cfg.data_path;
    j["queries"] = cfg.queries_path;
    j["out"] = cfg.out_path;
    j["report"] = cfg.report_path;
    return j;
}

/// Stage shares in percent over build / knn / interp, summing to exactly
/// 100 (interp takes the remainder); all zero when nothing was timed.
struct WorkloadPercent {
    double build = 0.0;
    double knn = 0.0;
    double interp = 0.0;
};

inline WorkloadPercent workload_percent(const StageTimings& t) {
    const double total = t.build_millis + t.knn_millis + t.interp_millis;
    WorkloadPercent w;
    if (total > 0.0) {
        w.build = 100.0 * t.build_millis / total;
        w.knn = 100.0 * t.knn_millis / total;
        w.interp = 100.0 - w.build - w.knn;
    }
    return w;
}

inline nlohmann::json timings_to_json(const StageTimings& t, double parse_millis) {
    const WorkloadPercent w = workload_percent(t);
    nlohmann::json j;
    j["sizes"] = {{"m", t.m}, {"n", t.n}, {"k", t.k}};
    j["workers"] = t.worker_count;
    j["timings_ms"] = {{"parse", parse_millis},     {"build", t.build_millis},
                       {"knn", t.knn_millis},       {"interp", t.interp_millis},
                       {"total", t.total_millis},   {"slack", t.slack_millis()}};
    j["workload_percent"] = {{"build", w.build}, {"knn", w.knn}, {"interp", w.interp}};
    return j;
}

struct PipelineOutcome {
    InterpolationResult result;
    StageTimings timings;
    int k_effective = 0;
};

namespace impl {  // (not `detail`: tests use both aidw and aidw::cli)

inline aidw_run_config run_config_c(const RunConfig& cfg, int workers) {
    aidw_run_config c{};
    c.mode = cfg.mode == Mode::idw ? AIDW_MODE_IDW : AIDW_MODE_AIDW;
    c.engine = cfg.knn_engine == KnnEngine::grid ? AIDW_ENGINE_GRID : AIDW_ENGINE_BRUTE;
    c.variant = ::aidw::detail::variant_c(cfg.variant);
    c.params = cfg.params.to_c();
    c.alpha = cfg.alpha;
    c.cell_factor = cfg.cell_factor;
    c.workers = workers;
    return c;
}

inline void fill_timings(PipelineOutcome& out, const aidw_run_stats& st, std::size_t m,
                         std::size_t n, int workers) {
    out.k_effective = st.k_effective;
    out.timings.m = m;
    out.timings.n = n;
    out.timings.k = st.k_effective;
    out.timings.worker_count = workers;
    out.timings.build_millis = st.build_ms;
    out.timings.knn_millis = st.knn_ms;
    out.timings.interp_millis = st.interp_ms;
    out.timings.total_millis = st.total_ms;
}

}  // namespace impl

/// (grid build ->) kNN -> weighting, fused on the GPU.  k is clamped to m;
/// idw mode has no kNN stage (build / knn report 0 ms).
inline PipelineOutcome run_pipeline(const PointSet& data, const PointSet& queries,
                                    const RunConfig& cfg) {
    const int workers = resolve_workers(cfg.workers);
    const aidw_run_config c = impl::run_config_c(cfg, workers);
    const std::size_t n = queries.count();
    PipelineOutcome out;
    out.result.predicted.resize(n);
    out.result.alphas.resize(n);
    aidw_run_stats st{};
    aidw_error err{};
    ::aidw::detail::raise_if(
        aidw_run_pipeline(data.xs.data(), data.ys.data(),
                          data.has_values() ? data.zs.data() : nullptr, data.count(),
                          queries.xs.data(), queries.ys.data(), n, &c, out.result.predicted.data(),
                          out.result.alphas.data(), &st, &err),
        err);
    impl::fill_timings(out, st, data.count(), n, workers);
    return out;
}

// ---------------------------------------------------------------- commands

enum class GenerateKind { data, queries };

/// Deterministic point file (cli.hpp:278-291); an empty path skips writing.
inline PointSet cmd_generate(std::size_t count, const BoundingBox& bbox, std::uint64_t seed,
                             ValueRule rule, GenerateKind kind, const std::string& out_path) {
    const bool data = kind == GenerateKind::data;
    PointSet set = data ? generate_random_points(count, bbox, seed, rule)
                        : generate_random_queries(count, bbox, seed);
    if (!out_path.empty()) {
        if (data) write_data_csv(out_path, set);
        else write_query_csv(out_path, set);
    }
    return set;
}

struct InterpolateOutcome {
    PipelineOutcome pipeline;
    double parse_millis = 0.0;
    nlohmann::json report;
};

/// CSV in -> run_pipeline -> result CSV + JSON report (cli.hpp:293-331).
inline InterpolateOutcome cmd_interpolate(const RunConfig& cfg) {
    if (cfg.data_path.empty() || cfg.queries_path.empty())
        throw std::invalid_argument("cmd_interpolate: data and queries paths are required");
    auto inputs = time_stage("parse", [&] {
        return std::pair<PointSet, PointSet>{read_data_csv(cfg.data_path),
                                             read_query_csv(cfg.queries_path)};
    });
    const PointSet& data = inputs.value.first;
    const PointSet& queries = inputs.value.second;
    InterpolateOutcome out;
    out.pipeline = run_pipeline(data, queries, cfg);
    out.parse_millis = inputs.millis;
    out.report["version"] = kVersion;
    out.report["config"] = config_to_json(cfg);
    out.report["k_effective"] = out.pipeline.k_effective;
    out.report["run"] = timings_to_json(out.pipeline.timings, out.parse_millis);
    if (!cfg.out_path.empty()) write_result_csv(cfg.out_path, queries, out.pipeline.result);
    if (!cfg.report_path.empty()) {
        auto f = ::aidw::detail::open_for_write(cfg.report_path);
        f << out.report.dump(2) << '\n';
    }
    return out;
}

/// One rung of the benchmark ladder (cli.hpp:333-352): both kNN engines and
/// both weighting variants on the same m = n instance, through the drop-in
/// batch calls (GPU kernels).
struct BenchRow {
    std::size_t m = 0;
    std::size_t n = 0;
    int k = 0;
    bool failed = false;
    std::string error;
    double build_ms = 0.0;
    double knn_grid_ms = 0.0;
    double knn_brute_ms = 0.0;
    double interp_naive_ms = 0.0;
    double interp_blocked_ms = 0.0;
    double build_share_pct = 0.0;
    double knn_share_pct = 0.0;
    double interp_share_pct = 0.0;
    double knn_ratio = 0.0;
    double e2e_grid_ms = 0.0;
    double e2e_brute_ms = 0.0;
    double e2e_speedup = 0.0;
};

inline BenchRow bench_rung(const RunConfig& cfg, std::size_t size, int workers) {
    BenchRow row;
    row.m = row.n = size;
    const BoundingBox unit{0.0, 0.0, 1.0, 1.0};
    try {
        const PointSet data = generate_random_points(size, unit, cfg.seed, ValueRule::uniform);
        const PointSet queries = generate_random_queries(size, unit, cfg.seed + 1);
        AidwParams params = cfg.params;
        params.k = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(params.k), size));
        row.k = params.k;
        const BoundingBox box = compute_bbox(data, queries);
        const GridConfig grid_cfg = make_grid_config(box, choose_cell_width(data, box, cfg.cell_factor));
        auto grid = time_stage("build", [&] { return build_index(data, grid_cfg); });
        auto knn_g = time_stage("knn-grid", [&] {
            return knn_stage(queries, &grid.value, data, params.k, KnnEngine::grid, workers);
        });
        auto knn_b = time_stage("knn-brute", [&] {
            return knn_stage(queries, nullptr, data, params.k, KnnEngine::brute, workers);
        });
        auto naive = time_stage("interp-naive", [&] {
            return aidw_predict_all(queries, data, knn_g.value, params, Variant::naive, workers);
        });
        auto blocked = time_stage("interp-blocked", [&] {
            return aidw_predict_all(queries, data, knn_g.value, params, Variant::blocked, workers);
        });
        row.build_ms = grid.millis;
        row.knn_grid_ms = knn_g.millis;
        row.knn_brute_ms = knn_b.millis;
        row.interp_naive_ms = naive.millis;
        row.interp_blocked_ms = blocked.millis;
        StageTimings t;
        t.build_millis = row.build_ms;
        t.knn_millis = row.knn_grid_ms;
        t.interp_millis = row.interp_blocked_ms;
        const WorkloadPercent w = workload_percent(t);
        row.build_share_pct = w.build;
        row.knn_share_pct = w.knn;
        row.interp_share_pct = w.interp;
        row.knn_ratio = row.knn_brute_ms > 0.0 ? row.knn_grid_ms / row.knn_brute_ms : 0.0;
        row.e2e_grid_ms = row.build_ms + row.knn_grid_ms + row.interp_blocked_ms;
        row.e2e_brute_ms = row.knn_brute_ms + row.interp_blocked_ms;
        row.e2e_speedup = row.e2e_grid_ms > 0.0 ? row.e2e_brute_ms / row.e2e_grid_ms : 0.0;
    } catch (const std::exception& e) {
        row.failed = true;
        row.error = e.what();
    }
    return row;
}

/// The ladder (cli.hpp:356-422): a failing rung records its error and the
/// later rungs still run; data generation is never timed.
inline std::vector<BenchRow> cmd_bench(const RunConfig& cfg, const std::vector<std::size_t>& sizes) {
    if (sizes.empty()) throw std::invalid_argument("cmd_bench: size ladder is empty");
    const int workers = resolve_workers(cfg.workers);
    std::vector<BenchRow> rows;
    for (const std::size_t size : sizes) rows.push_back(bench_rung(cfg, size, workers));
    return rows;
}

inline nlohmann::json bench_to_json(const RunConfig& cfg, const std::vector<BenchRow>& rows) {
    nlohmann::json j;
    j["version"] = kVersion;
    j["config"] = config_to_json(cfg);
    j["rows"] = nlohmann::json::array();
    for (const BenchRow& r : rows) {
        nlohmann::json o;
        o["m"] = r.m;
        o["n"] = r.n;
        o["k"] = r.k;
        o["failed"] = r.failed;
        o["error"] = r.error;
        o["build_ms"] = r.build_ms;
        o["knn_grid_ms"] = r.knn_grid_ms;
        o["knn_brute_ms"] = r.knn_brute_ms;
        o["interp_naive_ms"] = r.interp_naive_ms;
        o["interp_blocked_ms"] = r.interp_blocked_ms;
        o["build_share_pct"] = r.build_share_pct;
        o["knn_share_pct"] = r.knn_share_pct;
        o["interp_share_pct"] = r.interp_share_pct;
        o["knn_ratio"] = r.knn_ratio;
        o["e2e_grid_ms"] = r.e2e_grid_ms;
        o["e2e_brute_ms"] = r.e2e_brute_ms;
        o["e2e_speedup"] = r.e2e_speedup;
        j["rows"].push_back(std::move(o));
    }
    return j;
}

inline void write_bench_csv(const std::string& path, const std::vector<BenchRow>& rows) {
    auto out = ::aidw::detail::open_for_write(path);
    out << "m,n,k,failed,build_ms,knn_grid_ms,knn_brute_ms,interp_naive_ms,interp_blocked_ms,"
           "build_share_pct,knn_share_pct,interp_share_pct,knn_ratio,e2e_grid_ms,e2e_brute_ms,"
           "e2e_speedup\n";
    for (const BenchRow& r : rows) {
        out << r.m << ',' << r.n << ',' << r.k << ',' << (r.failed ? 1 : 0);
        for (const double v : {r.build_ms, r.knn_grid_ms, r.knn_brute_ms, r.interp_naive_ms,
                               r.interp_blocked_ms, r.build_share_pct, r.knn_share_pct,
                               r.interp_share_pct, r.knn_ratio, r.e2e_grid_ms, r.e2e_brute_ms,
                               r.e2e_speedup})
            out << ',' << ::aidw::detail::format_double(v);
        out << '\n';
    }
    if (!out) throw std::runtime_error(path + ": write failed");
}

struct RasterOutcome {
    Raster raster;
    PipelineOutcome pipeline;
};

/// Interpolate onto an nx x ny lattice of cell centres over the data bbox,
/// northernmost row first (cli.hpp:484-524).  The lattice is generated in
/// HBM and the fused pipeline runs on it (aidw_run_raster).
inline RasterOutcome cmd_raster(const RunConfig& cfg, std::size_t nx, std::size_t ny) {
    if (nx < 1 || ny < 1) throw std::invalid_argument("cmd_raster: nx and ny must be >= 1");
    if (cfg.data_path.empty()) throw std::invalid_argument("cmd_raster: data path is required");
    const PointSet data = read_data_csv(cfg.data_path);
    if (data.count() == 0) throw std::invalid_argument("cmd_raster: data set is empty");
    const int workers = resolve_workers(cfg.workers);
    const aidw_run_config c = impl::run_config_c(cfg, workers);
    const std::size_t n = nx * ny;
    RasterOutcome out;
    out.pipeline.result.predicted.resize(n);
    out.pipeline.result.alphas.resize(n);
    double box[4] = {0.0, 0.0, 0.0, 0.0};
    aidw_run_stats st{};
    aidw_error err{};
    ::aidw::detail::raise_if(
        aidw_run_raster(data.xs.data(), data.ys.data(), data.has_values() ? data.zs.data() : nullptr,
                        data.count(), nx, ny, &c, out.pipeline.result.predicted.data(),
                        out.pipeline.result.alphas.data(), box, &st, &err),
        err);
    impl::fill_timings(out.pipeline, st, data.count(), n, workers);
    out.raster = Raster{nx, ny, box[0], box[1], (box[2] - box[0]) / static_cast<double>(nx),
                        out.pipeline.result.predicted};
    if (!cfg.out_path.empty()) write_raster_asc(cfg.out_path, out.raster);
    if (!cfg.report_path.empty()) {
        nlohmann::json report;
        report["version"] = kVersion;
        report["config"] = config_to_json(cfg);
        report["raster"] = {{"ncols", nx}, {"nrows", ny}};
        report["run"] = timings_to_json(out.pipeline.timings, 0.0);
        auto f = ::aidw::detail::open_for_write(cfg.report_path);
        f << report.dump(2) << '\n';
    }
    return out;
}

}  // namespace aidw::cli
