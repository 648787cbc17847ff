// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// header library (/root/reference/proj/include/aidw, compiled in place by
// oracle/Makefile into oracle/_ref/libaidw_ref*.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  The product never links this.  Used
// by tests/golden/make_golden.py (fixtures pinning the C restatement), by
// tests, and by bench.py's cpu_baseline leg and `--impl reference` arm,
// which time the reference's own cli::run_pipeline on the host cores.
//
// Every wrapper converts flat C arrays to the reference's PointSet /
// KnnResult types, calls the reference function, and flattens the result.
// Exceptions become {code, message}: 1 invalid_argument, 2 domain_error,
// 3 out_of_range, 4 runtime_error, 5 other.

#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "aidw/cli.hpp"

namespace {

int classify(const std::exception& e, char* msg, std::size_t cap) {
    if (msg && cap) {
        std::strncpy(msg, e.what(), cap - 1);
        msg[cap - 1] = '\0';
    }
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::domain_error*>(&e)) return 2;
    if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
    if (dynamic_cast<const std::runtime_error*>(&e)) return 4;
    return 5;
}

aidw::PointSet make_set(const double* xs, const double* ys, const double* zs, std::size_t n) {
    aidw::PointSet s;
    s.xs.assign(xs, xs + n);
    s.ys.assign(ys, ys + n);
    if (zs) s.zs.assign(zs, zs + n);
    return s;
}

aidw::AidwParams make_params(int k, double r_min, double r_max, const double* levels,
                             double area) {
    aidw::AidwParams p;
    p.k = k;
    p.r_min = r_min;
    p.r_max = r_max;
    for (int i = 0; i < 5; ++i) p.alpha_levels[static_cast<std::size_t>(i)] = levels[i];
    p.area = area;
    return p;
}

}  // namespace

extern "C" {

int ref_generate_points(std::size_t count, const double* bbox, std::uint64_t seed, int rule,
                        double* xs, double* ys, double* zs, char* msg, std::size_t cap) {
    try {
        const aidw::PointSet s = aidw::generate_random_points(
            count, aidw::BoundingBox{bbox[0], bbox[1], bbox[2], bbox[3]}, seed,
            static_cast<aidw::ValueRule>(rule));
        std::memcpy(xs, s.xs.data(), count * sizeof(double));
        std::memcpy(ys, s.ys.data(), count * sizeof(double));
        std::memcpy(zs, s.zs.data(), count * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

int ref_generate_queries(std::size_t count, const double* bbox, std::uint64_t seed, double* xs,
                         double* ys, char* msg, std::size_t cap) {
    try {
        const aidw::PointSet s = aidw::generate_random_queries(
            count, aidw::BoundingBox{bbox[0], bbox[1], bbox[2], bbox[3]}, seed);
        std::memcpy(xs, s.xs.data(), count * sizeof(double));
        std::memcpy(ys, s.ys.data(), count * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// cfg_out = {cell_width, n_col, n_row, min_x, min_y}
int ref_grid_config(const double* dx, const double* dy, std::size_t m, const double* qx,
                    const double* qy, std::size_t n, double factor, double* cfg_out, char* msg,
                    std::size_t cap) {
    try {
        const aidw::PointSet data = make_set(dx, dy, nullptr, m);
        const aidw::PointSet queries = make_set(qx, qy, nullptr, n);
        const aidw::BoundingBox box = aidw::compute_bbox(data, queries);
        const aidw::GridConfig c =
            aidw::make_grid_config(box, aidw::choose_cell_width(data, box, factor));
        cfg_out[0] = c.cell_width;
        cfg_out[1] = c.n_col;
        cfg_out[2] = c.n_row;
        cfg_out[3] = c.min_x;
        cfg_out[4] = c.min_y;
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

int ref_build_index(const double* xs, const double* ys, std::size_t m, const double* cfg,
                    std::uint32_t* sorted_ids, std::uint32_t* cell_start, double* sorted_x,
                    double* sorted_y, char* msg, std::size_t cap) {
    try {
        aidw::GridConfig c;
        c.cell_width = cfg[0];
        c.n_col = static_cast<int>(cfg[1]);
        c.n_row = static_cast<int>(cfg[2]);
        c.min_x = cfg[3];
        c.min_y = cfg[4];
        const aidw::GridIndex g = aidw::build_index(make_set(xs, ys, nullptr, m), c);
        std::memcpy(sorted_ids, g.sorted_point_ids.data(), m * sizeof(std::uint32_t));
        std::memcpy(cell_start, g.cell_start.data(), g.cell_start.size() * sizeof(std::uint32_t));
        std::memcpy(sorted_x, g.sorted_x.data(), m * sizeof(double));
        std::memcpy(sorted_y, g.sorted_y.data(), m * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// knn_stage over a grid built with `factor` from bbox(data ∪ queries) (engine
// 0) or brute force (engine 1).  d2 is n x k row-major, padded with +inf
// when a list is shorter (exhausted); lens[i] = list length.
int ref_knn_stage(const double* qx, const double* qy, std::size_t n, const double* dx,
                  const double* dy, std::size_t m, int k, int engine, double factor, int workers,
                  double* d2, double* avg, int* exhausted, std::int64_t* lens, char* msg,
                  std::size_t cap) {
    try {
        const aidw::PointSet data = make_set(dx, dy, nullptr, m);
        const aidw::PointSet queries = make_set(qx, qy, nullptr, n);
        aidw::GridIndex index;
        if (engine == 0) {
            const aidw::BoundingBox box = aidw::compute_bbox(data, queries);
            index = aidw::build_index(
                data, aidw::make_grid_config(box, aidw::choose_cell_width(data, box, factor)));
        }
        const auto res = aidw::knn_stage(queries, engine == 0 ? &index : nullptr, data, k,
                                         engine == 0 ? aidw::KnnEngine::grid
                                                     : aidw::KnnEngine::brute,
                                         workers);
        for (std::size_t i = 0; i < n; ++i) {
            const auto& r = res[i];
            for (int j = 0; j < k; ++j) {
                d2[i * static_cast<std::size_t>(k) + static_cast<std::size_t>(j)] =
                    static_cast<std::size_t>(j) < r.size() ? r.distances_sq[static_cast<std::size_t>(j)]
                                                          : __builtin_inf();
            }
            avg[i] = r.average_distance;
            exhausted[i] = r.exhausted ? 1 : 0;
            lens[i] = static_cast<std::int64_t>(r.size());
        }
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// adaptive_alpha; rec = {r_exp, r_obs, R, mu, alpha}
int ref_adaptive_alpha(double r_obs, std::size_t list_len, int exhausted, std::size_t m,
                       double area, int k, double r_min, double r_max, const double* levels,
                       double* rec, char* msg, std::size_t cap) {
    try {
        aidw::KnnResult knn;
        knn.distances_sq.assign(list_len, r_obs * r_obs);
        knn.average_distance = r_obs;
        knn.exhausted = exhausted != 0;
        const aidw::AdaptiveAlpha a =
            aidw::adaptive_alpha(knn, m, area, make_params(k, r_min, r_max, levels, 0.0));
        rec[0] = a.r_exp;
        rec[1] = a.r_obs;
        rec[2] = a.r_statistic;
        rec[3] = a.mu_r;
        rec[4] = a.alpha;
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

double ref_normalize_mu(double R, double r_min, double r_max) {
    return aidw::normalize_mu(R, r_min, r_max);
}

int ref_alpha_from_mu(double mu, const double* levels, double* out, char* msg, std::size_t cap) {
    try {
        std::array<double, 5> lv{levels[0], levels[1], levels[2], levels[3], levels[4]};
        *out = aidw::alpha_from_mu(mu, lv);
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// Full run_pipeline (cli.hpp:217-268).  mode 0 = idw, 1 = aidw; engine 0 grid
// 1 brute; variant 0 naive 1 blocked.  timings = {build, knn, interp, total}.
int ref_run_pipeline(const double* dx, const double* dy, const double* dz, std::size_t m,
                     const double* qx, const double* qy, std::size_t n, int mode, int engine,
                     int variant, int k, double r_min, double r_max, const double* levels,
                     double area, double alpha, double factor, int workers, double* pred,
                     double* alphas, double* timings, int* k_eff, char* msg, std::size_t cap) {
    try {
        aidw::cli::RunConfig cfg;
        cfg.mode = mode == 0 ? aidw::cli::Mode::idw : aidw::cli::Mode::aidw;
        cfg.knn_engine = engine == 0 ? aidw::KnnEngine::grid : aidw::KnnEngine::brute;
        cfg.variant = variant == 0 ? aidw::Variant::naive : aidw::Variant::blocked;
        cfg.params = make_params(k, r_min, r_max, levels, area);
        cfg.alpha = alpha;
        cfg.cell_factor = factor;
        cfg.workers = workers;
        const aidw::PointSet data = make_set(dx, dy, dz, m);
        const aidw::PointSet queries = make_set(qx, qy, nullptr, n);
        const aidw::cli::PipelineOutcome out = aidw::cli::run_pipeline(data, queries, cfg);
        std::memcpy(pred, out.result.predicted.data(), n * sizeof(double));
        std::memcpy(alphas, out.result.alphas.data(), n * sizeof(double));
        timings[0] = out.timings.build_millis;
        timings[1] = out.timings.knn_millis;
        timings[2] = out.timings.interp_millis;
        timings[3] = out.timings.total_millis;
        *k_eff = out.k_effective;
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// aidw_predict_all fed by a grid (engine 0) or brute (engine 1) kNN stage,
// or idw_predict_all when mode == 0; pinned selects the pinned-order variant.
int ref_predict_all(const double* dx, const double* dy, const double* dz, std::size_t m,
                    const double* qx, const double* qy, std::size_t n, int mode, int engine,
                    int variant, int pinned, int k, double r_min, double r_max,
                    const double* levels, double area, double alpha, double factor, int workers,
                    double* pred, double* alphas, char* msg, std::size_t cap) {
    try {
        const aidw::PointSet data = make_set(dx, dy, dz, m);
        const aidw::PointSet queries = make_set(qx, qy, nullptr, n);
        const aidw::Variant v = variant == 0 ? aidw::Variant::naive : aidw::Variant::blocked;
        aidw::InterpolationResult r;
        if (mode == 0) {
            r = aidw::idw_predict_all(queries, data, alpha, v, workers, pinned != 0);
        } else {
            aidw::GridIndex index;
            if (engine == 0) {
                const aidw::BoundingBox box = aidw::compute_bbox(data, queries);
                index = aidw::build_index(
                    data, aidw::make_grid_config(box, aidw::choose_cell_width(data, box, factor)));
            }
            const auto knn = aidw::knn_stage(queries, engine == 0 ? &index : nullptr, data, k,
                                             engine == 0 ? aidw::KnnEngine::grid
                                                         : aidw::KnnEngine::brute,
                                             workers);
            r = aidw::aidw_predict_all(queries, data, knn,
                                       make_params(k, r_min, r_max, levels, area), v, workers,
                                       pinned != 0);
        }
        std::memcpy(pred, r.predicted.data(), n * sizeof(double));
        std::memcpy(alphas, r.alphas.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// cli::cmd_raster (cli.hpp:484-524) end to end: the data set goes through
// the reference's CSV writer and parser, the raster through its
// write_raster_asc.  meta = {ncols, nrows, xllcorner, yllcorner, cellsize}.
int ref_cmd_raster(const double* dx, const double* dy, const double* dz, std::size_t m,
                   std::size_t nx, std::size_t ny, int k, int workers, const char* csv_path,
                   const char* asc_path, double* values, double* meta, char* msg,
                   std::size_t cap) {
    try {
        aidw::write_data_csv(csv_path, make_set(dx, dy, dz, m));
        aidw::cli::RunConfig cfg;
        const double levels[5] = {0.5, 1.0, 2.0, 3.0, 4.0};  // types.hpp defaults
        cfg.params = make_params(k, 0.0, 2.0, levels, 0.0);
        cfg.workers = workers;
        cfg.data_path = csv_path;
        cfg.out_path = asc_path;
        const aidw::cli::RasterOutcome out = aidw::cli::cmd_raster(cfg, nx, ny);
        std::memcpy(values, out.raster.values.data(), nx * ny * sizeof(double));
        meta[0] = static_cast<double>(out.raster.ncols);
        meta[1] = static_cast<double>(out.raster.nrows);
        meta[2] = out.raster.xllcorner;
        meta[3] = out.raster.yllcorner;
        meta[4] = out.raster.cellsize;
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, cap);
    }
}

// read_data_csv / read_query_csv (io.hpp:103-145): up to `cap` points.
int ref_read_points_csv(const char* path, int with_values, std::size_t cap, double* xs,
                        double* ys, double* zs, std::size_t* count, char* msg, std::size_t mcap) {
    try {
        const aidw::PointSet set = with_values ? aidw::read_data_csv(path) : aidw::read_query_csv(path);
        *count = set.count();
        const std::size_t n = set.count() < cap ? set.count() : cap;
        std::memcpy(xs, set.xs.data(), n * sizeof(double));
        std::memcpy(ys, set.ys.data(), n * sizeof(double));
        if (with_values) std::memcpy(zs, set.zs.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return classify(e, msg, mcap);
    }
}

int ref_hardware_threads() { return aidw::resolve_workers(0); }

}  // extern "C"
