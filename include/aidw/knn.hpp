#pragma once

// aidw/knn.hpp — exact kNN (drop-in for proj/include/aidw/knn.hpp).
//
// knn_stage (:255-271), the batch entry point, runs on the GPU through
// aidw_knn_stage (K2: register-resident (d2, index) top-k, cell-sorted
// queries — paper_1601_05904_b200/csrc/knn.cu); its squared-distance lists
// and average distances are bit-identical to the reference's.
//
// The single-query helpers — dist_sq (:23-27), brute_force_knn (:100-114),
// determine_expansion_level (:130-156), grid_knn (:212-249) — stay scalar
// host functions: they are the API's per-point vocabulary (the reference's
// own tests use them as oracles) and never run inside a batch call.
// Build callers of these helpers with -ffp-contract=off, as the reference
// requires, so dist_sq keeps its two-products-then-add rounding.

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "aidw/executor.hpp"
#include "aidw/grid.hpp"
#include "aidw/types.hpp"

namespace aidw {

#if defined(__GNUC__) && !defined(__clang__)
__attribute__((optimize("fp-contract=off")))
#endif
inline double dist_sq(double qx, double qy, double px, double py) noexcept {
    const double dx = px - qx;
    const double dy = py - qy;
    return dx * dx + dy * dy;
}

struct KnnResult {
    std::vector<double> distances_sq;  ///< ascending
    double average_distance = 0.0;     ///< mean of sqrt, summed ascending
    bool exhausted = false;

    [[nodiscard]] std::size_t size() const noexcept { return distances_sq.size(); }
};

enum class KnnEngine { grid, brute };

namespace detail {

/// Bounded ascending buffer: fill, then admit only values strictly below the
/// current kth (ties at the kth stay out) and sift them into place.
class KSlotBuffer {
public:
    explicit KSlotBuffer(std::size_t k) : cap_(k) { vals_.reserve(k); }

    void offer(double d2) {
        if (vals_.size() < cap_) {
            vals_.push_back(d2);
        } else if (d2 < vals_.back()) {
            vals_.back() = d2;
        } else {
            return;
        }
        for (std::size_t j = vals_.size() - 1; j > 0 && vals_[j - 1] > vals_[j]; --j) {
            std::swap(vals_[j - 1], vals_[j]);
        }
    }
    [[nodiscard]] bool full() const noexcept { return vals_.size() == cap_; }
    [[nodiscard]] double kth() const noexcept { return vals_.back(); }

    [[nodiscard]] KnnResult finalize(bool exhausted) && {
        KnnResult r;
        r.exhausted = exhausted;
        double s = 0.0;
        for (double v : vals_) s += std::sqrt(v);
        r.average_distance = vals_.empty() ? 0.0 : s / static_cast<double>(vals_.size());
        r.distances_sq = std::move(vals_);
        return r;
    }

private:
    std::size_t cap_;
    std::vector<double> vals_;
};

}  // namespace detail

inline KnnResult brute_force_knn(const QueryPoint& q, const PointSet& data, int k) {
    const std::size_t m = data.count();
    if (m == 0) throw std::invalid_argument("brute_force_knn: data set is empty");
    if (k < 1 || static_cast<std::size_t>(k) > m) {
        throw std::invalid_argument("brute_force_knn: k = " + std::to_string(k) +
                                    " outside [1, " + std::to_string(m) + "]");
    }
    detail::KSlotBuffer buf(static_cast<std::size_t>(k));
    for (std::size_t i = 0; i < m; ++i) buf.offer(dist_sq(q.x, q.y, data.xs[i], data.ys[i]));
    return std::move(buf).finalize(false);
}

struct ExpansionLevel {
    int level = 0;
    bool exhausted = false;
};

namespace detail {
struct Block {
    int c0, c1, r0, r1;
};
inline Block clipped_block(const CellCoord& cc, int level, const GridConfig& g) {
    return Block{std::max(0, cc.col - level), std::min(g.n_col - 1, cc.col + level),
                 std::max(0, cc.row - level), std::min(g.n_row - 1, cc.row + level)};
}
}  // namespace detail

/// One past the smallest level whose clipped block holds >= k points;
/// whole-grid cover + exhausted when the grid holds fewer than k.
inline ExpansionLevel determine_expansion_level(const QueryPoint& q, const GridIndex& index,
                                                int k) {
    if (index.point_count() == 0) {
        throw std::invalid_argument("determine_expansion_level: index holds no points");
    }
    if (k < 1) throw std::invalid_argument("determine_expansion_level: k must be >= 1");
    const GridConfig& g = index.config;
    const CellCoord cc = locate_cell(q.x, q.y, g);
    if (index.point_count() < static_cast<std::size_t>(k)) {
        const int cover = std::max({cc.col, g.n_col - 1 - cc.col, cc.row, g.n_row - 1 - cc.row});
        return ExpansionLevel{cover, true};
    }
    int level = 0;
    for (;; ++level) {
        const detail::Block b = detail::clipped_block(cc, level, g);
        if (index.block_count(b.c0, b.c1, b.r0, b.r1) >= static_cast<std::size_t>(k)) break;
    }
    return ExpansionLevel{level + 1, false};
}

namespace detail {
inline void offer_rect(const GridIndex& index, KSlotBuffer& buf, const QueryPoint& q, int c0,
                       int c1, int r0, int r1) {
    for (int r = r0; r <= r1; ++r) {
        const auto [lo, hi] = index.row_slice(r, c0, c1);
        for (std::uint32_t s = lo; s < hi; ++s) {
            buf.offer(dist_sq(q.x, q.y, index.sorted_x[s], index.sorted_y[s]));
        }
    }
}
}  // namespace detail

/// Exact grid kNN for one query (host): block at the expansion level, then
/// rings until kth <= (L w)^2 (1 - 1e-9) or the block covers the grid.
inline KnnResult grid_knn(const QueryPoint& q, const GridIndex& index, int k) {
    const std::size_t m = index.point_count();
    if (m == 0) throw std::invalid_argument("grid_knn: index holds no points");
    if (k < 1) throw std::invalid_argument("grid_knn: k must be >= 1");
    const GridConfig& g = index.config;
    const CellCoord cc = locate_cell(q.x, q.y, g);
    const ExpansionLevel start = determine_expansion_level(q, index, k);
    detail::KSlotBuffer buf(std::min<std::size_t>(static_cast<std::size_t>(k), m));
    int level = start.level;
    {
        const detail::Block b = detail::clipped_block(cc, level, g);
        detail::offer_rect(index, buf, q, b.c0, b.c1, b.r0, b.r1);
    }
    for (;;) {
        if (cc.col - level <= 0 && cc.row - level <= 0 && cc.col + level >= g.n_col - 1 &&
            cc.row + level >= g.n_row - 1) {
            break;
        }
        const double reach = static_cast<double>(level) * g.cell_width;
        if (buf.full() && buf.kth() <= reach * reach * (1.0 - 1.0e-9)) break;
        ++level;
        const detail::Block b = detail::clipped_block(cc, level, g);
        const detail::Block inner = detail::clipped_block(cc, level - 1, g);
        if (cc.row - level >= 0) detail::offer_rect(index, buf, q, b.c0, b.c1, b.r0, b.r0);
        if (cc.row + level <= g.n_row - 1) detail::offer_rect(index, buf, q, b.c0, b.c1, b.r1, b.r1);
        if (cc.col - level >= 0) detail::offer_rect(index, buf, q, b.c0, b.c0, inner.r0, inner.r1);
        if (cc.col + level <= g.n_col - 1)
            detail::offer_rect(index, buf, q, b.c1, b.c1, inner.r0, inner.r1);
    }
    return std::move(buf).finalize(start.exhausted);
}

/// Batch kNN stage on the GPU (aidw_knn_stage).  Output order = input
/// order; `workers` / `chunk` are accepted and ignored (no CPU threading).
inline std::vector<KnnResult> knn_stage(const PointSet& queries, const GridIndex* index,
                                        const PointSet& data, int k, KnnEngine engine,
                                        int workers = 1, std::size_t chunk = 64) {
    (void)workers;
    (void)chunk;
    const bool grid = engine == KnnEngine::grid;
    if (grid && index == nullptr) {
        throw std::invalid_argument("knn_stage: grid engine requires a grid index");
    }
    const std::size_t n = queries.count();
    const std::size_t m = grid ? index->point_count() : data.count();
    const std::size_t k_alloc =
        k < 1 ? 0 : (grid ? std::min<std::size_t>(static_cast<std::size_t>(k), m)
                          : static_cast<std::size_t>(k));
    // Flat staging rows, first touched in parallel (page faults of a fresh
    // n * k buffer are most of a first call's host time at 100K queries).
    const std::size_t threads =
        std::min<std::size_t>(static_cast<std::size_t>(resolve_workers(0)), n / 8192 + 1);
    auto parallel = [threads, n](auto&& body) {
        if (threads <= 1) {
            body(std::size_t{0}, n);
            return;
        }
        std::vector<std::thread> pool;
        const std::size_t step = (n + threads - 1) / threads;
        for (std::size_t t = 0; t < threads; ++t) {
            pool.emplace_back(body, std::min(n, t * step), std::min(n, (t + 1) * step));
        }
        for (auto& th : pool) th.join();
    };
    std::unique_ptr<double[]> d2(new double[n * k_alloc + 1]);
    std::vector<double> avg(n);
    parallel([&](std::size_t lo, std::size_t hi) {
        std::fill(d2.get() + lo * k_alloc, d2.get() + hi * k_alloc, 0.0);
    });
    int32_t k_eff = 0, exhausted = 0;
    aidw_error err{};
    aidw_grid_config c{};
    if (grid) c = index->config.to_c();
    detail::raise_if(
        aidw_knn_stage(queries.xs.data(), queries.ys.data(), n, grid ? &c : nullptr,
                       grid ? index->cell_start.data() : nullptr,
                       grid ? index->sorted_point_ids.data() : nullptr,
                       grid ? index->sorted_x.data() : nullptr,
                       grid ? index->sorted_y.data() : nullptr, grid ? nullptr : data.xs.data(),
                       grid ? nullptr : data.ys.data(), m, k,
                       grid ? AIDW_ENGINE_GRID : AIDW_ENGINE_BRUTE, d2.get(), nullptr, avg.data(),
                       &k_eff, &exhausted, &err),
        err);
    // Materialise n heap vectors (the API's KnnResult shape).  This is host
    // allocation work, spread over the hardware threads (glibc arenas scale).
    std::vector<KnnResult> out(n);
    const auto ke = static_cast<std::size_t>(std::max(k_eff, 0));
    parallel([&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            out[i].distances_sq.assign(d2.get() + i * ke, d2.get() + (i + 1) * ke);
            out[i].average_distance = avg[i];
            out[i].exhausted = exhausted != 0;
        }
    });
    return out;
}

}  // namespace aidw
