// Host-boundary cost split of the drop-in knn_stage at the acceptance
// ladder's 100K rung (acceptance.cpp:356-414): the C-ABI call on the device
// mirror into pinned / pageable buffers, the full C++ knn_stage (C-ABI +
// KnnResult materialisation), and the brute engine — each repeated.
#include <chrono>
#include <cstdio>
#include <memory>
#include "aidw/aidw.hpp"
using namespace aidw;
using C = std::chrono::steady_clock;
static double ms(C::time_point a) { return std::chrono::duration<double, std::milli>(C::now() - a).count(); }
int main() {
    const BoundingBox box{0, 0, 1, 1};
    const std::size_t n = 102400;
    const int k = 15;
    const PointSet data = generate_random_points(n, box, 61, ValueRule::uniform);
    const PointSet queries = generate_random_queries(n, box, 62);
    const BoundingBox bb = compute_bbox(data, queries);
    GridIndex idx = build_index(data, make_grid_config(bb, choose_cell_width(data, bb, 4.0)));
    const aidw_index* mirror = idx.mirror();
    std::printf("mirror %s\n", mirror ? "valid" : "MISSING");
    double* pinned = static_cast<double*>(aidw_pinned_alloc(n * k * sizeof(double)));
    std::unique_ptr<double[]> pageable(new double[n * k]);
    std::vector<double> avg(n);
    int32_t ke = 0, ex = 0;
    aidw_error err{};
    for (int rep = 0; rep < 4; ++rep) {
        auto t = C::now();
        aidw_knn_stage_mirror(queries.xs.data(), queries.ys.data(), n, mirror, k, pinned, nullptr,
                              avg.data(), &ke, &ex, &err);
        const double t_pin = ms(t);
        t = C::now();
        aidw_knn_stage_mirror(queries.xs.data(), queries.ys.data(), n, mirror, k, pageable.get(),
                              nullptr, avg.data(), &ke, &ex, &err);
        const double t_page = ms(t);
        t = C::now();
        auto r = knn_stage(queries, &idx, data, k, KnnEngine::grid, 1);
        const double t_full = ms(t);
        t = C::now();
        std::vector<KnnResult> out(n);
        for (std::size_t i = 0; i < n; ++i) out[i].distances_sq.assign(pinned + i * k, pinned + (i + 1) * k);
        const double t_mat1 = ms(t);
        t = C::now();
        auto b = knn_stage(queries, nullptr, data, k, KnnEngine::brute, 1);
        const double t_brute = ms(t);
        t = C::now();
        auto p = aidw_predict_all(queries, data, r, AidwParams{}, Variant::blocked, 1);
        const double t_interp = ms(t);
        std::printf("rep%d: mirror->pinned %.2f  mirror->pageable %.2f  knn_stage %.2f  "
                    "serial materialise %.2f  brute %.2f  interp %.2f ms\n",
                    rep, t_pin, t_page, t_full, t_mat1, t_brute, t_interp);
    }
    aidw_pinned_free(pinned);
}
