// The acceptance gate's criteria 6-8 ladder (acceptance.cpp:356-414) with the
// drop-in knn_stage split into phases: how much of the grid kNN stage at
// each rung is the C-ABI call vs the KnnResult materialisation, on first
// and repeated calls.  Build: see tools/session/r02_s37.sh.
#include <chrono>
#include <cstdio>
#include "aidw/aidw.hpp"
using namespace aidw;
using C = std::chrono::steady_clock;
static double ms(C::time_point a) { return std::chrono::duration<double, std::milli>(C::now() - a).count(); }
int main() {
    const BoundingBox box{0, 0, 1, 1};
    const AidwParams params;
    for (int pass = 0; pass < 2; ++pass) {
        for (std::size_t size : {std::size_t{10240}, std::size_t{51200}, std::size_t{102400}}) {
            const PointSet data = generate_random_points(size, box, 61, ValueRule::uniform);
            const PointSet queries = generate_random_queries(size, box, 62);
            const BoundingBox bb = compute_bbox(data, queries);
            auto t = C::now();
            GridIndex idx = build_index(data, make_grid_config(bb, choose_cell_width(data, bb, 4.0)));
            const double tb = ms(t);
            t = C::now();
            auto r = knn_stage(queries, &idx, data, params.k, KnnEngine::grid, 1);
            const double tk = ms(t);
            t = C::now();
            auto p = aidw_predict_all(queries, data, r, params, Variant::blocked, 1);
            const double ti = ms(t);
            double tbr = 0;
            if (size == 102400) {
                t = C::now();
                auto b = knn_stage(queries, nullptr, data, params.k, KnnEngine::brute, 1);
                tbr = ms(t);
            }
            std::printf("pass %d %6zu: build %.2f knn %.2f interp %.2f brute %.2f ms (knn share %.1f%%)\n",
                        pass, size, tb, tk, ti, tbr, 100 * tk / (tb + tk + ti));
        }
    }
}
