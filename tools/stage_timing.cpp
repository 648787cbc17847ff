// Host-boundary timing of the drop-in C++ API on the acceptance ladder
// (acceptance.cpp:356-414 pattern): per call wall time of build_index,
// knn_stage (grid / brute) and aidw_predict_all, each run twice.
#include <chrono>
#include <cstdio>
#include "aidw/aidw.hpp"
using namespace aidw;
using C = std::chrono::steady_clock;
static double ms(C::time_point a) { return std::chrono::duration<double, std::milli>(C::now() - a).count(); }
int main() {
  const BoundingBox box{0, 0, 1, 1};
  const AidwParams params;
  for (std::size_t size : {10240u, 51200u, 102400u}) {
    const PointSet data = generate_random_points(size, box, 61, ValueRule::uniform);
    const PointSet queries = generate_random_queries(size, box, 62);
    for (int rep = 0; rep < 2; ++rep) {
      auto t = C::now();
      const BoundingBox bb = compute_bbox(data, queries);
      GridIndex idx = build_index(data, make_grid_config(bb, choose_cell_width(data, bb, 4.0)));
      double tb = ms(t); t = C::now();
      auto kg = knn_stage(queries, &idx, data, params.k, KnnEngine::grid, 1);
      double tk = ms(t); t = C::now();
      auto kb = knn_stage(queries, nullptr, data, params.k, KnnEngine::brute, 1);
      double tkb = ms(t); t = C::now();
      auto r = aidw_predict_all(queries, data, kg, params, Variant::blocked, 1);
      double ti = ms(t); t = C::now();
      auto r2 = aidw_predict_all(queries, data, kb, params, Variant::blocked, 1);
      double ti2 = ms(t);
      std::printf("%zu rep%d: build %.2f knn_grid %.2f knn_brute %.2f interp %.2f interp2 %.2f ms\n", size, rep, tb, tk, tkb, ti, ti2);
    }
  }
}
