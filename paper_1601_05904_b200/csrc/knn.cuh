// knn.cuh — argument blocks of K2 (grid / brute kNN) and K3 (alpha).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace aidwb {

// Scalars of the adaptive chain, precomputed on the host with the
// reference's own expressions (adaptive.hpp:20-60).
struct AlphaParams {
    double r_exp;         // 1 / (2 sqrt(m / area))
    double pi_over_rmax;  // std::numbers::pi / r_max
    double r_min, r_max;
    double lv[5];
};

struct KnnArgs {
    // grid (sorted CSR arrays) — grid engine
    GridGeom g;
    const uint32_t* cell_start = nullptr;
    const uint32_t* sorted_ids = nullptr;
    const double2* sorted_xy = nullptr;  // cell-sorted {x, y}
    // summed-area table of the cell counts, column-major (n_col + 1) x
    // (n_row + 1): PT[c][r] = points in rows < r, columns < c (built by
    // run_knn_grid); block counts in O(1)
    const uint32_t* rect_prefix = nullptr;
    // data in index order — brute engine
    const double* dx = nullptr;
    const double* dy = nullptr;
    size_t m = 0;
    // queries in input order, visiting order perm[pos], cells qcell[pos]
    const double* qx = nullptr;
    const double* qy = nullptr;
    const uint32_t* perm = nullptr;
    const uint32_t* qcell = nullptr;  // query keys (query_key: block-major, qkey_nbc blocks/row)
    int qkey_nbc = 0;
    int stage = 1;  // stage the CTA's cell patch in shared memory (AIDW_K2_STAGE=0: off)
    size_t n = 0;
    int k = 1;       // requested
    int k_eff = 1;   // min(k, m)
    double snap_sq = -1.0;
    double ring_margin = 1.0 - 1.0e-9;
    // outputs indexed by query index (nullable)
    double* d2_out = nullptr;   // n * k_eff
    uint32_t* id_out = nullptr; // n * k_eff
    double* avg_out = nullptr;  // n
    // outputs indexed by visiting position (nullable)
    double* alpha_s = nullptr;
    double* d2min_s = nullptr;
    uint32_t* nn_s = nullptr;
    uint32_t* snap_s = nullptr;
    int compute_alpha = 0;
    double const_alpha = 0.0;
    AlphaParams ap{};
    long long* fail_alpha = nullptr;
    unsigned long long* candidates = nullptr;      // points scanned (after pruning)
    unsigned long long* ref_candidates = nullptr;  // the reference's scan: final-level block
    // scratch for k > 64
    double* scratch_d = nullptr;
    uint32_t* scratch_id = nullptr;
};

void run_knn_grid(KnnArgs a, cudaStream_t s);
void run_knn_brute(KnnArgs a, cudaStream_t s);
void run_alpha(const double* d_robs, size_t n, const AlphaParams& p, double* d_alpha,
               long long* d_fail, cudaStream_t s);

}  // namespace aidwb
