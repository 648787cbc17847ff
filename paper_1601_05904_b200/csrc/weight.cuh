// weight.cuh — the weighting stage (K4) interface.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace aidwb {

// Normalisation frame of the FP32 path: X = (x - ox) * inv_scale maps the
// bbox into [0, 1]; z' = z * 2^zshift keeps |z'| <= 1 (exact scaling).  The
// value hull lives on the device (zhull = {zlo, zhi}, interpolate.hpp:73-80,
// reduced in the pass itself), so the kernels derive zshift from it and no
// host round trip is needed for it.
struct WeightFrame {
    double ox = 0.0, oy = 0.0, inv_scale = 1.0;
    const double* zhull = nullptr;  // device: {zlo, zhi}
    double snap_sq = 0.0;           // interpolate.hpp:86-89 (FP64 path)
};

// 2^zshift with |z 2^zshift| < 1 over the value hull.
__device__ __forceinline__ int frame_zshift(const double* zhull) {
    const double zmax = fmax(fabs(zhull[0]), fabs(zhull[1]));
    int e = 0;
    if (zmax > 0.0 && isfinite(zmax)) frexp(zmax, &e);
    return -e;
}

// Per-query inputs of the weighting stage, in visiting order `pos`
// (perm[pos] = query index; perm == nullptr means identity).
struct WeightQueries {
    const double* qx = nullptr;  // query index order
    const double* qy = nullptr;
    size_t n = 0;
    const uint32_t* perm = nullptr;
    const double* alpha_s = nullptr;   // by pos
    const double* d2min_s = nullptr;   // by pos (FP32 path)
    const uint32_t* nn_s = nullptr;    // by pos (FP32 path)
    const uint32_t* snap_s = nullptr;  // by pos (FP32 path)
};

struct WeightData {
    const double* x = nullptr;  // index order
    const double* y = nullptr;
    const double* z = nullptr;
    size_t m = 0;
    // FP32 path: record order (cell order of the factor-4 grid over the
    // bbox, so tiles are spatially compact); nullptr = index order
    const uint32_t* order = nullptr;
    // the grid behind `order` (its CSR cell_start and shape): K4 re-orders
    // the cells into 8 x 8-cell blocks so each 256-record tile is compact
    const uint32_t* cell_start = nullptr;
    int n_col = 0, n_row = 0;
};

// Optional instrumentation: events recorded around the K4 launch(es) and a
// device counter of recipe-path queries; the caller resolves them after its
// final synchronisation (no mid-pipeline host sync).
struct WeightTimes {
    cudaEvent_t k4_begin = nullptr, k4_end = nullptr;
    unsigned long long* d_alpha4 = nullptr;
};

// FP32 MUFU path (Variant::blocked default).  Writes pred/alpha by query
// index.  When `times` is non-null the K4 launches are bracketed by events.
void weighting_fp32(const WeightQueries& q, const WeightData& d, const WeightFrame& f,
                    double* d_pred, double* d_alpha, WeightTimes* times, cudaStream_t s);

// FP64 path (Variant::naive, pinned_order, AIDW_WEIGHT_FP64): index-order
// accumulation inside each data chunk (chunking a function of m), chunk sums
// added in chunk order; 1 / pow(sqrt(d2), alpha) (1 / (d2 d2) at alpha = 4),
// reference snap / fallback.
// `blocked` selects the reference's blocked-variant arithmetic (recipe /
// exp-log, chunked sums) instead of the naive pow form.
void weighting_fp64(const WeightQueries& q, const WeightData& d, const WeightFrame& f,
                    bool blocked, double* d_pred, double* d_alpha, WeightTimes* times,
                    cudaStream_t s);

// Chunking of the data set for the FP32 kernel; depends on m only, so the
// per-query summation order is independent of n and of the GPU count.
struct WeightSplit {
    size_t tiles = 0;            // padded m / kWeightTile
    unsigned chunks = 1;         // S
    size_t tiles_per_chunk = 0;
};
WeightSplit weight_split(size_t m);
constexpr int kWeightTile = 256;

// K4 on the tensor cores (weight_tc.cu): the far-form d2 of every (query,
// point) pair by tcgen05 MMA.  The engine is chosen from the data split
// alone (a function of m), so a query's result never depends on n, the
// shard or the GPU count; AIDW_K4_ENGINE=simt / tc overrides (tuning).
bool weight_tc_selected(const WeightSplit& sp);
struct WeightTcLaunch {
    const char* tc_rec = nullptr;   // weight_tc_records output
    size_t tiles = 0, tiles_per_chunk = 0;
    unsigned chunks = 1;
    const float4* qhl = nullptr;
    const float4* qpar = nullptr;
    size_t n = 0;
    const uint32_t* flag_a = nullptr;
    const uint32_t* scan_a = nullptr;
    size_t s0 = 0, s1 = 0;
    double2* part = nullptr;
    const float4* tile_box = nullptr;
    const float4* tile_geo = nullptr;
    unsigned classes = 3;  // 1: general-alpha region, 2: recipe region, 3: both
};
size_t weight_tc_record_bytes(size_t tiles);
void weight_tc_records(const float* rec, const float4* tile_geo, size_t tiles, size_t m,
                       char* tc_rec, cudaStream_t s);
void weight_tc_launch(const WeightTcLaunch& l, cudaStream_t s);

// Global switch of the alpha == 4 one-MUFU recipe (aidw_set_alpha4_recipe).
void set_alpha4_recipe(bool enabled);
bool alpha4_recipe_enabled();

// Queries per weighting launch (K4 + settle): bounds the FP64 partial sums
// to slab x chunks x 16 B whatever n is (aidw_set_query_slab; 0 = default,
// 2 GiB of partials).  Always a multiple of 1024.
void set_query_slab(size_t queries);
size_t query_slab(unsigned chunks);

}  // namespace aidwb
