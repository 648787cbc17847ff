// weight64.cu — the FP64 weighting kernels.
//
//  NAIVE   (Variant::naive, pinned_order): restates predict_naive + settle
//          (proj/include/aidw/interpolate.hpp:94-137): w = 1/pow(sqrt(d2), a),
//          sums in index order.
//  BLOCKED (Variant::blocked under AIDW_WEIGHT_FP64): restates the scalar
//          semantics of predict_blocked_fast (:168-209, :252-381): the exact
//          half-integer recipe d2^(n/4) via products and square roots when
//          2a is an integer in [1, 16], else exp(-a/2 log d2); 256-point
//          chunk partial sums folded into running sums.
// Both: one thread per query, data streamed through shared memory in index
// order, snap on the first index with d2 <= snap_sq, non-finite sums ->
// nearest value (strict <, lowest index), clamp to the value hull.
// Compiled with -fmad=false and explicit _rn intrinsics: roundings match
// the reference except CUDA's pow / exp / log (<= 2 ulp vs glibc; contract
// 2e-11 relative).

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "weight.cuh"

namespace aidwb {

namespace {

constexpr int kTile64 = 256;  // = the reference's kStageSize chunk

// d2^(n/4) for the half-integer recipe (interpolate.hpp:194-209).
__device__ __forceinline__ double recipe_denominator(double d2, int n4) {
    const int squares = n4 / 4;
    double den = squares > 0 ? d2 : 1.0;
    for (int p = 1; p < squares; ++p) den = __dmul_rn(den, d2);
    if (n4 & 3) {
        const double r = __dsqrt_rn(d2);
        if (n4 & 2) den = __dmul_rn(den, r);
        if (n4 & 1) den = __dmul_rn(den, __dsqrt_rn(r));
    }
    return den;
}

template <bool BLOCKED>
__global__ void __launch_bounds__(128) weight_fp64_kernel(const WeightQueries q,
                                                          const WeightFrame f,
                                                          const WeightData d,
                                                          double* __restrict__ pred,
                                                          double* __restrict__ alpha_out) {
    __shared__ double sx[kTile64], sy[kTile64], sz[kTile64];
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = p < q.n;
    uint32_t qi = 0;
    double qx = 0.0, qy = 0.0, alpha = 1.0;
    if (live) {
        qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
        qx = q.qx[qi];
        qy = q.qy[qi];
        alpha = q.alpha_s[p];
    }
    bool active = live;
    double out = 0.0;
    const double e = -0.5 * alpha;
    const double twice = 2.0 * alpha;
    const bool exact = twice == floor(twice) && twice >= 1.0 && twice <= 16.0;
    const int n4 = exact ? static_cast<int>(twice) : 0;
    double sw = 0.0, swz = 0.0;
    double best = 0.0;
    size_t best_i = 0;
    for (size_t base = 0; base < d.m; base += kTile64) {
        const int len = static_cast<int>(d.m - base < kTile64 ? d.m - base : kTile64);
        __syncthreads();
        for (int j = threadIdx.x; j < len; j += blockDim.x) {
            sx[j] = d.x[base + j];
            sy[j] = d.y[base + j];
            sz[j] = d.z[base + j];
        }
        __syncthreads();
        if (!active) continue;
        double cw = 0.0, cwz = 0.0;  // chunk partials (BLOCKED)
        for (int j = 0; j < len; ++j) {
            const double d2 = dsq_rn(qx, qy, sx[j], sy[j]);
            if (d2 <= f.snap_sq) {
                out = sz[j];
                active = false;
                break;
            }
            if ((base == 0 && j == 0) || d2 < best) {
                best = d2;
                best_i = base + j;
            }
            if (BLOCKED) {
                const double w = exact ? __ddiv_rn(1.0, recipe_denominator(d2, n4))
                                       : exp(__dmul_rn(e, log(d2)));
                cw = __dadd_rn(cw, w);
                cwz = __dadd_rn(cwz, __dmul_rn(w, sz[j]));
            } else {
                const double w = __ddiv_rn(1.0, pow(__dsqrt_rn(d2), alpha));
                sw = __dadd_rn(sw, w);
                swz = __dadd_rn(swz, __dmul_rn(w, sz[j]));
            }
        }
        if (BLOCKED && active) {
            sw = __dadd_rn(sw, cw);
            swz = __dadd_rn(swz, cwz);
        }
    }
    if (!live) return;
    if (active) {
        // settle (interpolate.hpp:109-118)
        bool ok = false;
        if (sw > 0.0 && isfinite(sw) && isfinite(swz)) {
            const double v = __ddiv_rn(swz, sw);
            if (isfinite(v)) {
                out = v < f.zlo ? f.zlo : (v > f.zhi ? f.zhi : v);
                ok = true;
            }
        }
        if (!ok) out = d.z[best_i];
    }
    pred[qi] = out;
    if (alpha_out) alpha_out[qi] = alpha;
}

}  // namespace

void weighting_fp64(const WeightQueries& q, const WeightData& d, const WeightFrame& f,
                    bool blocked, double* d_pred, double* d_alpha, WeightTimes* times,
                    cudaStream_t s) {
    if (q.n == 0) return;
    if (times && times->k4_begin) CK(cudaEventRecord(times->k4_begin, s));
    if (blocked) {
        LAUNCH(weight_fp64_kernel<true>, ceil_div(q.n, 128), 128, 0, s, q, f, d, d_pred, d_alpha);
    } else {
        LAUNCH(weight_fp64_kernel<false>, ceil_div(q.n, 128), 128, 0, s, q, f, d, d_pred, d_alpha);
    }
    if (times && times->k4_end) CK(cudaEventRecord(times->k4_end, s));
}

}  // namespace aidwb
