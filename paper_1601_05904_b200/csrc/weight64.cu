// weight64.cu — the FP64 weighting kernels.
//
//  NAIVE   (Variant::naive, pinned_order): restates predict_naive + settle
//          (proj/include/aidw/interpolate.hpp:94-137): w = 1/pow(sqrt(d2), a)
//          (1 / (d2 d2) to ~1 ulp when a == 4); running sums in index order
//          within each data chunk (up to 64, a function of m), the chunk sums
//          added in chunk order by fp64_settle_kernel — so the summation
//          order is chunk-ordered, not the reference's single index-order
//          loop (within the 2e-11 contract).
//  BLOCKED (Variant::blocked under AIDW_WEIGHT_FP64): restates the scalar
//          semantics of predict_blocked_fast (:168-209, :252-381): the exact
//          half-integer recipe d2^(n/4) via products and square roots when
//          2a is an integer in [1, 16], else exp(-a/2 log d2); 256-point
//          chunk partial sums folded into running sums.
// Both: four queries per thread, data streamed through shared memory in
// index order; snap on the first index with d2 <= snap_sq and the non-finite
// fallback to the nearest value (strict <, lowest index) use the indices of
// the k = 1 grid search; clamp to the value hull.
// Compiled with -fmad=false and explicit _rn intrinsics: roundings match
// the reference except CUDA's pow / exp / log (<= 2 ulp vs glibc; contract
// 2e-11 relative).

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

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

// One thread carries QT queries (visiting positions p, p + 128, ...; QT = 1
// by default, more warps beat per-thread ILP for the FP64 chains); the data
// stream through shared memory in index order, 256-point tiles.  The snap
// index and the nearest index come from the k = 1 grid search (FP64, the
// same d2 as here: identical first-index / lowest-index semantics), so the
// inner loop is branch-free FP64 arithmetic: d2, the weight, the sums.
__device__ __forceinline__ bool recipe_alpha(double alpha) {
    const double twice = 2.0 * alpha;
    return twice == floor(twice) && twice >= 1.0 && twice <= 16.0;
}

// Slots ordered alpha == 4 first, then the other recipe alphas, then
// exp / log (BLOCKED), so a warp's queries share one weight formula (a single
// exp/log query would otherwise put its whole warp on the exp/log path, and
// alpha == 4 warps take a specialised loop).
__global__ void fp64_class_kernel(const WeightQueries q, int blocked, uint32_t* __restrict__ flag) {
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < q.n) flag[p] = q.alpha_s[p] != 4.0 ? 1u : 0u;
    (void)blocked;
}

// 1 / x to ~1 ulp on the FP64 pipe: MUFU.RCP64H seed + two Newton steps,
// branch-free (x here is a positive normal d2^2).  The FP64 blocked
// kernel's contract is 2e-11 relative; its sums already differ in order from
// the reference's SIMD lanes.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}

__global__ void fp64_order_kernel(const uint32_t* __restrict__ flag,
                                  const uint32_t* __restrict__ scan, size_t n,
                                  uint32_t* __restrict__ order) {
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const size_t general = static_cast<size_t>(scan[n - 1]) + flag[n - 1];
    const size_t slot = flag[p] ? (n - general) + scan[p] : p - scan[p];
    order[slot] = static_cast<uint32_t>(p);
}

#ifndef AIDW_FP64_THREADS
#define AIDW_FP64_THREADS 256
#endif
constexpr int kFp64Threads = AIDW_FP64_THREADS;

// Each CTA covers QT x blockDim queries against ONE data chunk (blockIdx.y:
// points [chunk * chunk_pts, +chunk_pts), chunking a function of m only) and
// writes its FP64 partial sums; fp64_settle_kernel adds the chunks in order.
template <bool BLOCKED, int QT>
__global__ void __launch_bounds__(kFp64Threads) weight_fp64_kernel(const WeightQueries q,
                                                          const WeightData d,
                                                          const uint32_t* __restrict__ order,
                                                          size_t chunk_pts, size_t s0,
                                                          size_t s1,
                                                          double2* __restrict__ part) {
    __shared__ double2 sxy[kTile64];
    __shared__ double sz[kTile64];
    const size_t p0 = s0 + static_cast<size_t>(blockIdx.x) * blockDim.x * QT + threadIdx.x;
    double qx[QT], qy[QT], alpha[QT], e[QT], sw[QT], swz[QT];
    int n4[QT];
#pragma unroll
    for (int i = 0; i < QT; ++i) {
        const size_t slot = p0 + static_cast<size_t>(i) * blockDim.x;
        const size_t p = slot < s1 ? order[slot] : slot;
        qx[i] = qy[i] = 0.0;
        alpha[i] = 4.0;
        if (slot < s1) {
            const uint32_t qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
            qx[i] = q.qx[qi];
            qy[i] = q.qy[qi];
            alpha[i] = q.alpha_s[p];
        }
        e[i] = -0.5 * alpha[i];
        const double twice = 2.0 * alpha[i];
        // the half-integer recipe (interpolate.hpp:174-192): 2a in [1, 16]
        n4[i] = recipe_alpha(alpha[i]) ? static_cast<int>(twice) : 0;
        sw[i] = swz[i] = 0.0;
    }
    bool four = true;
#pragma unroll
    for (int i = 0; i < QT; ++i) four &= alpha[i] == 4.0;
    const bool all4 = __all_sync(0xFFFFFFFFu, four);
    const size_t c0 = static_cast<size_t>(blockIdx.y) * chunk_pts;
    const size_t c1 = c0 + chunk_pts < d.m ? c0 + chunk_pts : d.m;
    for (size_t base = c0; base < c1; base += kTile64) {
        const int len = static_cast<int>(c1 - base < kTile64 ? c1 - base : kTile64);
        __syncthreads();
        for (int j = threadIdx.x; j < len; j += blockDim.x) {
            sxy[j] = make_double2(d.x[base + j], d.y[base + j]);
            sz[j] = d.z[base + j];
        }
        __syncthreads();
        double cw[QT], cwz[QT];  // chunk partials (BLOCKED)
#pragma unroll
        for (int i = 0; i < QT; ++i) cw[i] = cwz[i] = 0.0;
        if (all4) {  // warp-uniform alpha == 4: w = 1 / (d2 d2) (naive: = 1 / pow(sqrt(d2), 4)
                     // to ~2 ulp, within the FP64 contract; naive and pinned share it)
            for (int j = 0; j < len; ++j) {
                const double2 xy = sxy[j];
                const double z = sz[j];
#pragma unroll
                for (int i = 0; i < QT; ++i) {
                    const double d2 = dsq_rn(qx[i], qy[i], xy.x, xy.y);
                    // d2^2 overflowing to inf weighs 0, as 1 / pow(sqrt(d2), 4)
                    // does in the reference (rcp_nr(inf) would give NaN); the
                    // test runs on the integer pipe (a4 >= 0: inf <=> bits >=
                    // those of inf), off the saturated FP64 pipe
                    const double a4 = __dmul_rn(d2, d2);
                    const double w =
                        __double_as_longlong(a4) < 0x7FF0000000000000LL ? rcp_nr(a4) : 0.0;
                    if (BLOCKED) {
                        cw[i] = __dadd_rn(cw[i], w);
                        cwz[i] = __dadd_rn(cwz[i], __dmul_rn(w, z));
                    } else {  // index-order running sums (predict_naive)
                        sw[i] = __dadd_rn(sw[i], w);
                        swz[i] = __dadd_rn(swz[i], __dmul_rn(w, z));
                    }
                }
            }
        } else
        for (int j = 0; j < len; ++j) {
            const double2 xy = sxy[j];
            const double z = sz[j];
#pragma unroll
            for (int i = 0; i < QT; ++i) {
                const double d2 = dsq_rn(qx[i], qy[i], xy.x, xy.y);
                if (BLOCKED) {
                    const double w = n4[i] ? __drcp_rn(recipe_denominator(d2, n4[i]))
                                           : exp(__dmul_rn(e[i], log(d2)));
                    cw[i] = __dadd_rn(cw[i], w);
                    cwz[i] = __dadd_rn(cwz[i], __dmul_rn(w, z));
                } else {
                    const double w = __drcp_rn(pow(__dsqrt_rn(d2), alpha[i]));
                    sw[i] = __dadd_rn(sw[i], w);
                    swz[i] = __dadd_rn(swz[i], __dmul_rn(w, z));
                }
            }
        }
        if (BLOCKED) {
#pragma unroll
            for (int i = 0; i < QT; ++i) {
                sw[i] = __dadd_rn(sw[i], cw[i]);
                swz[i] = __dadd_rn(swz[i], cwz[i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < QT; ++i) {
        const size_t slot = p0 + static_cast<size_t>(i) * blockDim.x;
        if (slot < s1)
            part[static_cast<size_t>(blockIdx.y) * (s1 - s0) + (slot - s0)] = make_double2(sw[i], swz[i]);
    }
}

// Chunk partials added in chunk order, then the reference's settle
// (interpolate.hpp:109-118): snap -> z[first index within snap distance];
// non-finite or non-positive sums -> nearest value (lowest index on ties);
// clamp to the value hull.
__global__ void fp64_settle_kernel(const WeightQueries q, const WeightFrame f, const WeightData d,
                                   const uint32_t* __restrict__ order,
                                   const double2* __restrict__ part, unsigned chunks,
                                   size_t s0, size_t s1, double* __restrict__ pred,
                                   double* __restrict__ alpha_out) {
    const size_t slot = s0 + static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= s1) return;
    const size_t p = order[slot];
    const uint32_t qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
    double out;
    const uint32_t snap = q.snap_s[p];
    if (snap != kNoId) {
        out = d.z[snap];
    } else {
        double sw = 0.0, swz = 0.0;
        const double2* pp = part + (slot - s0);
        const size_t ld = s1 - s0;
        unsigned c = 0;
        for (; c + 8 <= chunks; c += 8) {  // loads in flight, chunk-order sums
            double2 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = pp[static_cast<size_t>(c + k) * ld];
#pragma unroll
            for (int k = 0; k < 8; ++k) sw = __dadd_rn(sw, v[k].x), swz = __dadd_rn(swz, v[k].y);
        }
        for (; c < chunks; ++c) {
            const double2 v = pp[static_cast<size_t>(c) * ld];
            sw = __dadd_rn(sw, v.x);
            swz = __dadd_rn(swz, v.y);
        }
        bool ok = false;
        out = 0.0;
        if (sw > 0.0 && isfinite(sw) && isfinite(swz)) {
            const double v = __ddiv_rn(swz, sw);
            if (isfinite(v)) {
                const double zlo = f.zhull[0], zhi = f.zhull[1];
                out = v < zlo ? zlo : (v > zhi ? zhi : v);
                ok = true;
            }
        }
        if (!ok) out = d.z[q.nn_s[p]];
    }
    pred[qi] = out;
    if (alpha_out) alpha_out[qi] = q.alpha_s[p];
}

}  // namespace

void weighting_fp64(const WeightQueries& q, const WeightData& d, const WeightFrame& f,
                    bool blocked, double* d_pred, double* d_alpha, WeightTimes* times,
                    cudaStream_t s) {
    if (q.n == 0) return;
    if (!q.snap_s || !q.nn_s)
        throw Failure(AIDW_ERR_RUNTIME, "weighting_fp64: nearest / snap indices missing");
    // queries per thread: 1 (measured at 1M x 1M: 1.18 s vs 1.32 s at 2 and
    // 1.79 s at 4 — the FP64 chains need warps more than per-thread ILP);
    // the per-query arithmetic and order are the same for any QT
    int qt = 1;
    static const int force_qt = [] {  // AIDW_FP64_QT: tuning experiments
        const char* v = std::getenv("AIDW_FP64_QT");
        return v ? std::atoi(v) : 0;
    }();
    if (force_qt == 1 || force_qt == 2 || force_qt == 4) qt = force_qt;
    DBuf<uint32_t> flag(q.n, s), scan(q.n, s), order(q.n, s);
    LAUNCH(fp64_class_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q, blocked ? 1 : 0,
           flag.get());
    exclusive_scan_u32(flag.get(), scan.get(), q.n, s);
    LAUNCH(fp64_order_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, flag.get(), scan.get(), q.n,
           order.get());
    // data chunks: the FP32 path's split (a function of m only) — enough CTAs
    // at small n (100K x 100K: 391 query blocks x 64 chunks)
    const WeightSplit sp = weight_split(d.m);
    const size_t chunk_pts = sp.tiles_per_chunk * static_cast<size_t>(kWeightTile);
    const unsigned chunks = static_cast<unsigned>((d.m + chunk_pts - 1) / chunk_pts);
    // queries in slabs (see query_slab): partials bounded whatever n is
    const size_t slab = std::min(q.n, query_slab(chunks));
    DBuf<double2> part(static_cast<size_t>(chunks) * slab, s);
    size_t s0 = 0, s1 = 0;
    auto go = [&](auto kernel, int k) {
        const dim3 grid(ceil_div(s1 - s0, static_cast<size_t>(kFp64Threads * k)), chunks);
        LAUNCH(kernel, grid, kFp64Threads, 0, s, q, d, order.get(), chunk_pts, s0, s1, part.get());
    };
    if (times && times->k4_begin) record_event(times->k4_begin, s);
    for (s0 = 0; s0 < q.n; s0 += slab) {
        s1 = std::min(q.n, s0 + slab);
        if (blocked) {
            if (qt == 4) go(weight_fp64_kernel<true, 4>, 4);
            else if (qt == 2) go(weight_fp64_kernel<true, 2>, 2);
            else go(weight_fp64_kernel<true, 1>, 1);
        } else {
            if (qt == 4) go(weight_fp64_kernel<false, 4>, 4);
            else if (qt == 2) go(weight_fp64_kernel<false, 2>, 2);
            else go(weight_fp64_kernel<false, 1>, 1);
        }
        if (times && times->k4_end && s1 == q.n) record_event(times->k4_end, s);
        LAUNCH(fp64_settle_kernel, ceil_div(s1 - s0, kThreads), kThreads, 0, s, q, f, d,
               order.get(), part.get(), chunks, s0, s1, d_pred, d_alpha);
    }
}

}  // namespace aidwb
