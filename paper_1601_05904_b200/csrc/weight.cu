// weight.cu — K4: the O(m·n) inverse-distance weighting on sm_100a (FP32).
//
// Replaces the weighting loops of aidw_predict_all / idw_predict_all
// (proj/include/aidw/interpolate.hpp:252-381, :426-489).  Design:
//
//  * Data records: 256-point tiles of 9 SoA float components in 8 x 8-cell
//    block order of the factor-4 grid (compact squares): x / y / z as FP32
//    hi/lo pairs of the unit-box-normalised FP64 values (the NEAR form,
//    dx = (x_hi - q_hi) + (x_lo - q_lo), ~48 bits, no FP64 op or F2F per
//    pair) and the tile-centred FAR form -2 p'x, -2 p'y, |p'|^2 (d2 in three
//    FP32 ops).  Padded records weigh exactly 0 in the near form, the only
//    one a partial tile uses.
//  * Each CTA (256 threads, 4 queries per thread as two f32x2 pairs) streams
//    the tiles of one data chunk through a 4-stage shared-memory ring filled
//    by the bulk-copy engine (cp.async.bulk + mbarrier complete_tx; SASS
//    UBLKCP); the last warp done with a stage refills it, so warps drift
//    instead of meeting at a barrier.  Queries are visited in Morton order.
//  * Per (query, tile): FAR when the query's distance to the tile's box
//    exceeds max(R_far, half the tile diagonal), else NEAR (Kahan-compensated
//    sums with hi/lo z).  A function of the (query, tile) pair only.
//  * Weights: general alpha, ratio-scaled w' = (d2 / d2_min)^(-alpha/2) =
//    ex2(c lg2(d2) + b) (G1: MUFU ex2; G2: ex2 as a degree-5 polynomial on
//    the FMA pipe, interleaved 1:1 per warp); alpha == 4 exactly (98 % of
//    uniform-data queries, the reference's half-integer recipe,
//    interpolate.hpp:174-209): w' = 1 / (d2 s)^2, and in far tiles two of
//    every four points share one reciprocal.  One launch serves both classes
//    (general CTAs first); the formula is chosen per query, never per warp.
//  * Per-tile FP32 sums are folded into FP64 accumulators; data chunks
//    (S = f(m) only) give enough CTAs at small n and are summed in chunk
//    order by the settle kernel, deterministically (no atomics).
//  * settle: snap -> z[first index within snap distance]; analytic overflow
//    test in log space reproduces the FP64 reference's non-finite sums ->
//    nearest value (lowest index on ties); clamp to the value hull.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <string>

#include "common.cuh"
#include "weight.cuh"
#include "weight_ops.cuh"

namespace aidwb {

namespace {

using namespace wops;

#ifndef AIDW_K4_THREADS
#define AIDW_K4_THREADS 256
#endif
#ifndef AIDW_K4_MINB
#define AIDW_K4_MINB 2
#endif
constexpr int kK4Threads = AIDW_K4_THREADS;
#ifndef AIDW_K4_ALLPAIRS
#define AIDW_K4_ALLPAIRS 0
#endif
#ifndef AIDW_K4_MIXPAIRS
#define AIDW_K4_MIXPAIRS 0
#endif
#ifndef AIDW_K4_FAR_UNROLL
#define AIDW_K4_FAR_UNROLL 2
#endif
constexpr int kFarUnroll = AIDW_K4_FAR_UNROLL;  // 4-point groups per far-loop trip
#ifndef AIDW_K4_STAGES
#define AIDW_K4_STAGES 4
#endif
constexpr int kStages = AIDW_K4_STAGES;
constexpr int kMaxChunks = 32;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------ record prep
__device__ __forceinline__ void split_hilo(double v, float& hi, float& lo) {
    hi = __double2float_rn(v);
    lo = __double2float_rn(v - static_cast<double>(hi));
}

// Record i = data point order[i] (8 x 8-cell blocks of the factor-4 grid, so
// a 256-point tile is a compact square), or point i without order.
__global__ void prep_data_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ z, const uint32_t* __restrict__ order,
                                 size_t m, size_t mp, double ox, double oy, double inv_scale,
                                 const double* __restrict__ zhull, float* __restrict__ rec) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= mp) return;
    const double zmul = ldexp(1.0, frame_zshift(zhull));
    float* r = rec + (i / kWeightTile) * kTileFloats + (i % kWeightTile);
    if (i < m) {
        const size_t j = order ? order[i] : i;
        float xh, xl, yh, yl, zh, zl;
        split_hilo((x[j] - ox) * inv_scale, xh, xl);
        split_hilo((y[j] - oy) * inv_scale, yh, yl);
        split_hilo(z[j] * zmul, zh, zl);
        r[kXH * kWeightTile] = xh, r[kYH * kWeightTile] = yh;
        r[kXL * kWeightTile] = xl, r[kYL * kWeightTile] = yl;
        r[kZH * kWeightTile] = zh, r[kZL * kWeightTile] = zl;
    } else {  // padding: weight exactly 0 in the near form (the only one a
              // partial tile uses)
        r[kXH * kWeightTile] = 1.0e30f, r[kYH * kWeightTile] = 1.0e30f;
        r[kXL * kWeightTile] = 0.0f, r[kYL * kWeightTile] = 0.0f;
        r[kZH * kWeightTile] = 0.0f, r[kZL * kWeightTile] = 0.0f;
    }
}

// One CTA per tile (a thread per record): bounding box of the real records
// (hi parts), centre c,
// near threshold, and the far-form components.  A (query, tile) pair is FAR
// when the query's distance d to the box exceeds both R_far and 0.3 box
// diagonals: then |q'| + |p'| <= d + diag <= 4.4 d, so the expanded d2 loses
// at most a few ulp of 19 d2 (the measured contract error is unchanged from
// a 0.5-diagonal rule: tools/accuracy sweeps in DESIGN.md).
// Partial (padded) tiles are always NEAR.
__global__ void __launch_bounds__(kWeightTile) tile_geo_kernel(float* __restrict__ rec, size_t m,
                                                              size_t tiles, float rfar2, float diagf2,
                                                              float4* __restrict__ box,
                                                              float4* __restrict__ geo) {
    // one CTA per tile, one thread per record
    __shared__ float s_red[4][kWeightTile / 32];
    const size_t tile = blockIdx.x;
    const int j = threadIdx.x, lane = j & 31, warp = j >> 5;
    float* t = rec + tile * kTileFloats;
    const bool real = tile * kWeightTile + j < m;
    const float pxh = t[kXH * kWeightTile + j], pyh = t[kYH * kWeightTile + j];
    float x0 = real ? pxh : 3.0e38f, y0 = real ? pyh : 3.0e38f;
    float x1 = real ? pxh : -3.0e38f, y1 = real ? pyh : -3.0e38f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        x0 = fminf(x0, __shfl_xor_sync(0xFFFFFFFFu, x0, o));
        y0 = fminf(y0, __shfl_xor_sync(0xFFFFFFFFu, y0, o));
        x1 = fmaxf(x1, __shfl_xor_sync(0xFFFFFFFFu, x1, o));
        y1 = fmaxf(y1, __shfl_xor_sync(0xFFFFFFFFu, y1, o));
    }
    if (lane == 0) {
        s_red[0][warp] = x0, s_red[1][warp] = y0, s_red[2][warp] = x1, s_red[3][warp] = y1;
    }
    __syncthreads();
    x0 = s_red[0][0], y0 = s_red[1][0], x1 = s_red[2][0], y1 = s_red[3][0];
#pragma unroll
    for (int w = 1; w < kWeightTile / 32; ++w) {
        x0 = fminf(x0, s_red[0][w]), y0 = fminf(y0, s_red[1][w]);
        x1 = fmaxf(x1, s_red[2][w]), y1 = fmaxf(y1, s_red[3][w]);
    }
    const float cx = 0.5f * (x0 + x1), cy = 0.5f * (y0 + y1);
    const float gx = x1 - x0, gy = y1 - y0;
    const bool partial = (tile + 1) * kWeightTile > m;
#if AIDW_K4_EXPERIMENT_ALLFAR  // timing experiment only: every full tile far
    const float thr2 = partial ? INFINITY : 1.0e-8f;
#else
    const float thr2 =
        partial ? INFINITY : fmaxf(fmaxf(rfar2, 1.0e-8f), 1.001f * diagf2 * fmaf(gx, gx, gy * gy));
#endif
    if (j == 0) {
        box[tile] = make_float4(x0, y0, x1, y1);
        geo[tile] = make_float4(cx, cy, thr2, 0.0f);
    }
    float px2 = 0.0f, py2 = 0.0f, pp = 0.0f;
    if (real) {
        const double px = (static_cast<double>(pxh) - cx) + static_cast<double>(t[kXL * kWeightTile + j]);
        const double py = (static_cast<double>(pyh) - cy) + static_cast<double>(t[kYL * kWeightTile + j]);
        px2 = __double2float_rn(-2.0 * px);
        py2 = __double2float_rn(-2.0 * py);
        pp = __double2float_rn(px * px + py * py);
    }
    t[kPX * kWeightTile + j] = px2;
    t[kPY * kWeightTile + j] = py2;
    t[kPP * kWeightTile + j] = pp;
}

std::atomic<bool> g_alpha4_recipe{true};

// Recipe-class range: alpha == 4 queries take w' = 1 / (d2 s)^2 with s a
// power of two (exact) putting d2min s in [1e-9, 2e-9) when d2min < 1e-9,
// else s = 1; the far path pairs two points per reciprocal, so (d2 s)^4
// products must stay inside FP32: d2min >= kRecipeMinD2 (unit-box units).
// Smaller non-snapped d2min (< 1e-8.5 of the domain) take the general path.
constexpr double kRecipeMinD2 = 1.0e-17;
constexpr double kRecipeLowD2 = 1.0e-9;

// Query classes: A = the exact alpha == 4 recipe (or snapped: result
// replaced anyway); the other (general-alpha) queries split into G1 (exp2 on
// MUFU) and G2 (exp2 as a polynomial on the FMA pipe) by a hash of the
// query's normalised FP32 coordinates (the hi parts K4 itself uses) — a
// function of the query alone, so its formula (and result) never depends on
// sharding, order or GPU count, and frame-relative, so translating the whole
// problem (acceptance criterion 5, 1e-9) does not re-class it.  Half / half
// balances the MUFU and FMA pipes.
__device__ __forceinline__ bool poly_class(float xh, float yh, unsigned g2_threshold) {
    unsigned h = static_cast<unsigned>(__float_as_int(xh)) * 0x9E3779B1u;
    h ^= static_cast<unsigned>(__float_as_int(yh)) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0xC2B2AE3Du;
    return h < g2_threshold;
}

// K4 visiting order: positions sorted along a Morton (Z) curve of the
// normalised query coordinates, so the 128 queries of a warp and the 1024 of
// a CTA are spatially compact — they agree on which tiles are near, which
// keeps the warps of a CTA in step.  (The order never changes a result.)
__device__ __forceinline__ uint32_t spread16(uint32_t v) {
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

__global__ void morton_keys_kernel(const WeightQueries q, WeightFrame f, uint32_t* __restrict__ key,
                                   uint32_t* __restrict__ pos) {
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= q.n) return;
    const uint32_t qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
    const double xn = (q.qx[qi] - f.ox) * f.inv_scale, yn = (q.qy[qi] - f.oy) * f.inv_scale;
    // 256 x 256 Morton cells: fine enough for warp / CTA locality, and a
    // 16-bit key sorts in two radix passes
    const uint32_t cx = static_cast<uint32_t>(fmin(fmax(xn * 256.0, 0.0), 255.0));
    const uint32_t cy = static_cast<uint32_t>(fmin(fmax(yn * 256.0, 0.0), 255.0));
    key[p] = spread16(cx) | (spread16(cy) << 1);
    pos[p] = static_cast<uint32_t>(p);
}

// Flags by Morton rank j (p = zpos[j]).
// Recipe sub-classes after alpha = 4 (region order): alpha = 2, 1, 3, and
// the class codes the records carry (qpar.x and .w; general classes: 0, 2).
constexpr int kRecipeSubs = 3;
struct RecipeFlags {
    uint32_t* flag[kRecipeSubs];
    uint32_t* scan[kRecipeSubs];
};

__global__ void class_flags_kernel(const WeightQueries q, WeightFrame f, int recipe,
                                   unsigned g2_threshold, const uint32_t* __restrict__ zpos,
                                   uint32_t* __restrict__ flag_a, RecipeFlags rf,
                                   uint32_t* __restrict__ flag_g2) {
    const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= q.n) return;
    const size_t p = zpos[j];
    const double d2n = q.d2min_s[p] * f.inv_scale * f.inv_scale;
    const bool snapped = q.snap_s[p] != kNoId;
    const double alpha = q.alpha_s[p];
    // recipe classes — integer alpha among the reference's half-integer
    // recipes (interpolate.hpp:174-209): alpha = 4 (w = 1/d^4; also every
    // snapped query), 2 (1/d^2, the reference's default IDW exponent), 1 and 3
    const bool ok = recipe && !snapped && d2n >= kRecipeMinD2;
    const bool sub[kRecipeSubs] = {ok && alpha == 2.0, ok && alpha == 1.0, ok && alpha == 3.0};
    const bool a = (ok && alpha == 4.0) || snapped || sub[0] || sub[1] || sub[2];
    const uint32_t qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
    flag_a[j] = a ? 1u : 0u;
#pragma unroll
    for (int k = 0; k < kRecipeSubs; ++k) rf.flag[k][j] = sub[k] ? 1u : 0u;
    const float xh = __double2float_rn((q.qx[qi] - f.ox) * f.inv_scale);
    const float yh = __double2float_rn((q.qy[qi] - f.oy) * f.inv_scale);
    flag_g2[j] = (!a && poly_class(xh, yh, g2_threshold)) ? 1u : 0u;
}

// 3-way partition (general G1/G2 interleaved, then A) fused with the
// per-query record build.
__global__ void query_records_kernel(const WeightQueries q, WeightFrame f,
                                     const uint32_t* __restrict__ zpos,
                                     const uint32_t* __restrict__ flag_a,
                                     const uint32_t* __restrict__ scan_a,
                                     const RecipeFlags rf,
                                     const uint32_t* __restrict__ flag_g2,
                                     const uint32_t* __restrict__ scan_g2,
                                     uint32_t* __restrict__ order, float4* __restrict__ qhl,
                                     float4* __restrict__ qpar, double* __restrict__ lshift,
                                     unsigned long long* __restrict__ alpha4) {
    const size_t jz = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (jz >= q.n) return;
    const size_t p = zpos[jz];
    // the five flag arrays are scanned as one concatenation: an array's
    // exclusive scan is offset by its first value (the earlier arrays' total)
    const uint32_t base_g2 = scan_g2[0];
    const size_t num_a = static_cast<size_t>(scan_a[q.n - 1]) + flag_a[q.n - 1];
    const size_t num_g2 = static_cast<size_t>(scan_g2[q.n - 1] - base_g2) + flag_g2[q.n - 1];
    const size_t num_g1 = q.n - num_a - num_g2;
    const bool is_a = flag_a[jz] != 0, is_g2 = flag_g2[jz] != 0;
    int sub = -1;  // recipe sub-class (-1: alpha = 4)
    // General queries: 64-query blocks of G1 and G2 alternate, so a warp's
    // pair 0 (slots 0, 1) is G1 and pair 1 (slots 2, 3) is G2 — each warp
    // issues MUFU and FMA-pipe exponentials side by side.  Leftovers follow.
    // The general region comes first so its 128-query blocks align with warps.
    size_t i;
    if (is_a) {  // recipe region: alpha = 4 first, then alpha = 2, 1, 3
        size_t cnt[kRecipeSubs], before = 0, total = 0;
#pragma unroll
        for (int k = 0; k < kRecipeSubs; ++k) {
            const uint32_t base = rf.scan[k][0];
            cnt[k] = static_cast<size_t>(rf.scan[k][q.n - 1] - base) + rf.flag[k][q.n - 1];
            total += cnt[k];
            before += rf.scan[k][jz] - base;
            if (rf.flag[k][jz]) sub = k;
        }
        size_t off = num_a - total;  // alpha = 4 count
        if (sub < 0) {
            i = num_g1 + num_g2 + (scan_a[jz] - before);
        } else {
            for (int k = 0; k < sub; ++k) off += cnt[k];
            i = num_g1 + num_g2 + off + (rf.scan[sub][jz] - rf.scan[sub][0]);
        }
    } else {
        const size_t sg2 = scan_g2[jz] - base_g2;
        const size_t j = is_g2 ? sg2 : jz - scan_a[jz] - sg2;
        const size_t both = (num_g1 < num_g2 ? num_g1 : num_g2) / 64;  // full block pairs
        if (j < 64 * both) {
            i = (j / 64) * 128 + (is_g2 ? 64 : 0) + (j % 64);
        } else if (!is_g2) {
            i = 128 * both + (j - 64 * both);
        } else {
            i = 128 * both + (num_g1 - 64 * both) + (j - 64 * both);
        }
    }
    order[i] = static_cast<uint32_t>(p);
    const uint32_t qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
    float xh, xl, yh, yl;
    split_hilo((q.qx[qi] - f.ox) * f.inv_scale, xh, xl);
    split_hilo((q.qy[qi] - f.oy) * f.inv_scale, yh, yl);
    qhl[i] = make_float4(xh, yh, xl, yl);
    const double alpha = q.alpha_s[p];
    const double d2n = q.d2min_s[p] * f.inv_scale * f.inv_scale;
    const float c = __double2float_rn(-0.5 * alpha);
    // general path: w' = ex2(c lg2(d2) + b) with b = -c lg2(d2min) so w' <= 1
    const float b = __double2float_rn(-static_cast<double>(c) * log2(d2n));
    // recipe path: w' = rcp((d2 s)^2), s = 1 or a power of two (exact)
    const bool snapped = q.snap_s[p] != kNoId;
    const double s = (snapped || d2n >= kRecipeLowD2) ? 1.0 : exp2(ceil(log2(kRecipeLowD2 / d2n)));
    // recipe queries carry their class code in x and w (recipe_a / recipe_rsq)
    if (is_a) {
        const float code = sub == 0 ? kCodeA2 : sub == 1 ? kCodeA1 : sub == 2 ? kCodeA3 : kCodeA4;
        qpar[i] = make_float4(code, 0.0f, sub < 0 ? static_cast<float>(s) : 1.0f, code);
    } else {
        qpar[i] = make_float4(c, b, static_cast<float>(s), is_g2 ? 2.0f : 0.0f);
    }
    // log2(true weight) = log2(kernel weight) + shift (settle's overflow test)
    const double l2inv = log2(f.inv_scale);
    // (recipe weights are the true ones scaled by inv_scale^alpha, alpha = 4
    // also by s^2)
    lshift[i] = !is_a    ? -static_cast<double>(b) - 2.0 * static_cast<double>(c) * l2inv
              : sub < 0  ? 2.0 * log2(s) + 4.0 * l2inv
                         : alpha * l2inv;
    if (alpha == 4.0 && alpha4) atomicAdd(alpha4, 1ull);
}

// ------------------------------------------------------------ K4
struct K4Args {
    const float* rec;  // SoA tiles, kTileFloats floats each
    size_t tiles, tiles_per_chunk;
    unsigned chunks;
    const float4* qhl;
    const float4* qpar;
    size_t n;
    const uint32_t* flag_a;  // class counts: A = scan_a[n-1] + flag_a[n-1]
    const uint32_t* scan_a;
    size_t s0, s1;            // this launch's query slab [s0, s1) of the visiting order
    double2* part;            // chunks x (s1 - s0) (chunk-major: coalesced), by position - s0
    const float4* tile_box;   // hi-coordinate box of every tile's real records
    const float4* tile_geo;   // {cx, cy, near threshold^2, 0}
    unsigned classes;         // 1: general region, 2: recipe region, 3: both
};

// Recipe classes (qpar.x / qpar.w code): 1 alpha = 4 (w = 1/t^2, paired
// reciprocals), 3 alpha = 2 (w = 1/t, paired), 4 alpha = 1 (w = rsqrt t),
// 5 alpha = 3 (w = (rsqrt t)^3).  Mixed warps (only those straddling a class
// boundary of the recipe region) evaluate every form and pick per slot, with
// the same roundings as the pure modes, so a query's result never depends
// on its warp-mates.  Selects, not arithmetic blends: padding gives t = inf.
__device__ __forceinline__ bool paired_code(float c) { return c == kCodeA4 || c == kCodeA2; }
__device__ __forceinline__ f2 recipe_a(f2 t, f2 code) {  // paired classes: t^2 or t
    float t0, t1, c0, c1;
    up2(t, t0, t1);
    up2(code, c0, c1);
    return pk2(c0 == kCodeA4 ? __fmul_rn(t0, t0) : t0, c1 == kCodeA4 ? __fmul_rn(t1, t1) : t1);
}
__device__ __forceinline__ f2 recipe_rsq(f2 t, f2 code) {  // rsqrt classes: r or r^3
    const f2 r = rsq2(t);
    const f2 r3 = cube2(r);
    float a0, a1, b0, b1, c0, c1;
    up2(r, a0, a1);
    up2(r3, b0, b1);
    up2(code, c0, c1);
    return pk2(c0 == kCodeA3 ? b0 : a0, c1 == kCodeA3 ? b1 : a1);
}
__device__ __forceinline__ f2 sel_paired(f2 code, f2 x, f2 y) {
    float x0, x1, y0, y1, c0, c1;
    up2(x, x0, x1);
    up2(y, y0, y1);
    up2(code, c0, c1);
    return pk2(paired_code(c0) ? x0 : y0, paired_code(c1) ? x1 : y1);
}

// Per-thread query state: QT queries as QT/2 f32x2 pairs.
// The coordinates are re-read per tile (L1-resident, 4 x 16 B per thread per
// 256-point tile) instead of being held across the tile loop: the far pass
// needs only the tile-relative q', and registers bound occupancy.
template <int QT>
struct QState {
    static constexpr int kPairs = QT / 2;
    f2 c[kPairs], b[kPairs], s[kPairs];
    bool g2[QT];  // class G2 (FMA-pipe exp2), per query
    bool v[QT];   // query slot holds a real query
};

// Query coordinates {x_hi, y_hi, x_lo, y_lo} of a pair of slots (volatile:
// each pass re-reads instead of keeping them live).
struct QCoords {
    f2 xh, yh, xl, yl;
};
__device__ __forceinline__ float4 ld_q(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
template <int QT>
__device__ __forceinline__ void load_coords(const float4* qhl, size_t wbase, int lane, size_t q1,
                                            QCoords (&qc)[QT / 2]) {
#pragma unroll
    for (int k = 0; k < QT / 2; ++k) {
        const size_t p0 = wbase + static_cast<size_t>(2 * k) * 32 + lane;
        const size_t p1 = p0 + 32;
        const float4 h0 = p0 < q1 ? ld_q(qhl + p0) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 h1 = p1 < q1 ? ld_q(qhl + p1) : make_float4(0.f, 0.f, 0.f, 0.f);
        qc[k].xh = pk2(h0.x, h1.x);
        qc[k].yh = pk2(h0.y, h1.y);
        qc[k].xl = pk2(h0.z, h1.z);
        qc[k].yl = pk2(h0.w, h1.w);
    }
}

// Weight formula modes (warp-uniform; per query the arithmetic is the same
// in every mode that can hold it, so grouping never changes a result):
//   3  recipe, s == 1 for the whole warp      w' = rcp(d2^2)
//   0  recipe, some s != 1                    w' = rcp((d2 s)^2)
//   1  general, all G1                        w' = ex2(c lg2(d2) + b)  (2 MUFU)
//   4  general, all G2                        ex2 on the FMA pipe      (1 MUFU)
//   5  general, pair 0 G1 / pair 1 G2 (the interleaved layout)
//   2  general, G1 and G2 mixed otherwise (per query, scalar)
//   9, 10  recipe alpha = 1 / alpha = 3 (one MUFU.RSQ per pair)
template <int MODE, int QT>
__device__ __forceinline__ f2 general_w(f2 d2, const QState<QT>& q, int r) {
    if (MODE == 9) return rsq2(d2);           // recipe alpha = 1
    if (MODE == 10) return cube2(rsq2(d2));   // recipe alpha = 3
    float lo, hi;
    up2(d2, lo, hi);
    if (MODE == 2) {
        const bool g0 = q.g2[2 * r], g1 = q.g2[2 * r + 1];
        float c0, c1, b0, b1;
        up2(q.c[r], c0, c1);
        up2(q.b[r], b0, b1);
        const float e0 = fmaf(c0, mufu_lg2(lo), b0), e1 = fmaf(c1, mufu_lg2(hi), b1);
        return pk2(g0 ? exp2_fma(e0) : mufu_ex2(e0), g1 ? exp2_fma(e1) : mufu_ex2(e1));
    }
    const f2 e = fma2(q.c[r], pk2(mufu_lg2(lo), mufu_lg2(hi)), q.b[r]);
    if (MODE == 4 || (MODE == 5 && r % 2 == 1)) return exp2_fma2(e);
    up2(e, lo, hi);
    return pk2(mufu_ex2(lo), mufu_ex2(hi));
}

// FAR tile: d2 = fma(py2, q'y, fma(px2, q'x, |q'|^2)) + pp, 3 FP32 ops per
// pair; sums plain (far pairs carry a small weight share or average out).
// Recipe modes pair points 4j and 4j+1 on one reciprocal,
//   w0 + w1 = (a0 + a1) rcp(a0 a1),  w0 z0 + w1 z1 = (a1 z0 + a0 z1) rcp(a0 a1),
// a = d2^2 (far d2 >= 1e-8: no range scaling) — 6.5 FP32 ops + 0.75 MUFU per
// pair, balancing the FMA pipe
// (128 lanes / clk / SM) against MUFU (16 / clk / SM).
template <int MODE, int QT>
__device__ __forceinline__ void k4_far(const float* __restrict__ t, const QState<QT>& q,
                                       const f2 (&fx)[QT / 2], const f2 (&fy)[QT / 2],
                                       const f2 (&fq)[QT / 2], f2 (&sw)[QT / 2],
                                       f2 (&swz)[QT / 2]) {
    constexpr int kPairs = QT / 2;
#pragma unroll 1
    for (int j0 = 0; j0 < kWeightTile; j0 += 4 * kFarUnroll) {
#pragma unroll
    for (int h = 0; h < kFarUnroll; ++h) {
        const int j = j0 + 4 * h;
        // points 2, 3 of the group paired too (AIDW_K4_MIXPAIRS: every other group)
        const bool pair23 = AIDW_K4_ALLPAIRS || (AIDW_K4_MIXPAIRS && h == 0);
        const float4 X = *reinterpret_cast<const float4*>(t + kPX * kWeightTile + j);
        const float4 Y = *reinterpret_cast<const float4*>(t + kPY * kWeightTile + j);
        const float4 P = *reinterpret_cast<const float4*>(t + kPP * kWeightTile + j);
        const float4 Z = *reinterpret_cast<const float4*>(t + kZH * kWeightTile + j);
#pragma unroll
        for (int r = 0; r < kPairs; ++r) {
            const f2 d0 = add2(fma2(bc2(Y.x), fy[r], fma2(bc2(X.x), fx[r], fq[r])), bc2(P.x));
            const f2 d1 = add2(fma2(bc2(Y.y), fy[r], fma2(bc2(X.y), fx[r], fq[r])), bc2(P.y));
            const f2 d2 = add2(fma2(bc2(Y.z), fy[r], fma2(bc2(X.z), fx[r], fq[r])), bc2(P.z));
            const f2 d3 = add2(fma2(bc2(Y.w), fy[r], fma2(bc2(X.w), fx[r], fq[r])), bc2(P.w));
            if (MODE == 3 || MODE == 7) {
                // a = d2^2 (alpha 4), d2 (alpha 2)
                const f2 a0 = MODE == 3 ? mul2(d0, d0) : d0;
                const f2 a1 = MODE == 3 ? mul2(d1, d1) : d1;
                const f2 a2 = MODE == 3 ? mul2(d2, d2) : d2;
                const f2 a3 = MODE == 3 ? mul2(d3, d3) : d3;
                const f2 r01 = rcp2(mul2(a0, a1));
                sw[r] = fma2(r01, add2(a0, a1), sw[r]);
                swz[r] = fma2(r01, fma2(a1, bc2(Z.x), mul2(a0, bc2(Z.y))), swz[r]);
                if (pair23) {
                    const f2 r23 = rcp2(mul2(a2, a3));
                    sw[r] = fma2(r23, add2(a2, a3), sw[r]);
                    swz[r] = fma2(r23, fma2(a3, bc2(Z.z), mul2(a2, bc2(Z.w))), swz[r]);
                } else {
                    const f2 w2 = rcp2(a2);
                    sw[r] = add2(sw[r], w2);
                    swz[r] = fma2(w2, bc2(Z.z), swz[r]);
                    const f2 w3 = rcp2(a3);
                    sw[r] = add2(sw[r], w3);
                    swz[r] = fma2(w3, bc2(Z.w), swz[r]);
                }
            } else if (MODE == 8) {
                // mixed recipe warp: both the paired (alpha 4 / 2) and the
                // rsqrt (alpha 1 / 3) forms, picked per slot
                const f2 code = q.c[r];
                const f2 a0 = recipe_a(d0, code), a1 = recipe_a(d1, code);
                const f2 a2 = recipe_a(d2, code), a3 = recipe_a(d3, code);
                const f2 v0 = recipe_rsq(d0, code), v1 = recipe_rsq(d1, code);
                const f2 v2 = recipe_rsq(d2, code), v3 = recipe_rsq(d3, code);
                const f2 r01 = rcp2(mul2(a0, a1));
                sw[r] = sel_paired(code, fma2(r01, add2(a0, a1), sw[r]),
                                   add2(add2(sw[r], v0), v1));
                swz[r] = sel_paired(code,
                                    fma2(r01, fma2(a1, bc2(Z.x), mul2(a0, bc2(Z.y))), swz[r]),
                                    fma2(v1, bc2(Z.y), fma2(v0, bc2(Z.x), swz[r])));
                if (pair23) {
                    const f2 r23 = rcp2(mul2(a2, a3));
                    sw[r] = sel_paired(code, fma2(r23, add2(a2, a3), sw[r]),
                                       add2(add2(sw[r], v2), v3));
                    swz[r] = sel_paired(code,
                                        fma2(r23, fma2(a3, bc2(Z.z), mul2(a2, bc2(Z.w))), swz[r]),
                                        fma2(v3, bc2(Z.w), fma2(v2, bc2(Z.z), swz[r])));
                } else {
                    const f2 w2 = sel_paired(code, rcp2(a2), v2);
                    sw[r] = add2(sw[r], w2);
                    swz[r] = fma2(w2, bc2(Z.z), swz[r]);
                    const f2 w3 = sel_paired(code, rcp2(a3), v3);
                    sw[r] = add2(sw[r], w3);
                    swz[r] = fma2(w3, bc2(Z.w), swz[r]);
                }
            } else {
                const f2 w0 = general_w<MODE, QT>(d0, q, r);
                sw[r] = add2(sw[r], w0);
                swz[r] = fma2(w0, bc2(Z.x), swz[r]);
                const f2 w1 = general_w<MODE, QT>(d1, q, r);
                sw[r] = add2(sw[r], w1);
                swz[r] = fma2(w1, bc2(Z.y), swz[r]);
                const f2 w2 = general_w<MODE, QT>(d2, q, r);
                sw[r] = add2(sw[r], w2);
                swz[r] = fma2(w2, bc2(Z.z), swz[r]);
                const f2 w3 = general_w<MODE, QT>(d3, q, r);
                sw[r] = add2(sw[r], w3);
                swz[r] = fma2(w3, bc2(Z.w), swz[r]);
            }
        }
    }
    }
}

// NEAR tile (the query lies within the near threshold of the tile's box, or
// the tile is padded): hi/lo differences dx = (x_hi - q_hi) + (x_lo - q_lo)
// (~48 bits), one reciprocal / exponential per pair, and sum w z
// Kahan-compensated with hi/lo z — a query's dominant terms live here.
template <int MODE, int QT>
__device__ __forceinline__ void k4_near_point(float pxh, float pyh, float pxl, float pyl,
                                              float pzh, float pzl, const QState<QT>& q,
                                              const QCoords (&qc)[QT / 2], f2 (&sw)[QT / 2],
                                              f2 (&swz)[QT / 2], f2 (&cz)[QT / 2],
                                              f2 (&cw)[QT / 2]) {
    constexpr int kPairs = QT / 2;
#pragma unroll
    for (int r = 0; r < kPairs; ++r) {
        const f2 dx = add2(sub2(bc2(pxh), qc[r].xh), sub2(bc2(pxl), qc[r].xl));
        const f2 dy = add2(sub2(bc2(pyh), qc[r].yh), sub2(bc2(pyl), qc[r].yl));
        f2 d2 = fma2(dx, dx, mul2(dy, dy));
        f2 w;
        if (MODE == 3 || MODE == 0) {
            if (MODE == 0) d2 = mul2(d2, q.s[r]);
            w = rcp2(mul2(d2, d2));
        } else if (MODE == 7) {  // alpha == 2: s == 1
            w = rcp2(d2);
        } else if (MODE == 8) {  // mixed recipe: t = d2 s (s == 1 unless alpha 4), per slot
            d2 = mul2(d2, q.s[r]);
            w = sel_paired(q.c[r], rcp2(recipe_a(d2, q.c[r])), recipe_rsq(d2, q.c[r]));
        } else {
            w = general_w<MODE, QT>(d2, q, r);
        }
        {
            const f2 yw = sub2(w, cw[r]);
            const f2 s1 = add2(sw[r], yw);
            cw[r] = sub2(sub2(s1, sw[r]), yw);
            sw[r] = s1;
        }
        const f2 tz = fma2(w, bc2(pzh), mul2(w, bc2(pzl)));
        const f2 y = sub2(tz, cz[r]);
        const f2 s2 = add2(swz[r], y);
        cz[r] = sub2(sub2(s2, swz[r]), y);
        swz[r] = s2;
    }
}

template <int MODE, int QT>
__device__ __forceinline__ void k4_near(const float* __restrict__ t, const QState<QT>& q,
                                        const QCoords (&qc)[QT / 2], f2 (&sw)[QT / 2],
                                        f2 (&swz)[QT / 2], f2 (&cz)[QT / 2],
                                        f2 (&cw)[QT / 2]) {
#pragma unroll 1
    for (int j = 0; j < kWeightTile; j += 4) {
        const float4 X = *reinterpret_cast<const float4*>(t + kXH * kWeightTile + j);
        const float4 Y = *reinterpret_cast<const float4*>(t + kYH * kWeightTile + j);
        const float4 XL = *reinterpret_cast<const float4*>(t + kXL * kWeightTile + j);
        const float4 YL = *reinterpret_cast<const float4*>(t + kYL * kWeightTile + j);
        const float4 Z = *reinterpret_cast<const float4*>(t + kZH * kWeightTile + j);
        const float4 ZL = *reinterpret_cast<const float4*>(t + kZL * kWeightTile + j);
        k4_near_point<MODE, QT>(X.x, Y.x, XL.x, YL.x, Z.x, ZL.x, q, qc, sw, swz, cz, cw);
        k4_near_point<MODE, QT>(X.y, Y.y, XL.y, YL.y, Z.y, ZL.y, q, qc, sw, swz, cz, cw);
        k4_near_point<MODE, QT>(X.z, Y.z, XL.z, YL.z, Z.z, ZL.z, q, qc, sw, swz, cz, cw);
        k4_near_point<MODE, QT>(X.w, Y.w, XL.w, YL.w, Z.w, ZL.w, q, qc, sw, swz, cz, cw);
    }
}

// One tile against the thread's queries: far part (queries FAR from the
// tile) and near part (queries NEAR), each over the whole tile with its own
// accumulators, only when some query of the warp needs it; each query folds
// the part its own (query, tile) classification selects into FP64.
template <int MODE, int QT>
__device__ __forceinline__ void k4_tile(const float* __restrict__ t, const QState<QT>& q,
                                        const float4* qhl, size_t wbase, int lane, size_t q1,
                                        const bool (&nq)[QT], bool any_far, bool any_near,
                                        float cx, float cy, double (&SW)[QT], double (&SWZ)[QT]) {
    constexpr int kPairs = QT / 2;
    if (any_far) {
        f2 fx[kPairs], fy[kPairs], fq[kPairs], sw[kPairs], swz[kPairs];
        {
            QCoords qc[kPairs];
            load_coords<QT>(qhl, wbase, lane, q1, qc);
#pragma unroll
            for (int r = 0; r < kPairs; ++r) {
                fx[r] = add2(sub2(qc[r].xh, bc2(cx)), qc[r].xl);
                fy[r] = add2(sub2(qc[r].yh, bc2(cy)), qc[r].yl);
                fq[r] = fma2(fx[r], fx[r], mul2(fy[r], fy[r]));
                sw[r] = swz[r] = 0ull;
            }
        }
        // far pairs never need the recipe's range scaling (d2 >= the near
        // threshold >= 1e-8): mode 0 runs the s-free form and rescales the
        // tile sums by s^-2 (a power of two: exact)
        k4_far<MODE == 0 ? 3 : MODE, QT>(t, q, fx, fy, fq, sw, swz);  // 7, 8: s-free too
#pragma unroll
        for (int r = 0; r < kPairs; ++r) {
            float w0, w1, z0, z1;
            up2(sw[r], w0, w1);
            up2(swz[r], z0, z1);
            double m0 = 1.0, m1 = 1.0;
            if (MODE == 0 || MODE == 8) {  // (alpha == 2 queries have s == 1)
                float s0, s1;
                up2(q.s[r], s0, s1);
                m0 = 1.0 / (static_cast<double>(s0) * s0);
                m1 = 1.0 / (static_cast<double>(s1) * s1);
            }
            if (!nq[2 * r]) SW[2 * r] += w0 * m0, SWZ[2 * r] += z0 * m0;
            if (!nq[2 * r + 1]) SW[2 * r + 1] += w1 * m1, SWZ[2 * r + 1] += z1 * m1;
        }
    }
    if (any_near) {
        QCoords qc[kPairs];
        load_coords<QT>(qhl, wbase, lane, q1, qc);
        f2 sw[kPairs], swz[kPairs], cz[kPairs], cw[kPairs];
#pragma unroll
        for (int r = 0; r < kPairs; ++r) sw[r] = swz[r] = cz[r] = cw[r] = 0ull;
        k4_near<MODE, QT>(t, q, qc, sw, swz, cz, cw);
#pragma unroll
        for (int r = 0; r < kPairs; ++r) {
            float w0, w1, z0, z1, c0, c1;
            up2(sw[r], w0, w1);
            up2(swz[r], z0, z1);
            up2(cz[r], c0, c1);
            float e0, e1;
            up2(cw[r], e0, e1);
            if (nq[2 * r])
                SW[2 * r] += static_cast<double>(w0) - static_cast<double>(e0),
                    SWZ[2 * r] += static_cast<double>(z0) - static_cast<double>(c0);
            if (nq[2 * r + 1])
                SW[2 * r + 1] += static_cast<double>(w1) - static_cast<double>(e1),
                    SWZ[2 * r + 1] += static_cast<double>(z1) - static_cast<double>(c1);
        }
    }
}

// The CTA body for one query class.  RECIPE: alpha == 4 queries (modes 3 /
// 0); else the general queries (modes 1 / 4 / 5 / 2).  Each CTA streams the
// tiles of one data chunk through a kStages-deep shared-memory ring filled
// by the bulk-copy engine (cp.async.bulk + mbarrier complete_tx; SASS
// UBLKCP), one elected thread producing, all warps consuming broadcast
// LDS.128 reads of one component of 4 consecutive points.
template <bool RECIPE, int kQT>
__device__ __forceinline__ void k4_body(const K4Args& a, size_t q0, size_t q1, size_t cta,
                                        float* stile, uint64_t* bar, unsigned* done) {
    constexpr int kPairs = kQT / 2;
    const unsigned chunk = blockIdx.y;
    const size_t t0 = static_cast<size_t>(chunk) * a.tiles_per_chunk;
    const size_t t1 = t0 + a.tiles_per_chunk < a.tiles ? t0 + a.tiles_per_chunk : a.tiles;
    const size_t ntl = t1 > t0 ? t1 - t0 : 0;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t wbase = q0 + cta * (kK4Threads * kQT) + static_cast<size_t>(warp) * (32 * kQT);
    QState<kQT> q;
    bool any_g1 = false, any_g2 = false, any_scaled = false;
    unsigned rcodes = 0;  // recipe class codes present (bit per code)
    {
        float4 r[kQT];
#pragma unroll
        for (int i = 0; i < kQT; ++i) {
            const size_t p = wbase + static_cast<size_t>(i) * 32 + lane;
            r[i] = make_float4(-1.f, 0.f, 1.f, RECIPE ? 1.f : 0.f);
            q.v[i] = p < q1;
            if (q.v[i]) r[i] = a.qpar[p];
            q.g2[i] = r[i].w == 2.0f;
            if (RECIPE && q.v[i]) rcodes |= 1u << static_cast<int>(r[i].w);
            any_g2 |= q.v[i] && q.g2[i];
            any_g1 |= q.v[i] && !q.g2[i];
            any_scaled |= q.v[i] && r[i].z != 1.0f;
        }
#pragma unroll
        for (int k = 0; k < kPairs; ++k) {
            const int i0 = 2 * k, i1 = 2 * k + 1;
            q.c[k] = pk2(r[i0].x, r[i1].x);
            q.b[k] = pk2(r[i0].y, r[i1].y);
            q.s[k] = pk2(r[i0].z, r[i1].z);
        }
    }
    any_g1 = __any_sync(0xFFFFFFFFu, any_g1);
    any_g2 = __any_sync(0xFFFFFFFFu, any_g2);
    any_scaled = __any_sync(0xFFFFFFFFu, any_scaled);
    rcodes = __reduce_or_sync(0xFFFFFFFFu, rcodes);
    int mode;
    if (RECIPE) {
        // one class in the warp: its pure mode; several: the per-slot form
        mode = rcodes == (1u << 3)  ? 7
             : rcodes == (1u << 4)  ? 9
             : rcodes == (1u << 5)  ? 10
             : rcodes == (1u << 1) || rcodes == 0 ? (any_scaled ? 0 : 3)
                                    : 8;
#ifdef AIDW_K4_FORCE_MIXED
        mode = 8;
#endif
    } else {
        // the interleaved layout: pair 0 all G1 and pair 1 all G2 across the warp
        bool split = kQT == 4;
#pragma unroll
        for (int i = 0; i < kQT; ++i) split &= !q.v[i] || (q.g2[i] == (i >= kQT / 2));
        split = __all_sync(0xFFFFFFFFu, split) && any_g1 && any_g2;
        mode = split ? 5 : (any_g1 && any_g2) ? 2 : any_g2 ? 4 : 1;
    }

    double SW[kQT], SWZ[kQT];
#pragma unroll
    for (int i = 0; i < kQT; ++i) SW[i] = SWZ[i] = 0.0;

    constexpr uint32_t kTileBytes = kTileFloats * sizeof(float);
    if (threadIdx.x == 0) {
        for (size_t s = 0; s < ntl && s < static_cast<size_t>(kStages); ++s) {
            mbar_expect_tx(&bar[s], kTileBytes);
            bulk_load(stile + s * kTileFloats, a.rec + (t0 + s) * kTileFloats, kTileBytes, &bar[s]);
        }
    }
    for (size_t it = 0; it < ntl; ++it) {
        const int st = static_cast<int>(it % kStages);
        mbar_wait(&bar[st], static_cast<uint32_t>((it / kStages) & 1));
        const float* tt = stile + st * kTileFloats;
        // per-(query, tile) near flags, then a warp-uniform dispatch
        const float4 tb = __ldg(a.tile_box + t0 + it);
        const float4 tg = __ldg(a.tile_geo + t0 + it);
        bool nq[kQT];
        bool any_near = false, any_far = false;
#pragma unroll
        for (int i = 0; i < kQT; ++i) {
            const size_t p = wbase + static_cast<size_t>(i) * 32 + lane;
            const float2 xy = q.v[i] ? __ldg(reinterpret_cast<const float2*>(a.qhl + p))
                                     : make_float2(0.f, 0.f);
            const float ex = fmaxf(0.0f, fmaxf(tb.x - xy.x, xy.x - tb.z));
            const float ey = fmaxf(0.0f, fmaxf(tb.y - xy.y, xy.y - tb.w));
            nq[i] = fmaf(ex, ex, ey * ey) <= tg.z;
            if (q.v[i]) {  // empty slots never force a pass
                any_near |= nq[i];
                any_far |= !nq[i];
            }
        }
        any_near = __any_sync(0xFFFFFFFFu, any_near);
        any_far = __any_sync(0xFFFFFFFFu, any_far);
        if (RECIPE) {
            if (mode == 3) k4_tile<3, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else if (mode == 7) k4_tile<7, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else if (mode == 8) k4_tile<8, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else if (mode == 9) k4_tile<9, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else if (mode == 10) k4_tile<10, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else k4_tile<0, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
        } else {
            if (mode == 5) k4_tile<5, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else if (mode == 1) k4_tile<1, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else if (mode == 4) k4_tile<4, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
            else k4_tile<2, kQT>(tt, q, a.qhl, wbase, lane, q1, nq, any_far, any_near, tg.x, tg.y, SW, SWZ);
        }
        // release the stage: the last warp done with it refills it, so warps
        // drift up to kStages tiles apart instead of meeting at a CTA barrier
        // (a warp with near work on a tile catches up on the far tiles after)
        __syncwarp();
        if (lane == 0 && it + kStages < ntl) {
            __threadfence_block();
            // counts never reset: the last arrival of round k sees 8k + 7
            if ((atomicAdd(&done[st], 1u) + 1u) % (kK4Threads / 32) == 0u) {
                __threadfence_block();
                fence_proxy_async();
                const size_t tile = t0 + it + kStages;
                mbar_expect_tx(&bar[st], kTileBytes);
                bulk_load(stile + st * kTileFloats, a.rec + tile * kTileFloats, kTileBytes,
                          &bar[st]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < kQT; ++i) {
        const size_t p = wbase + static_cast<size_t>(i) * 32 + lane;
        if (p < q1)
            a.part[static_cast<size_t>(chunk) * (a.s1 - a.s0) + (p - a.s0)] = make_double2(SW[i], SWZ[i]);
    }
}

// One launch for both classes of a query slab [s0, s1): CTAs
// [0, ceil(|G| / Q)) take G = [s0, s1) ∩ [0, nG), the general region of the
// visiting order, the rest R = [s0, s1) ∩ [nG, n), the recipe region
// (Q = queries per CTA; s0 is a multiple of Q, so G keeps the warp-aligned
// G1 / G2 interleave).  The class counts live on the device (no host sync
// mid-pipeline); the grid is sized for ceil((s1 - s0) / Q) + 1 CTAs, any
// surplus CTA exits at once.
template <int kQT, int kMinBlocks>
__global__ void __launch_bounds__(kK4Threads, kMinBlocks) weight_fp32_kernel(K4Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* stile = reinterpret_cast<float*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(stile + kStages * kTileFloats);
    unsigned* done = reinterpret_cast<unsigned*>(bar + kStages);
    constexpr size_t kQ = static_cast<size_t>(kK4Threads) * kQT;
    const size_t num_a = static_cast<size_t>(a.scan_a[a.n - 1]) + a.flag_a[a.n - 1];
    const size_t num_g = a.n - num_a;
    const size_t g0 = a.s0, g1 = a.s1 < num_g ? a.s1 : num_g;
    const size_t r0 = a.s0 > num_g ? a.s0 : num_g, r1 = a.s1;
    const size_t ctas_g = g1 > g0 ? (g1 - g0 + kQ - 1) / kQ : 0;
    const size_t b = blockIdx.x;
    if (b >= ctas_g && (r1 <= r0 || (b - ctas_g) * kQ >= r1 - r0)) return;
    if (!(a.classes & (b < ctas_g ? 1u : 2u))) return;  // that region runs on the other engine
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bar[s], 1);
            done[s] = 0u;
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (b < ctas_g) k4_body<false, kQT>(a, g0, g1, b, stile, bar, done);
    else k4_body<true, kQT>(a, r0, r1, b - ctas_g, stile, bar, done);
}

// ------------------------------------------------------------ settle
__global__ void settle_kernel(const WeightQueries q, WeightFrame f, const WeightData d,
                              const uint32_t* __restrict__ order,
                              const double2* __restrict__ part,
                              const double* __restrict__ lshift, unsigned chunks,
                              size_t s0, size_t s1, double* __restrict__ pred,
                              double* __restrict__ alpha_out) {
    const size_t i = s0 + static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s1) return;
    const uint32_t p = order[i];
    const uint32_t qi = q.perm ? q.perm[p] : p;
    const double alpha = q.alpha_s[p];
    double out;
    const uint32_t snap = q.snap_s[p];
    if (snap != kNoId) {
        out = d.z[snap];
    } else {
        double sw = 0.0, swz = 0.0;
        const double2* pp = part + (i - s0);
        const size_t ld = s1 - s0;
        unsigned c = 0;
        // eight independent loads in flight, added in chunk order (the
        // summation order of the one-at-a-time loop)
        for (; c + 8 <= chunks; c += 8) {
            double2 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = pp[static_cast<size_t>(c + k) * ld];
#pragma unroll
            for (int k = 0; k < 8; ++k) sw += v[k].x, swz += v[k].y;
        }
        for (; c < chunks; ++c) {
            const double2 v = pp[static_cast<size_t>(c) * ld];
            sw += v.x;
            swz += v.y;
        }
        const int zshift = frame_zshift(f.zhull);
        const double zlo = f.zhull[0], zhi = f.zhull[1];
        // The FP64 reference overflows / underflows where the true (unscaled)
        // weights do (interpolate.hpp:109-118): its largest weight is
        // 2^e, e = -alpha/2 log2 d2_min; its sums are 2^lshift * (sw, swz / 2^zshift).
        const double e = -0.5 * alpha * log2(q.d2min_s[p]);
        const double sh = lshift[i];
        bool fallback = !(sw > 0.0) || !isfinite(sw) || !isfinite(swz) || !(e < 1024.0) ||
                        !(sh + log2(sw) < 1024.0) || e < -1075.0;
        if (!fallback && swz != 0.0 && !(sh + log2(fabs(swz)) - zshift < 1024.0)) fallback = true;
        if (fallback) {
            out = d.z[q.nn_s[p]];
        } else {
            double v = ldexp(swz / sw, -zshift);
            out = v < zlo ? zlo : (v > zhi ? zhi : v);
        }
    }
    pred[qi] = out;
    if (alpha_out) alpha_out[qi] = alpha;
}

}  // namespace

void set_alpha4_recipe(bool enabled) { g_alpha4_recipe.store(enabled); }
bool alpha4_recipe_enabled() { return g_alpha4_recipe.load(); }

namespace {
std::atomic<size_t> g_query_slab{0};
}

void set_query_slab(size_t queries) { g_query_slab.store(queries); }

size_t query_slab(unsigned chunks) {
    // default: 2 GiB of FP64 partials (4M queries at 32 data chunks, 2M at
    // 64); a multiple of 1024 so every slab starts on a K4 CTA boundary
    size_t v = g_query_slab.load();
    if (v == 0) v = (size_t(2) << 30) / (16 * static_cast<size_t>(chunks ? chunks : 1));
    v = std::max<size_t>(1024, v & ~size_t(1023));
    return v;
}

WeightSplit weight_split(size_t m) {
    // Data chunks per query (the grid's y dimension): enough CTAs to fill
    // 148 SMs at small n without a partial last wave dominating — up to 64
    // chunks (one tile each for m <= 16K: 10K x 10K 0.23 -> 0.10 ms) while
    // m <= 256K, 32 chunks beyond (partials
    // 512 B per query; 32 vs 16: -0.6 % K4 time at 1M x 1M).  A function of m only, so a query's summation order
    // never depends on n, the shard or the GPU count.
    WeightSplit w;
    w.tiles = (m + kWeightTile - 1) / kWeightTile;
    if (w.tiles == 0) w.tiles = 1;
    const size_t cap = w.tiles <= 1024 ? 64 : static_cast<size_t>(kMaxChunks);
    static const size_t min_tiles = [] {  // AIDW_K4_CHUNK_TILES: tuning only
        const char* v = std::getenv("AIDW_K4_CHUNK_TILES");
        return static_cast<size_t>(v ? std::max(1, std::atoi(v)) : 1);
    }();
    size_t chunks = std::min(cap, std::max<size_t>(1, w.tiles / min_tiles));
    static const size_t big_chunks = [] {  // AIDW_K4_MAX_CHUNKS: tuning only
        const char* v = std::getenv("AIDW_K4_MAX_CHUNKS");
        return static_cast<size_t>(v ? std::max(1, std::atoi(v)) : kMaxChunks);
    }();
    if (w.tiles > 1024) chunks = std::min(w.tiles, big_chunks);
    w.tiles_per_chunk = (w.tiles + chunks - 1) / chunks;
    w.chunks = static_cast<unsigned>((w.tiles + w.tiles_per_chunk - 1) / w.tiles_per_chunk);
    return w;
}

bool weight_tc_selected(const WeightSplit& sp) {
    static const int forced = [] {  // AIDW_K4_ENGINE: tuning / A-B only
        const char* v = std::getenv("AIDW_K4_ENGINE");
        if (!v) return -1;
        return std::string(v) == "tc" ? 1 : std::string(v) == "simt" ? 0 : -1;
    }();
    if (forced >= 0) return forced == 1;
    // enough tiles per CTA to amortise its TMEM / pipeline setup
    return sp.tiles_per_chunk >= 4;
}

// A second stream (and fork / join events) per host thread and device for
// the general-alpha K4 launch that runs beside the tensor-core launch.
struct SideStream {
    int device = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream* side_stream() {
    static thread_local SideStream cache[16];
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 16) return nullptr;
    SideStream& c = cache[dev];
    if (!c.s) {
        CK(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming));
        c.device = dev;
    }
    return &c;
}

bool weight_tc_general() {  // AIDW_TC_GENERAL=1: general-alpha queries on the TC engine too (A/B)
    static const bool v = [] {
        const char* e = std::getenv("AIDW_TC_GENERAL");
        return e && std::atoi(e) != 0;
    }();
    return v;
}

void weighting_fp32(const WeightQueries& q, const WeightData& d, const WeightFrame& f,
                    double* d_pred, double* d_alpha, WeightTimes* times, cudaStream_t s) {
    if (q.n == 0) return;
    const WeightSplit sp = weight_split(d.m);
    const size_t mp = sp.tiles * kWeightTile;
    // record order: the grid's cells in 8 x 8-cell blocks (compact tiles)
    DBuf<uint32_t> border;
    const uint32_t* order = d.order;
    if (d.order && d.cell_start) {
        border.alloc(d.m, s);
        blocked_cell_order(d.cell_start, d.order, d.n_col, d.n_row, d.m, border.get(), s);
        order = border.get();
    }
    DBuf<float> rec(sp.tiles * kTileFloats, s);
    DBuf<float4> tbox(sp.tiles, s), tgeo(sp.tiles, s);
    LAUNCH(prep_data_kernel, ceil_div(mp, kThreads), kThreads, 0, s, d.x, d.y, d.z, order, d.m,
           mp, f.ox, f.oy, f.inv_scale, f.zhull, rec.get());
    // near threshold R_far (unit-box units): closer (query, tile) pairs take
    // the hi/lo form (AIDW_K4_RFAR to tune)
    static const float rfar = [] {
        const char* v = std::getenv("AIDW_K4_RFAR");
        return v ? static_cast<float>(std::atof(v)) : 0.01f;
    }();
    // far form needs box distance >= diagf * tile diagonal (AIDW_K4_DIAGF)
    static const float diagf = [] {
        const char* v = std::getenv("AIDW_K4_DIAGF");
        return v ? static_cast<float>(std::atof(v)) : 0.3f;
    }();
    LAUNCH(tile_geo_kernel, sp.tiles, kWeightTile, 0, s, rec.get(), d.m, sp.tiles, rfar * rfar,
           diagf * diagf, tbox.get(), tgeo.get());
    border.release();
    const bool tc = weight_tc_selected(sp);
    DBuf<char> tcrec;
    if (tc) {
        tcrec.alloc(weight_tc_record_bytes(sp.tiles), s);
        weight_tc_records(rec.get(), tgeo.get(), sp.tiles, d.m, tcrec.get(), s);
    }

    // class flags, concatenated [A | alpha 2 | alpha 1 | alpha 3 | G2]: one scan
    DBuf<uint32_t> flags(5 * q.n, s), scans(5 * q.n, s), order_q(q.n, s);
    uint32_t *flag = flags.get(), *scan_a = scans.get();
    uint32_t *flag_g2 = flags.get() + 4 * q.n, *scan_g2 = scans.get() + 4 * q.n;
    RecipeFlags rf;
    for (int k = 0; k < kRecipeSubs; ++k) {
        rf.flag[k] = flags.get() + (1 + k) * q.n;
        rf.scan[k] = scans.get() + (1 + k) * q.n;
    }
    DBuf<float4> qhl(q.n, s), qpar(q.n, s);
    DBuf<double> lshift(q.n, s);
    DBuf<uint32_t> zkey(q.n, s), zpos(q.n, s);
    LAUNCH(morton_keys_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q, f, zkey.get(),
           zpos.get());
    if (q.n <= small_sort_n())  // (visiting order only: results never depend on it)
        bucket_by_key_small(zkey.get(), zpos.get(), q.n, 16, s);
    else
        radix_sort_pairs(zkey.get(), zpos.get(), q.n, 16, s);
    zkey.release();
    // share of general-alpha queries on the FMA-pipe exp2 (G2); the rest of
    // a G1 / G2 interleave runs as all-G2 warps (AIDW_K4_G2 to tune)
    static const unsigned g2_threshold = [] {
        const char* v = std::getenv("AIDW_K4_G2");
        const double share = v ? std::atof(v) : 0.5;
        return static_cast<unsigned>(std::fmin(share, 1.0) * 4294967295.0);
    }();
    LAUNCH(class_flags_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q, f,
           g_alpha4_recipe.load() ? 1 : 0, g2_threshold, zpos.get(), flag, rf,
           flag_g2);
    exclusive_scan_u32(flags.get(), scans.get(), 5 * q.n, s);
    LAUNCH(query_records_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q, f, zpos.get(),
           flag, scan_a, rf, flag_g2, scan_g2, order_q.get(), qhl.get(), qpar.get(),
           lshift.get(), times ? times->d_alpha4 : nullptr);

    // queries in slabs: the FP64 partials (16 B x chunks per query) are
    // bounded by the slab, not by n; per-query results never depend on it
    const size_t slab = std::min(q.n, query_slab(sp.chunks));
    DBuf<double2> part(slab * sp.chunks, s);
    K4Args ka{rec.get(), sp.tiles, sp.tiles_per_chunk, sp.chunks, qhl.get(), qpar.get(),
              q.n, flag, scan_a, 0, 0, part.get(), tbox.get(), tgeo.get(), 3u};
    const size_t smem = kStages * kTileFloats * sizeof(float) + kStages * sizeof(uint64_t) +
                        kStages * sizeof(unsigned);
    // K4 variant: queries per thread x min resident CTAs (AIDW_K4_VARIANT for
    // tuning; default 4 x 2: 124 registers, no spills — faster than 4 x 3 at
    // 80 registers).  Per-query arithmetic is identical in all.
    static const int variant = [] {
        const char* v = std::getenv("AIDW_K4_VARIANT");
        return v ? std::atoi(v) : 0;
    }();
    auto launch_on = [&](auto kernel, int qt, cudaStream_t st) {
        CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        dim3 grid(ceil_div(ka.s1 - ka.s0, static_cast<size_t>(kK4Threads) * qt) + 1, sp.chunks);
        LAUNCH(kernel, grid, kK4Threads, smem, st, ka);
    };
    auto launch = [&](auto kernel, int qt) { launch_on(kernel, qt, s); };
    // Few queries for the data size (n / 1024 x chunks CTAs short of ~16
    // waves of 148 x 2): 2 queries per thread, 4 CTAs / SM — twice the CTAs
    // (e.g. 20K queries x 20M points: 369 -> 215 ms).  The per-query
    // arithmetic is the same in every launch shape.
    const size_t ctas4 = ceil_div(slab, static_cast<size_t>(kK4Threads) * 4) * sp.chunks;
    const int shape = variant != 0 ? variant : (ctas4 < static_cast<size_t>(16 * 148 * 2) ? 2 : 0);
    // (with several slabs the K4 events also bracket the settles between
    // them: ~1e-4 of a K4 slab)
    if (times && times->k4_begin) record_event(times->k4_begin, s);
    for (size_t s0 = 0; s0 < q.n; s0 += slab) {
        ka.s0 = s0;
        ka.s1 = std::min(q.n, s0 + slab);
        if (tc) {
            // recipe queries on the tensor-core engine; general-alpha queries
            // (MUFU-bound exp2 / log2, no gain from a free d2) stay on the
            // CUDA-core kernel — the engine is a function of the query's
            // class and of m, never of n or the shard
            const bool gen_tc = weight_tc_general();
            SideStream* side = gen_tc ? nullptr : side_stream();
            if (side) {
                // the general region on a side stream, concurrent with the TC
                // launch (each fills the other's tail), joined before settle
                CK(cudaEventRecord(side->fork, s));  // (a capture dependency when capturing)
                CK(cudaStreamWaitEvent(side->s, side->fork, 0));
                ka.classes = 1u;
                switch (shape) {
                    case 2: launch_on(weight_fp32_kernel<2, 4>, 2, side->s); break;
                    default: launch_on(weight_fp32_kernel<4, AIDW_K4_MINB>, 4, side->s); break;
                }
                CK(cudaEventRecord(side->join, side->s));
            }
            WeightTcLaunch l;
            l.tc_rec = tcrec.get();
            l.tiles = sp.tiles, l.tiles_per_chunk = sp.tiles_per_chunk, l.chunks = sp.chunks;
            l.qhl = qhl.get(), l.qpar = qpar.get(), l.n = q.n;
            l.flag_a = flag, l.scan_a = scan_a;
            l.s0 = ka.s0, l.s1 = ka.s1, l.part = part.get();
            l.tile_box = tbox.get(), l.tile_geo = tgeo.get();
            l.classes = gen_tc ? 3u : 2u;
            weight_tc_launch(l, s);
            if (side) CK(cudaStreamWaitEvent(s, side->join, 0));
        } else switch (shape) {
            case 1: launch(weight_fp32_kernel<4, 3>, 4); break;
            case 2: launch(weight_fp32_kernel<2, 4>, 2); break;
            case 3: launch(weight_fp32_kernel<4, AIDW_K4_MINB>, 4); break;
            case 4: launch(weight_fp32_kernel<2, 3>, 2); break;
            default: launch(weight_fp32_kernel<4, AIDW_K4_MINB>, 4); break;
        }
        if (times && times->k4_end && ka.s1 == q.n) record_event(times->k4_end, s);
        LAUNCH(settle_kernel, ceil_div(ka.s1 - ka.s0, kThreads), kThreads, 0, s, q, f, d,
               order_q.get(), part.get(), lshift.get(), sp.chunks, ka.s0, ka.s1, d_pred, d_alpha);
    }
}

}  // namespace aidwb
