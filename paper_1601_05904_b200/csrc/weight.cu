// weight.cu — K4: the O(m·n) inverse-distance weighting on sm_100a (FP32).
//
// Replaces the weighting loops of aidw_predict_all / idw_predict_all
// (proj/include/aidw/interpolate.hpp:252-381, :426-489).  Design:
//
//  * Data records live in HBM as {x_hi, y_hi, x_lo, y_lo} float4 + z float,
//    coordinates normalised to the unit box in FP64 first and split into an
//    FP32 hi/lo pair, so dx = (x_hi - q_hi) + (x_lo - q_lo) keeps ~48 bits
//    without any FP64 op or F2F conversion per pair.  Padded to 256-point
//    tiles with records at 1e30 (weight exactly 0).
//  * Each CTA (256 threads, QT queries per thread in registers) streams the
//    tiles of one data chunk through a NSTAGE-deep shared-memory ring filled
//    by the bulk-copy engine (cp.async.bulk + mbarrier complete_tx; SASS
//    UBLKCP), one elected thread producing, all warps consuming broadcast
//    LDS.128 reads.
//  * Ratio scaling: w' = (d2 / d2_min)^(-alpha/2) <= 1, evaluated as
//    ex2(c * lg2(d2) + b) with c = -alpha/2, b = -c * lg2(d2_min) — two MUFU
//    ops (MUFU.LG2, MUFU.EX2) + 9 FP32 ops per pair.  Queries with
//    alpha == 4 exactly (98 % of uniform-data queries, the reference's
//    half-integer recipe, interpolate.hpp:174-209) use w' = rcp((d2*s)^2),
//    one MUFU.  Queries are partitioned so warps are class-uniform; the
//    formula is chosen per query, never per warp, so results do not depend
//    on the partition (or on the GPU count).
//  * Per-tile FP32 sums are folded into FP64 accumulators; data chunks
//    (S = f(m) only) give enough CTAs at small n and are summed in chunk
//    order by the settle kernel, deterministically (no atomics).
//  * settle: snap -> z[first index within snap distance]; analytic overflow
//    test in log space reproduces the FP64 reference's non-finite sums ->
//    nearest value (lowest index on ties); clamp to the value hull.

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "common.cuh"
#include "weight.cuh"

namespace aidwb {

namespace {

constexpr int kK4Threads = 256;
constexpr int kStages = 4;
constexpr int kMaxChunks = 16;
constexpr int kTileFloats = 6 * kWeightTile;  // SoA tile: xh yh xl yl zh zl

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

__device__ __forceinline__ float mufu_lg2(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float mufu_ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float mufu_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ------------------------------------------------------------ record prep
__device__ __forceinline__ void split_hilo(double v, float& hi, float& lo) {
    hi = __double2float_rn(v);
    lo = __double2float_rn(v - static_cast<double>(hi));
}

// Record i = data point order[i] (cell order of the factor-4 grid, so a
// 256-point tile is a compact strip of cells), or point i without order.
__global__ void prep_data_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ z, const uint32_t* __restrict__ order,
                                 size_t m, size_t mp, double ox, double oy, double inv_scale,
                                 double zmul, float* __restrict__ rec) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= mp) return;
    if (i < m) {
        const size_t j = order ? order[i] : i;
        float xh, xl, yh, yl;
        split_hilo((x[j] - ox) * inv_scale, xh, xl);
        split_hilo((y[j] - oy) * inv_scale, yh, yl);
        float* r = rec + (i / kWeightTile) * kTileFloats + (i % kWeightTile);
        float zh, zl;
        split_hilo(z[j] * zmul, zh, zl);
        r[0] = xh, r[kWeightTile] = yh, r[2 * kWeightTile] = xl, r[3 * kWeightTile] = yl;
        r[4 * kWeightTile] = zh, r[5 * kWeightTile] = zl;
    } else {
        float* r = rec + (i / kWeightTile) * kTileFloats + (i % kWeightTile);
        r[0] = 1.0e30f, r[kWeightTile] = 1.0e30f, r[2 * kWeightTile] = 0.0f;
        r[3 * kWeightTile] = 0.0f, r[4 * kWeightTile] = 0.0f, r[5 * kWeightTile] = 0.0f;
    }
}

// Bounding box (hi parts) of each 256-point tile's real records; one warp
// per tile.  Drives the per-(query, tile) near / far choice in K4.
__global__ void tile_box_kernel(const float* __restrict__ rec, size_t m, size_t tiles,
                                float4* __restrict__ box) {
    const size_t tile = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (tile >= tiles) return;
    float x0 = 3.0e38f, y0 = 3.0e38f, x1 = -3.0e38f, y1 = -3.0e38f;
    for (int j = lane; j < kWeightTile; j += 32) {
        const size_t i = tile * kWeightTile + j;
        if (i < m) {
            const float px = rec[tile * kTileFloats + j];
            const float py = rec[tile * kTileFloats + kWeightTile + j];
            x0 = fminf(x0, px), y0 = fminf(y0, py), x1 = fmaxf(x1, px), y1 = fmaxf(y1, py);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        x0 = fminf(x0, __shfl_xor_sync(0xFFFFFFFFu, x0, o));
        y0 = fminf(y0, __shfl_xor_sync(0xFFFFFFFFu, y0, o));
        x1 = fmaxf(x1, __shfl_xor_sync(0xFFFFFFFFu, x1, o));
        y1 = fmaxf(y1, __shfl_xor_sync(0xFFFFFFFFu, y1, o));
    }
    if (lane == 0) box[tile] = make_float4(x0, y0, x1, y1);
}

std::atomic<bool> g_alpha4_recipe{true};

// Query classes: A = the exact alpha == 4 recipe (or snapped: result
// replaced anyway); the other (general-alpha) queries split into G1 (exp2 on
// MUFU) and G2 (exp2 as a polynomial on the FMA pipe) by a hash of the
// query's own coordinates — a function of the query alone, so its formula
// (and result) never depends on sharding, order or GPU count.  Half / half
// balances the MUFU and FMA pipes.
__device__ __forceinline__ bool poly_class(double x, double y) {
    unsigned long long h = static_cast<unsigned long long>(__double_as_longlong(x)) *
                           0x9E3779B97F4A7C15ull;
    h ^= static_cast<unsigned long long>(__double_as_longlong(y)) * 0xC2B2AE3D27D4EB4Full;
    h ^= h >> 29;
    return (h >> 63) != 0;
}

__global__ void class_flags_kernel(const WeightQueries q, int recipe,
                                   uint32_t* __restrict__ flag_a, uint32_t* __restrict__ flag_g2) {
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= q.n) return;
    const bool a = (recipe && q.alpha_s[p] == 4.0) || q.snap_s[p] != kNoId;
    const uint32_t qi = q.perm ? q.perm[p] : static_cast<uint32_t>(p);
    flag_a[p] = a ? 1u : 0u;
    flag_g2[p] = (!a && poly_class(q.qx[qi], q.qy[qi])) ? 1u : 0u;
}

// 3-way partition (general G1/G2 interleaved, then A) fused with the
// per-query record build.
__global__ void query_records_kernel(const WeightQueries q, WeightFrame f,
                                     const uint32_t* __restrict__ flag_a,
                                     const uint32_t* __restrict__ scan_a,
                                     const uint32_t* __restrict__ flag_g2,
                                     const uint32_t* __restrict__ scan_g2,
                                     uint32_t* __restrict__ order, float4* __restrict__ qhl,
                                     float4* __restrict__ qpar, double* __restrict__ lshift,
                                     unsigned long long* __restrict__ alpha4) {
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= q.n) return;
    const size_t num_a = static_cast<size_t>(scan_a[q.n - 1]) + flag_a[q.n - 1];
    const size_t num_g2 = static_cast<size_t>(scan_g2[q.n - 1]) + flag_g2[q.n - 1];
    const size_t num_g1 = q.n - num_a - num_g2;
    const bool is_a = flag_a[p] != 0, is_g2 = flag_g2[p] != 0;
    // General queries: 64-query blocks of G1 and G2 alternate, so a warp's
    // pair 0 (slots 0, 1) is G1 and pair 1 (slots 2, 3) is G2 — each warp
    // issues MUFU and FMA-pipe exponentials side by side.  Leftovers follow.
    // The general region comes first so its 128-query blocks align with warps.
    size_t i;
    if (is_a) {
        i = num_g1 + num_g2 + scan_a[p];
    } else {
        const size_t j = is_g2 ? scan_g2[p] : p - scan_a[p] - scan_g2[p];
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
    // recipe path: w' = rcp((d2 s)^2).  s = 1 (no multiply needed, exact)
    // whenever d2 >= d2min >= 1e-15 keeps d2^2 and 1/d2^2 inside FP32;
    // otherwise s = 1/d2min.  Snapped queries: result replaced, s = 1.
    const bool snapped = q.snap_s[p] != kNoId;
    const float s = (snapped || d2n >= 1.0e-15) ? 1.0f : __double2float_rn(1.0 / d2n);
    qpar[i] = make_float4(c, b, s, is_a ? 1.0f : (is_g2 ? 2.0f : 0.0f));
    // log2(true weight) = log2(kernel weight) + shift (settle's overflow test)
    const double l2inv = log2(f.inv_scale);
    lshift[i] = is_a ? 2.0 * log2(static_cast<double>(s)) + 4.0 * l2inv
                     : -static_cast<double>(b) - 2.0 * static_cast<double>(c) * l2inv;
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
    double2* part;  // n * chunks
    const float4* tile_box;  // hi-coordinate box of every tile's real records
    float rfar2;             // squared near / far threshold (unit-box units)
};

// ---- packed f32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2): two queries per
// 64-bit register pair; each lane rounds exactly like the scalar op, so a
// query's result does not depend on which lane / pair it occupies.
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void up2(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// exp2 on the FMA pipe for class-G2 queries (x <= ~0 after ratio scaling):
// Cody-Waite split x = n + f, n = rint(x) via the 1.5 * 2^23 magic add,
// f in [-0.5, 0.5], 2^f by a degree-6 fit (max rel. error 9.7e-8 incl. FP32
// Horner rounding, vs ~1.2e-7 for MUFU.EX2), 2^n added into the exponent.
// Arguments clamp at -125 (results < 2^-125 are ~0 relative to the leading
// weight, which is 1).  Scalar and packed forms round identically.
constexpr float kExpMagic = 12582912.0f;  // 1.5 * 2^23
constexpr float kE0 = 1.0f, kE1 = 0.6931471824645996f, kE2 = 0.24022646248340607f,
                kE3 = 0.05550329014658928f, kE4 = 0.009618519805371761f,
                kE5 = 0.0013399859890341759f, kE6 = 0.00015337577497120947f;

__device__ __forceinline__ float exp2_fma(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + kExpMagic;
    const float f = x - (t - kExpMagic);
    float p = fmaf(kE6, f, kE5);
    p = fmaf(p, f, kE4);
    p = fmaf(p, f, kE3);
    p = fmaf(p, f, kE2);
    p = fmaf(p, f, kE1);
    p = fmaf(p, f, kE0);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ f2 exp2_fma2(f2 x) {
    float lo, hi;
    up2(x, lo, hi);
    const f2 xc = pk2(fmaxf(lo, -125.0f), fmaxf(hi, -125.0f));
    const f2 m = pk2(kExpMagic, kExpMagic);
    const f2 t = add2(xc, m);
    const f2 f = sub2(xc, sub2(t, m));
    f2 p = fma2(pk2(kE6, kE6), f, pk2(kE5, kE5));
    p = fma2(p, f, pk2(kE4, kE4));
    p = fma2(p, f, pk2(kE3, kE3));
    p = fma2(p, f, pk2(kE2, kE2));
    p = fma2(p, f, pk2(kE1, kE1));
    p = fma2(p, f, pk2(kE0, kE0));
    float plo, phi, tlo, thi;
    up2(p, plo, phi);
    up2(t, tlo, thi);
    return pk2(__int_as_float(__float_as_int(plo) + (__float_as_int(tlo) << 23)),
               __int_as_float(__float_as_int(phi) + (__float_as_int(thi) << 23)));
}

// Per-thread query state: QT queries as QT/2 f32x2 pairs.
template <int QT>
struct QState {
    static constexpr int kPairs = QT / 2;
    f2 xh[kPairs], yh[kPairs], xl[kPairs], yl[kPairs];
    f2 c[kPairs], b[kPairs], s[kPairs];
    bool a[QT];   // class A (alpha == 4 recipe), per query
    bool g2[QT];  // class G2 (FMA-pipe exp2), per query
    bool v[QT];  // query slot holds a real query
};

// One 256-point tile against the thread's QT queries.  Per data point and
// query pair:
//   NEAR tile (the query lies within R_far of the tile's box): hi/lo
//     differences, dx = (x_hi - q_hi) + (x_lo - q_lo): 3 FADD2 each for dx, dy
//   FAR tile: dx = x_hi - q_hi: 1 FADD2 each (relative error <= 6e-8 / R_far
//     on pairs that carry a small share of the weight)
//   d2 = dx dx + dy dy: FMUL2 + FFMA2, then
//   MODE 3 (alpha == 4 recipe, s == 1): FMUL2 (d2^2), 2 x MUFU.RCP
//   MODE 0 (alpha == 4 recipe, scaled): FMUL2 (d2 s), FMUL2 (^2), 2 x MUFU.RCP
//   MODE 1 (general, G1):       2 x MUFU.LG2, FFMA2 (c lg + b), 2 x MUFU.EX2
//   MODE 4 (general, G2):       2 x MUFU.LG2, FFMA2, exp2 on the FMA pipe
//   MODE 5 (G1 pair 0, G2 pair 1): both of the above in one instruction stream
//   MODE 2 (mixed class warp):  per query class and near flag, scalar, same roundings
// and FADD2 (sum w) + FFMA2 (sum w z) — Kahan-compensated with hi/lo z in
// NEAR tiles, where a query's large terms live.  DIST: 0 = every query of
// the warp far, 1 = every query near, 2 = mixed (both forms, per-lane
// select).  The formula is a function of the (query, tile) pair only, so a
// query's result never depends on its warp or lane.
__device__ __forceinline__ f2 sel2(f2 a, f2 b, bool take_a_lo, bool take_a_hi) {
    float alo, ahi, blo, bhi;
    up2(a, alo, ahi);
    up2(b, blo, bhi);
    return pk2(take_a_lo ? alo : blo, take_a_hi ? ahi : bhi);
}

// One data point (scalars from the SoA tile) against the thread's queries.
template <int MODE, int DIST, int QT>
__device__ __forceinline__ void k4_point(float pxh, float pyh, float pxl, float pyl, float pzh,
                                         float pzl, const QState<QT>& q, const bool (&nq)[QT],
                                         f2 (&sw)[QT / 2], f2 (&swz)[QT / 2],
                                         f2 (&cz)[QT / 2]) {
    constexpr int kPairs = QT / 2;
    const f2 px = pk2(pxh, pxh), py = pk2(pyh, pyh), pz = pk2(pzh, pzh);
#pragma unroll
    for (int r = 0; r < kPairs; ++r) {
        f2 w;
        if (MODE == 2) {
            float xh[2], yh[2], xl[2], yl[2], cc[2], bb[2], ss[2], ww[2];
            up2(q.xh[r], xh[0], xh[1]);
            up2(q.yh[r], yh[0], yh[1]);
            up2(q.xl[r], xl[0], xl[1]);
            up2(q.yl[r], yl[0], yl[1]);
            up2(q.c[r], cc[0], cc[1]);
            up2(q.b[r], bb[0], bb[1]);
            up2(q.s[r], ss[0], ss[1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float dx = pxh - xh[h], dy = pyh - yh[h];
                if (nq[2 * r + h]) {
                    dx = dx + (pxl - xl[h]);
                    dy = dy + (pyl - yl[h]);
                }
                const float d2 = fmaf(dx, dx, dy * dy);
                if (q.a[2 * r + h]) {
                    const float t = d2 * ss[h];
                    ww[h] = mufu_rcp(t * t);
                } else {
                    const float e = fmaf(cc[h], mufu_lg2(d2), bb[h]);
                    ww[h] = q.g2[2 * r + h] ? exp2_fma(e) : mufu_ex2(e);
                }
            }
            w = pk2(ww[0], ww[1]);
        } else {
            f2 dx = sub2(px, q.xh[r]), dy = sub2(py, q.yh[r]);
            if (DIST == 1) {
                dx = add2(dx, sub2(pk2(pxl, pxl), q.xl[r]));
                dy = add2(dy, sub2(pk2(pyl, pyl), q.yl[r]));
            } else if (DIST == 2) {
                dx = sel2(add2(dx, sub2(pk2(pxl, pxl), q.xl[r])), dx, nq[2 * r], nq[2 * r + 1]);
                dy = sel2(add2(dy, sub2(pk2(pyl, pyl), q.yl[r])), dy, nq[2 * r], nq[2 * r + 1]);
            }
            const f2 d2 = fma2(dx, dx, mul2(dy, dy));
            float lo, hi;
            if (MODE == 3) {  // recipe, s == 1 for every query of the warp
                up2(mul2(d2, d2), lo, hi);
                w = pk2(mufu_rcp(lo), mufu_rcp(hi));
            } else if (MODE == 0) {
                const f2 t = mul2(d2, q.s[r]);
                up2(mul2(t, t), lo, hi);
                w = pk2(mufu_rcp(lo), mufu_rcp(hi));
            } else if (MODE == 4 || (MODE == 5 && r % 2 == 1)) {  // G2: FMA-pipe exp2
                up2(d2, lo, hi);
                w = exp2_fma2(fma2(q.c[r], pk2(mufu_lg2(lo), mufu_lg2(hi)), q.b[r]));
            } else {
                up2(d2, lo, hi);
                up2(fma2(q.c[r], pk2(mufu_lg2(lo), mufu_lg2(hi)), q.b[r]), lo, hi);
                w = pk2(mufu_ex2(lo), mufu_ex2(hi));
            }
        }
        sw[r] = add2(sw[r], w);
        if (MODE == 2) {  // per query: compensated when near, plain when far
            float wv[2], sv[2], cv[2];
            up2(w, wv[0], wv[1]);
            up2(swz[r], sv[0], sv[1]);
            up2(cz[r], cv[0], cv[1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (nq[2 * r + h]) {
                    const float t = fmaf(wv[h], pzh, wv[h] * pzl);
                    const float y = t - cv[h];
                    const float s2 = sv[h] + y;
                    cv[h] = (s2 - sv[h]) - y;
                    sv[h] = s2;
                } else {
                    sv[h] = fmaf(wv[h], pzh, sv[h]);
                }
            }
            swz[r] = pk2(sv[0], sv[1]);
            cz[r] = pk2(cv[0], cv[1]);
        } else if (DIST == 0) {
            swz[r] = fma2(w, pz, swz[r]);
        } else {  // Kahan-compensated w z with hi/lo z
            const f2 t = fma2(w, pz, mul2(w, pk2(pzl, pzl)));
            const f2 y = sub2(t, cz[r]);
            const f2 s2 = add2(swz[r], y);
            const f2 c2 = sub2(sub2(s2, swz[r]), y);
            if (DIST == 1) {
                cz[r] = c2;
                swz[r] = s2;
            } else {
                cz[r] = sel2(c2, cz[r], nq[2 * r], nq[2 * r + 1]);
                swz[r] = sel2(s2, fma2(w, pz, swz[r]), nq[2 * r], nq[2 * r + 1]);
            }
        }
    }
}

// One 256-point tile, stored SoA in shared memory as
//   [x_hi | y_hi | x_lo | y_lo | z_hi | z_lo] x 256 floats,
// so one LDS.128 fetches a component of 4 consecutive points (far tiles read
// 3 components, near tiles 6: 0.75-1.5 LDS per 4 points per thread instead
// of 8), which keeps the MIO queue free for the MUFU work.
template <int MODE, int DIST, int QT>
__device__ __forceinline__ void k4_tile(const float* __restrict__ t, const QState<QT>& q,
                                        const bool (&nq)[QT], f2 (&sw)[QT / 2],
                                        f2 (&swz)[QT / 2], f2 (&cz)[QT / 2]) {
#pragma unroll 1
    for (int j = 0; j < kWeightTile; j += 4) {
        const float4 X = *reinterpret_cast<const float4*>(t + j);
        const float4 Y = *reinterpret_cast<const float4*>(t + kWeightTile + j);
        const float4 Z = *reinterpret_cast<const float4*>(t + 4 * kWeightTile + j);
        float4 XL = make_float4(0.f, 0.f, 0.f, 0.f), YL = XL, ZL = XL;
        if (DIST != 0 || MODE == 2) {
            XL = *reinterpret_cast<const float4*>(t + 2 * kWeightTile + j);
            YL = *reinterpret_cast<const float4*>(t + 3 * kWeightTile + j);
            ZL = *reinterpret_cast<const float4*>(t + 5 * kWeightTile + j);
        }
        k4_point<MODE, DIST, QT>(X.x, Y.x, XL.x, YL.x, Z.x, ZL.x, q, nq, sw, swz, cz);
        k4_point<MODE, DIST, QT>(X.y, Y.y, XL.y, YL.y, Z.y, ZL.y, q, nq, sw, swz, cz);
        k4_point<MODE, DIST, QT>(X.z, Y.z, XL.z, YL.z, Z.z, ZL.z, q, nq, sw, swz, cz);
        k4_point<MODE, DIST, QT>(X.w, Y.w, XL.w, YL.w, Z.w, ZL.w, q, nq, sw, swz, cz);
    }
}

template <int kQT, int kMinBlocks>
__global__ void __launch_bounds__(kK4Threads, kMinBlocks) weight_fp32_kernel(K4Args a) {
    constexpr int kPairs = kQT / 2;
    extern __shared__ __align__(128) unsigned char smem[];
    float* stile = reinterpret_cast<float*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(stile + kStages * kTileFloats);

    const unsigned chunk = blockIdx.y;
    const size_t t0 = static_cast<size_t>(chunk) * a.tiles_per_chunk;
    const size_t t1 = t0 + a.tiles_per_chunk < a.tiles ? t0 + a.tiles_per_chunk : a.tiles;
    const size_t ntl = t1 > t0 ? t1 - t0 : 0;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t wbase = static_cast<size_t>(blockIdx.x) * (kK4Threads * kQT) +
                         static_cast<size_t>(warp) * (32 * kQT);
    QState<kQT> q;
    bool any_a = false, any_g = false, any_g2 = false, any_scaled = false;
    {
        float4 h[kQT], r[kQT];
#pragma unroll
        for (int i = 0; i < kQT; ++i) {
            const size_t p = wbase + static_cast<size_t>(i) * 32 + lane;
            h[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            r[i] = make_float4(-1.f, 0.f, 1.f, 1.f);
            if (p < a.n) {
                h[i] = a.qhl[p];
                r[i] = a.qpar[p];
                q.a[i] = r[i].w == 1.0f;
                q.g2[i] = r[i].w == 2.0f;
                any_g2 |= q.g2[i];
                q.v[i] = true;
                any_a |= q.a[i];
                any_g |= !q.a[i] && !q.g2[i];
                any_scaled |= r[i].z != 1.0f;
            } else {
                q.a[i] = true;
                q.g2[i] = false;
                q.v[i] = false;
            }
        }
#pragma unroll
        for (int k = 0; k < kPairs; ++k) {
            const int i0 = 2 * k, i1 = 2 * k + 1;
            q.xh[k] = pk2(h[i0].x, h[i1].x);
            q.yh[k] = pk2(h[i0].y, h[i1].y);
            q.xl[k] = pk2(h[i0].z, h[i1].z);
            q.yl[k] = pk2(h[i0].w, h[i1].w);
            q.c[k] = pk2(r[i0].x, r[i1].x);
            q.b[k] = pk2(r[i0].y, r[i1].y);
            q.s[k] = pk2(r[i0].z, r[i1].z);
        }
    }
    any_a = __any_sync(0xFFFFFFFFu, any_a);
    any_g = __any_sync(0xFFFFFFFFu, any_g);
    any_g2 = __any_sync(0xFFFFFFFFu, any_g2);
    any_scaled = __any_sync(0xFFFFFFFFu, any_scaled);
    // warp-uniform formula group; per query the arithmetic is identical in
    // every mode (s == 1 makes d2 * s == d2 exactly), so grouping never
    // changes a result
    const int classes = (any_a ? 1 : 0) + (any_g ? 1 : 0) + (any_g2 ? 1 : 0);
    // the interleaved layout: pair 0 all G1 and pair 1 all G2 across the warp
    bool split = kQT == 4;
#pragma unroll
    for (int i = 0; i < kQT; ++i) {
        const bool want_g2 = i >= kQT / 2;
        split &= !q.v[i] || (!q.a[i] && q.g2[i] == want_g2);
    }
    split = __all_sync(0xFFFFFFFFu, split) && any_g && any_g2;
    const int mode = split ? 5
                     : classes > 1 ? 2 : any_g2 ? 4 : any_g ? 1 : (any_scaled ? 0 : 3);

    double SW[kQT], SWZ[kQT];
#pragma unroll
    for (int i = 0; i < kQT; ++i) SW[i] = SWZ[i] = 0.0;

    constexpr uint32_t kTileBytes = kTileFloats * sizeof(float);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
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
        f2 sw[kPairs], swz[kPairs], cz[kPairs];
#pragma unroll
        for (int k = 0; k < kPairs; ++k) sw[k] = swz[k] = cz[k] = 0ull;
        // per-(query, tile) near flags, then a warp-uniform dispatch
        const float4 tb = __ldg(a.tile_box + t0 + it);
        bool nq[kQT];
        bool any_near = false, all_near = true;
#pragma unroll
        for (int k = 0; k < kPairs; ++k) {
            float x[2], y[2];
            up2(q.xh[k], x[0], x[1]);
            up2(q.yh[k], y[0], y[1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float ex = fmaxf(0.0f, fmaxf(tb.x - x[h], x[h] - tb.z));
                const float ey = fmaxf(0.0f, fmaxf(tb.y - y[h], y[h] - tb.w));
                nq[2 * k + h] = fmaf(ex, ex, ey * ey) <= a.rfar2;
                if (q.v[2 * k + h]) {  // empty slots never force a mixed tile
                    any_near |= nq[2 * k + h];
                    all_near &= nq[2 * k + h];
                }
            }
        }
        any_near = __any_sync(0xFFFFFFFFu, any_near);
        all_near = __all_sync(0xFFFFFFFFu, all_near);
        const int dist = !any_near ? 0 : (all_near ? 1 : 2);
        if (mode == 3) {
            if (dist == 0) k4_tile<3, 0, kQT>(tt, q, nq, sw, swz, cz);
            else if (dist == 1) k4_tile<3, 1, kQT>(tt, q, nq, sw, swz, cz);
            else k4_tile<3, 2, kQT>(tt, q, nq, sw, swz, cz);
        } else if (mode == 0) {
            if (dist == 0) k4_tile<0, 0, kQT>(tt, q, nq, sw, swz, cz);
            else k4_tile<0, 2, kQT>(tt, q, nq, sw, swz, cz);
        } else if (mode == 5) {
            if (dist == 0) k4_tile<5, 0, kQT>(tt, q, nq, sw, swz, cz);
            else if (dist == 1) k4_tile<5, 1, kQT>(tt, q, nq, sw, swz, cz);
            else k4_tile<5, 2, kQT>(tt, q, nq, sw, swz, cz);
        } else if (mode == 4) {
            if (dist == 0) k4_tile<4, 0, kQT>(tt, q, nq, sw, swz, cz);
            else if (dist == 1) k4_tile<4, 1, kQT>(tt, q, nq, sw, swz, cz);
            else k4_tile<4, 2, kQT>(tt, q, nq, sw, swz, cz);
        } else if (mode == 1) {
            if (dist == 0) k4_tile<1, 0, kQT>(tt, q, nq, sw, swz, cz);
            else if (dist == 1) k4_tile<1, 1, kQT>(tt, q, nq, sw, swz, cz);
            else k4_tile<1, 2, kQT>(tt, q, nq, sw, swz, cz);
        } else {
            k4_tile<2, 2, kQT>(tt, q, nq, sw, swz, cz);
        }
#pragma unroll
        for (int k = 0; k < kPairs; ++k) {
            float lo, hi;
            up2(sw[k], lo, hi);
            SW[2 * k] += static_cast<double>(lo);
            SW[2 * k + 1] += static_cast<double>(hi);
            up2(swz[k], lo, hi);
            float clo, chi;
            up2(cz[k], clo, chi);
            SWZ[2 * k] += static_cast<double>(lo) - static_cast<double>(clo);
            SWZ[2 * k + 1] += static_cast<double>(hi) - static_cast<double>(chi);
        }
        __syncthreads();
        if (threadIdx.x == 0 && it + kStages < ntl) {
            fence_proxy_async();
            const size_t tile = t0 + it + kStages;
            mbar_expect_tx(&bar[st], kTileBytes);
            bulk_load(stile + st * kTileFloats, a.rec + tile * kTileFloats, kTileBytes, &bar[st]);
        }
    }
#pragma unroll
    for (int i = 0; i < kQT; ++i) {
        const size_t p = wbase + static_cast<size_t>(i) * 32 + lane;
        if (p < a.n) a.part[p * a.chunks + chunk] = make_double2(SW[i], SWZ[i]);
    }
}

// ------------------------------------------------------------ settle
__global__ void settle_kernel(const WeightQueries q, WeightFrame f, const WeightData d,
                              const uint32_t* __restrict__ order,
                              const double2* __restrict__ part,
                              const double* __restrict__ lshift, unsigned chunks,
                              double* __restrict__ pred, double* __restrict__ alpha_out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= q.n) return;
    const uint32_t p = order[i];
    const uint32_t qi = q.perm ? q.perm[p] : p;
    const double alpha = q.alpha_s[p];
    double out;
    const uint32_t snap = q.snap_s[p];
    if (snap != kNoId) {
        out = d.z[snap];
    } else {
        double sw = 0.0, swz = 0.0;
        for (unsigned c = 0; c < chunks; ++c) {
            const double2 v = part[static_cast<size_t>(i) * chunks + c];
            sw += v.x;
            swz += v.y;
        }
        // The FP64 reference overflows / underflows where the true (unscaled)
        // weights do (interpolate.hpp:109-118): its largest weight is
        // 2^e, e = -alpha/2 log2 d2_min; its sums are 2^lshift * (sw, swz / 2^zshift).
        const double e = -0.5 * alpha * log2(q.d2min_s[p]);
        const double sh = lshift[i];
        bool fallback = !(sw > 0.0) || !isfinite(sw) || !isfinite(swz) || !(e < 1024.0) ||
                        !(sh + log2(sw) < 1024.0) || e < -1075.0;
        if (!fallback && swz != 0.0 && !(sh + log2(fabs(swz)) - f.zshift < 1024.0)) fallback = true;
        if (fallback) {
            out = d.z[q.nn_s[p]];
        } else {
            double v = ldexp(swz / sw, -f.zshift);
            out = v < f.zlo ? f.zlo : (v > f.zhi ? f.zhi : v);
        }
    }
    pred[qi] = out;
    if (alpha_out) alpha_out[qi] = alpha;
}

}  // namespace

void set_alpha4_recipe(bool enabled) { g_alpha4_recipe.store(enabled); }

WeightSplit weight_split(size_t m) {
    WeightSplit w;
    w.tiles = (m + kWeightTile - 1) / kWeightTile;
    if (w.tiles == 0) w.tiles = 1;
    size_t chunks = w.tiles < static_cast<size_t>(kMaxChunks) ? w.tiles : kMaxChunks;
    w.tiles_per_chunk = (w.tiles + chunks - 1) / chunks;
    w.chunks = static_cast<unsigned>((w.tiles + w.tiles_per_chunk - 1) / w.tiles_per_chunk);
    return w;
}

void weighting_fp32(const WeightQueries& q, const WeightData& d, const WeightFrame& f,
                    double* d_pred, double* d_alpha, WeightTimes* times, cudaStream_t s) {
    if (q.n == 0) return;
    const WeightSplit sp = weight_split(d.m);
    const size_t mp = sp.tiles * kWeightTile;
    DBuf<float> rec(sp.tiles * kTileFloats, s);
    DBuf<float4> tbox(sp.tiles, s);
    LAUNCH(prep_data_kernel, ceil_div(mp, kThreads), kThreads, 0, s, d.x, d.y, d.z, d.order, d.m,
           mp, f.ox, f.oy, f.inv_scale, std::ldexp(1.0, f.zshift), rec.get());
    LAUNCH(tile_box_kernel, ceil_div(sp.tiles * 32, kThreads), kThreads, 0, s, rec.get(), d.m,
           sp.tiles, tbox.get());

    DBuf<uint32_t> flag(q.n, s), scan_a(q.n, s), flag_g2(q.n, s), scan_g2(q.n, s), order(q.n, s);
    DBuf<float4> qhl(q.n, s), qpar(q.n, s);
    DBuf<double> lshift(q.n, s);
    LAUNCH(class_flags_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q,
           g_alpha4_recipe.load() ? 1 : 0, flag.get(), flag_g2.get());
    exclusive_scan_u32(flag.get(), scan_a.get(), q.n, s);
    exclusive_scan_u32(flag_g2.get(), scan_g2.get(), q.n, s);
    LAUNCH(query_records_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q, f, flag.get(),
           scan_a.get(), flag_g2.get(), scan_g2.get(), order.get(), qhl.get(), qpar.get(),
           lshift.get(),
           times ? times->d_alpha4 : nullptr);

    DBuf<double2> part(q.n * sp.chunks, s);
    // near / far threshold (unit-box units): beyond it a pair's plain FP32
    // difference has relative error <= ~8.4e-8 / R_far (AIDW_K4_RFAR to tune)
    static const float rfar = [] {
        const char* v = std::getenv("AIDW_K4_RFAR");
        return v ? static_cast<float>(std::atof(v)) : 0.05f;
    }();
    K4Args ka{rec.get(), sp.tiles, sp.tiles_per_chunk, sp.chunks, qhl.get(), qpar.get(),
              q.n, part.get(), tbox.get(), rfar * rfar};
    const size_t smem = kStages * kTileFloats * sizeof(float) +
                        kStages * sizeof(uint64_t);
    // K4 variant: queries per thread x min resident CTAs (AIDW_K4_VARIANT for
    // tuning; default 4 x 3).  Per-query arithmetic is identical in all.
    static const int variant = [] {
        const char* v = std::getenv("AIDW_K4_VARIANT");
        return v ? std::atoi(v) : 0;
    }();
    auto launch = [&](auto kernel, int qt) {
        CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        dim3 grid(ceil_div(q.n, static_cast<size_t>(kK4Threads) * qt), sp.chunks);
        if (times && times->k4_begin) CK(cudaEventRecord(times->k4_begin, s));
        LAUNCH(kernel, grid, kK4Threads, smem, s, ka);
    };
    switch (variant) {
        case 1: launch(weight_fp32_kernel<4, 2>, 4); break;
        case 2: launch(weight_fp32_kernel<2, 4>, 2); break;
        default: launch(weight_fp32_kernel<4, 3>, 4); break;
    }
    if (times && times->k4_end) CK(cudaEventRecord(times->k4_end, s));
    LAUNCH(settle_kernel, ceil_div(q.n, kThreads), kThreads, 0, s, q, f, d, order.get(),
           part.get(), lshift.get(), sp.chunks, d_pred, d_alpha);
}

}  // namespace aidwb
