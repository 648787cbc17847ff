// weight_tc.cu — K4 with the far-form d2 on the 5th-generation tensor cores.
//
// Same contract as the CUDA-core K4 in weight.cu (interpolate.hpp:252-381,
// :426-489): per (data chunk, query) FP64 partials {sum w', sum w' z'} that
// settle_kernel adds in chunk order.  What moves to the tensor cores is the
// far-form distance of every (query, point) pair of a tile,
//     d2 = |q'|^2 - 2 q'.p' + |p'|^2        (q' = q - c, p' = p - c, c the tile centre)
// as one kind::tf32 tcgen05.mma per (128 queries x 64 points): the A row of a
// query holds exact TF32 pieces of q'x, q'y (hi / mid / lo, 24 bits) and
// |q'|^2, the B row of a point the 22-bit pieces of -2 p'x, -2 p'y, |p'|^2
// (K = 16, the hi x lo cross terms included), so the FP32 accumulator sees
// exact products: d2 carries the rounding of the FP32 far form, a few ulp of
// (|q'| + |p'|)^2 (measured max 1.6e-6 relative on far pairs, tools/tc_proto.cu).
//
// Layout: one CTA per SM, 3 query groups x 128 queries (one TMEM lane each),
// 12 epilogue warps (a group's 4 warps cover TMEM lanes 0-127), a producer
// warp whose lane 0 streams 22.5 KB tile records (B operand + near
// components) into a 4-stage shared-memory ring with the bulk-copy engine,
// and a control warp whose lane 0 issues the MMAs into two 64-column TMEM
// buffers per group.  An
// epilogue thread owns one query: per 64-point part it loads its 64 d2 with
// one tcgen05.ld (32x32b.x64), releases the buffer to the next MMA at once
// and runs its class's weight form on the registers (alpha = 4: two points
// per reciprocal, w0 + w2 = (a0 + a2) rcp(a0 a2)); it rebuilds its A row for
// each tile's centre.  (Query, tile) pairs within the near threshold (and
// partial tiles) discard the far sums and take the hi/lo near form on the
// CUDA cores, Kahan-compensated, exactly as in weight.cu.
//
// Every per-query result is a function of the query and the data only (the
// MMA row, the class form and the per-thread accumulation order do not
// depend on the other queries of the CTA), so sharding and GPU count never
// change a bit.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"
#include "weight.cuh"
#include "weight_ops.cuh"

namespace aidwb {

namespace {

using namespace wops;
using namespace tc;

#ifndef AIDW_TC_N
#define AIDW_TC_N 64
#endif
#ifndef AIDW_TC_BUFS
#define AIDW_TC_BUFS 2
#endif
#ifndef AIDW_TC_SPLITLD
#define AIDW_TC_SPLITLD 0
#endif
#ifndef AIDW_TC_STAGES
#define AIDW_TC_STAGES 4
#endif
#ifndef AIDW_TC_GROUPS
#define AIDW_TC_GROUPS 3
#endif
constexpr int kGroups = AIDW_TC_GROUPS;          // query groups (one MMA M = 128 each)
constexpr int kN = AIDW_TC_N;                    // MMA N: points per part
constexpr int kParts = kWeightTile / kN;         // parts per tile
constexpr int kBufs = AIDW_TC_BUFS;              // TMEM accumulators per group
constexpr int kStages = AIDW_TC_STAGES;          // tile records in flight
#ifndef AIDW_TC_NONEAR_DEBUG
#define AIDW_TC_NONEAR_DEBUG 0  // timing experiments only: skip the near passes (wrong sums)
#endif
#ifndef AIDW_TC_TRACE
#define AIDW_TC_TRACE 0  // timing experiments only: per-warp wait cycles of one CTA (printf)
#endif
#if AIDW_TC_TRACE
#define TRACE_T0(v) const long long v = clock64()
#define TRACE_ADD(acc, v0) acc += clock64() - (v0)
#define TRACE_CTA (blockIdx.x == 200 && blockIdx.y == 5)
#else
#define TRACE_T0(v)
#define TRACE_ADD(acc, v0)
#endif
constexpr int kEpiWarps = 4 * kGroups;
constexpr int kCtlWarp = kEpiWarps;              // MMA issue (lane 0), TMEM owner
constexpr int kProdWarp = kEpiWarps + 1;         // stage refills (lane 0)
constexpr int kTcThreads = (kEpiWarps + 2) * 32;
constexpr int kCtaQ = 128 * kGroups;             // queries per CTA
constexpr uint32_t kBBytes = kWeightTile * kK * 4;           // 16 KB B operand
constexpr uint32_t kNearBytes = 6 * kWeightTile * 4;         // z and near-form coordinates
constexpr uint32_t kRecBytes = kBBytes + kNearBytes;         // per tile record
constexpr uint32_t kABytes = 128 * kK * 4;                   // 8 KB A operand per group
constexpr uint32_t kTmemCols = 512;                          // >= 2 buffers x groups x kN
static_assert(kBufs * kGroups * kN <= static_cast<int>(kTmemCols), "TMEM budget");
enum : int { kNZH, kNZL, kNXH, kNYH, kNXL, kNYL };         // near components after B

constexpr size_t kSmemBytes = kStages * kRecBytes + 2 * kGroups * kABytes +
                              (2 * kStages + (2 + 2 * kBufs) * kGroups) * sizeof(uint64_t) + 16;

// Query classes of the TC engine (from qpar): the recipe codes and the two
// general exponential forms.
enum : int { kClsA4, kClsA2, kClsA1, kClsA3, kClsG, kClsMixed };
#ifndef AIDW_TC_GMUFU
#define AIDW_TC_GMUFU 1
#endif
constexpr int kGMufu = AIDW_TC_GMUFU;  // general class: MUFU exp2 slots of 4
// General class: lg2 on MUFU for every pair; the exp2 of one point slot in
// four on MUFU, of the other three as the degree-5 polynomial on the FMA pipe
// (1.25 MUFU + ~10 FP32 ops per pair balances the two pipes; the split is by
// point position, so every warp carries the same mix).

// ------------------------------------------------------------ records
__device__ __forceinline__ void split_tf32(double v, float& hi, float& lo) {
    hi = tf32_hi(__double2float_rn(v));
    lo = tf32_hi(__double2float_rn(__dsub_rn(v, static_cast<double>(hi))));
}

// One CTA per tile: the B operand rows (-2 p'x, -2 p'y, |p'|^2 in 22-bit
// TF32 pieces, p' about the tile centre exactly as tile_geo_kernel forms it)
// in the canonical K-major layout, then the near-form components.
__global__ void __launch_bounds__(kWeightTile) tc_records_kernel(const float* __restrict__ rec,
                                                                const float4* __restrict__ geo,
                                                                size_t m, char* __restrict__ out) {
    const size_t tile = blockIdx.x;
    const int j = threadIdx.x;
    const float* t = rec + tile * kTileFloats;
    char* o = out + tile * kRecBytes;
    const bool real = tile * kWeightTile + j < m;
    const float xh = t[kXH * kWeightTile + j], yh = t[kYH * kWeightTile + j];
    const float xl = t[kXL * kWeightTile + j], yl = t[kYL * kWeightTile + j];
    float b[16] = {};
    if (real) {
        const float4 g = geo[tile];
        const double px = __dadd_rn(__dsub_rn(static_cast<double>(xh), static_cast<double>(g.x)),
                                    static_cast<double>(xl));
        const double py = __dadd_rn(__dsub_rn(static_cast<double>(yh), static_cast<double>(g.y)),
                                    static_cast<double>(yl));
        float bxh, bxl, byh, byl, ph, pl;
        split_tf32(-2.0 * px, bxh, bxl);
        split_tf32(-2.0 * py, byh, byl);
        split_tf32(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), ph, pl);
        const float r[16] = {bxh, bxl, bxh, bxl, bxh, byh, byl, byh, byl, byh,
                             1.0f, 1.0f, 1.0f, ph, pl, 0.0f};
#pragma unroll
        for (int k = 0; k < 16; ++k) b[k] = r[k];
    }
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4)
        *reinterpret_cast<float4*>(o + operand_offset(j, 4 * c4)) =
            make_float4(b[4 * c4], b[4 * c4 + 1], b[4 * c4 + 2], b[4 * c4 + 3]);
    float* nf = reinterpret_cast<float*>(o + kBBytes);
    nf[kNZH * kWeightTile + j] = t[kZH * kWeightTile + j];
    nf[kNZL * kWeightTile + j] = t[kZL * kWeightTile + j];
    nf[kNXH * kWeightTile + j] = xh;
    nf[kNYH * kWeightTile + j] = yh;
    nf[kNXL * kWeightTile + j] = xl;
    nf[kNYL * kWeightTile + j] = yl;
}

// ------------------------------------------------------------ A operand
// The query's A row for one tile centre: q' = (q_hi - c) + q_lo in FP32 (the
// CUDA-core far form's q'), split exactly into TF32 hi / mid / lo pieces.
__device__ __forceinline__ void build_a(char* abuf, int r, float4 q, float4 c) {
    const float fx = (q.x - c.x) + q.z;
    const float fy = (q.y - c.y) + q.w;
    const float fq = fmaf(fx, fx, fy * fy);
    const float xh = tf32_hi(fx), xr = fx - xh, xm = tf32_hi(xr), xl = xr - xm;
    const float yh = tf32_hi(fy), yr = fy - yh, ym = tf32_hi(yr), yl = yr - ym;
    const float qh = tf32_hi(fq), qr = fq - qh, qm = tf32_hi(qr), ql = qr - qm;
    const float a[16] = {xh, xh, xm, xm, xl, yh, yh, ym, ym, yl, qh, qm, ql, 1.0f, 1.0f, 0.0f};
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4)
        *reinterpret_cast<float4*>(abuf + operand_offset(r, 4 * c4)) =
            make_float4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
}

// ------------------------------------------------------------ weight forms
struct QConst {
    f2 c, b;  // general: w' = ex2(c lg2(d2) + b), broadcast to both lanes
    f2 s;     // alpha = 4 near-form range scale (a power of two)
};

// Far sums of one part (64 d2 in registers, lanes = points j, j + 1).
// Paired classes take points (j, j + 2) and (j + 1, j + 3) on one reciprocal.
template <int CLS, int C = kN>
__device__ __forceinline__ void far_part(const uint32_t (&v)[C], const float* __restrict__ z,
                                         const QConst& qc, f2& sw0, f2& swz0, f2& sw1, f2& swz1) {
#pragma unroll
    for (int j = 0; j < C; j += 8) {
        const float4 Za = *reinterpret_cast<const float4*>(z + j);
        const float4 Zb = *reinterpret_cast<const float4*>(z + j + 4);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int o = j + 4 * hh;
            const float4 Z = hh ? Zb : Za;
            const f2 d01 = pk2(__uint_as_float(v[o]), __uint_as_float(v[o + 1]));
            const f2 d23 = pk2(__uint_as_float(v[o + 2]), __uint_as_float(v[o + 3]));
            const f2 Z01 = pk2(Z.x, Z.y), Z23 = pk2(Z.z, Z.w);
            f2& sw = hh ? sw1 : sw0;
            f2& swz = hh ? swz1 : swz0;
            if (CLS == kClsA4 || CLS == kClsA2) {
                const f2 A = CLS == kClsA4 ? mul2(d01, d01) : d01;
                const f2 B = CLS == kClsA4 ? mul2(d23, d23) : d23;
                const f2 R = rcp2(mul2(A, B));
                sw = fma2(R, add2(A, B), sw);
                swz = fma2(R, fma2(B, Z01, mul2(A, Z23)), swz);
            } else {
                f2 w0, w1;
                if (CLS == kClsA1) {
                    w0 = rsq2(d01), w1 = rsq2(d23);
                } else if (CLS == kClsA3) {
                    w0 = cube2(rsq2(d01)), w1 = cube2(rsq2(d23));
                } else {
                    float a0, a1, b0, b1;
                    up2(d01, a0, a1);
                    up2(d23, b0, b1);
                    const f2 e0 = fma2(qc.c, pk2(mufu_lg2(a0), mufu_lg2(a1)), qc.b);
                    const f2 e1 = fma2(qc.c, pk2(mufu_lg2(b0), mufu_lg2(b1)), qc.b);
                    // MUFU exp2 on kGMufu of every 4 f32x2 slots (slot = 2 hh + k)
                    if (2 * hh < kGMufu) {
                        up2(e0, a0, a1);
                        w0 = pk2(mufu_ex2(a0), mufu_ex2(a1));
                    } else {
                        w0 = exp2_fma2(e0);
                    }
                    if (2 * hh + 1 < kGMufu) {
                        up2(e1, b0, b1);
                        w1 = pk2(mufu_ex2(b0), mufu_ex2(b1));
                    } else {
                        w1 = exp2_fma2(e1);
                    }
                }
                sw = add2(sw, w0);
                swz = fma2(w0, Z01, swz);
                sw = add2(sw, w1);
                swz = fma2(w1, Z23, swz);
            }
        }
    }
}

template <int C>
__device__ __forceinline__ void far_part_mixed(int cls, const uint32_t (&v)[C],
                                               const float* __restrict__ z, const QConst& qc,
                                               f2& sw0, f2& swz0, f2& sw1, f2& swz1) {
    switch (cls) {  // divergent, each lane its own class's form
        case kClsA4: far_part<kClsA4, C>(v, z, qc, sw0, swz0, sw1, swz1); break;
        case kClsA2: far_part<kClsA2, C>(v, z, qc, sw0, swz0, sw1, swz1); break;
        case kClsA1: far_part<kClsA1, C>(v, z, qc, sw0, swz0, sw1, swz1); break;
        case kClsA3: far_part<kClsA3, C>(v, z, qc, sw0, swz0, sw1, swz1); break;
        default: far_part<kClsG, C>(v, z, qc, sw0, swz0, sw1, swz1); break;
    }
}

// One part's far sums from TMEM.  Default: one x64 load, released at once,
// then the sums.  AIDW_TC_SPLITLD: two x32 loads, the second in flight
// while the first half's sums run.
template <int MODE>
__device__ __forceinline__ void far_tmem_part(uint32_t ta, const float* __restrict__ z, int cls,
                                              const QConst& qc, uint64_t* tempty, int lane,
                                              f2& sw0, f2& swz0, f2& sw1, f2& swz1) {
#if AIDW_TC_SPLITLD
    static_assert(kN == 64, "split load: two 32-column halves");
    uint32_t lo[32], hi[32];
    tmem_ld32(ta, lo);
    tmem_wait_ld();
    tmem_hold(lo);
    tmem_ld32_after(ta + 32, hi, lo);
    if (MODE == kClsMixed) far_part_mixed<32>(cls, lo, z, qc, sw0, swz0, sw1, swz1);
    else far_part<MODE, 32>(lo, z, qc, sw0, swz0, sw1, swz1);
    tmem_wait_ld_after(sw0, swz0, sw1, swz1);
    tmem_hold(hi);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty);
    if (MODE == kClsMixed) far_part_mixed<32>(cls, hi, z + 32, qc, sw0, swz0, sw1, swz1);
    else far_part<MODE, 32>(hi, z + 32, qc, sw0, swz0, sw1, swz1);
#else
    uint32_t v[kN];
    tmem_ld(ta, v);
    tmem_wait_ld();
    tmem_hold(v);
    // the registers hold the part: release the buffer to the next MMA
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty);
    if (MODE == kClsMixed) far_part_mixed<kN>(cls, v, z, qc, sw0, swz0, sw1, swz1);
    else far_part<MODE>(v, z, qc, sw0, swz0, sw1, swz1);
#endif
}

// Near weight of a pair of points for one query (the hi/lo distance d2).
template <int CLS>
__device__ __forceinline__ f2 near_w(f2 d2, const QConst& qc) {
    if (CLS == kClsA4) {
        const f2 t = mul2(d2, qc.s);
        return rcp2(mul2(t, t));
    }
    if (CLS == kClsA2) return rcp2(d2);
    if (CLS == kClsA1) return rsq2(d2);
    if (CLS == kClsA3) return cube2(rsq2(d2));
    float lo, hi;
    up2(d2, lo, hi);
    const f2 e = fma2(qc.c, pk2(mufu_lg2(lo), mufu_lg2(hi)), qc.b);
    up2(e, lo, hi);
    return pk2(mufu_ex2(lo), mufu_ex2(hi));
}

// Near form over one tile: dx = (x_hi - q_hi) + (x_lo - q_lo), Kahan sums
// with hi / lo z (lanes = even / odd points); returns the compensated sums.
template <int CLS>
__device__ __forceinline__ void near_tile(const float* __restrict__ nf, float4 q, const QConst& qc,
                                          double& SW, double& SWZ) {
    const f2 qxh = bc2(q.x), qyh = bc2(q.y), qxl = bc2(q.z), qyl = bc2(q.w);
    f2 sw = 0ull, swz = 0ull, cw = 0ull, cz = 0ull;
#pragma unroll 4
    for (int j = 0; j < kWeightTile; j += 2) {
        const float2 X = *reinterpret_cast<const float2*>(nf + kNXH * kWeightTile + j);
        const float2 Y = *reinterpret_cast<const float2*>(nf + kNYH * kWeightTile + j);
        const float2 XL = *reinterpret_cast<const float2*>(nf + kNXL * kWeightTile + j);
        const float2 YL = *reinterpret_cast<const float2*>(nf + kNYL * kWeightTile + j);
        const float2 Z = *reinterpret_cast<const float2*>(nf + kNZH * kWeightTile + j);
        const float2 ZL = *reinterpret_cast<const float2*>(nf + kNZL * kWeightTile + j);
        const f2 dx = add2(sub2(pk2(X.x, X.y), qxh), sub2(pk2(XL.x, XL.y), qxl));
        const f2 dy = add2(sub2(pk2(Y.x, Y.y), qyh), sub2(pk2(YL.x, YL.y), qyl));
        const f2 d2 = fma2(dx, dx, mul2(dy, dy));
        const f2 w = near_w<CLS>(d2, qc);
        {
            const f2 yw = sub2(w, cw);
            const f2 s1 = add2(sw, yw);
            cw = sub2(sub2(s1, sw), yw);
            sw = s1;
        }
        const f2 tz = fma2(w, pk2(Z.x, Z.y), mul2(w, pk2(ZL.x, ZL.y)));
        const f2 y = sub2(tz, cz);
        const f2 s2 = add2(swz, y);
        cz = sub2(sub2(s2, swz), y);
        swz = s2;
    }
    float w0, w1, e0, e1, z0, z1, c0, c1;
    up2(sw, w0, w1);
    up2(cw, e0, e1);
    up2(swz, z0, z1);
    up2(cz, c0, c1);
    SW += (static_cast<double>(w0) - static_cast<double>(e0)) +
          (static_cast<double>(w1) - static_cast<double>(e1));
    SWZ += (static_cast<double>(z0) - static_cast<double>(c0)) +
           (static_cast<double>(z1) - static_cast<double>(c1));
}

__device__ __forceinline__ void near_tile_any(int cls, const float* nf, float4 q, const QConst& qc,
                                              double& SW, double& SWZ) {
    switch (cls) {
        case kClsA4: near_tile<kClsA4>(nf, q, qc, SW, SWZ); break;
        case kClsA2: near_tile<kClsA2>(nf, q, qc, SW, SWZ); break;
        case kClsA1: near_tile<kClsA1>(nf, q, qc, SW, SWZ); break;
        case kClsA3: near_tile<kClsA3>(nf, q, qc, SW, SWZ); break;
        default: near_tile<kClsG>(nf, q, qc, SW, SWZ); break;
    }
}

// ------------------------------------------------------------ kernel
struct TcArgs {
    const char* rec;  // tiles x kRecBytes
    size_t tiles, tiles_per_chunk;
    const float4* qhl;
    const float4* qpar;
    size_t n;
    const uint32_t* flag_a;  // class counts: A = scan_a[n-1] + flag_a[n-1]
    const uint32_t* scan_a;
    size_t s0, s1;            // query slab [s0, s1) of the visiting order
    double2* part;            // chunks x (s1 - s0), chunk-major
    const float4* tile_box;
    const float4* tile_geo;
    unsigned classes;  // 1: general region, 2: recipe region, 3: both
};

struct Smem {
    char* stage;
    char* abuf;
    uint64_t *bfull, *bempty, *afull, *tfull, *tempty;
    uint32_t* tmem_slot;
};

__device__ __forceinline__ Smem carve(char* smem) {
    Smem s;
    s.stage = smem;
    s.abuf = smem + kStages * kRecBytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(s.abuf + 2 * kGroups * kABytes);
    s.bfull = bar;
    s.bempty = bar + kStages;
    s.afull = bar + 2 * kStages;           // [group][2]
    s.tfull = s.afull + 2 * kGroups;       // [group][buffer]
    s.tempty = s.tfull + kBufs * kGroups;  // [group][buffer]
    s.tmem_slot = reinterpret_cast<uint32_t*>(s.tempty + kBufs * kGroups);
    return s;
}

// Producer warp, lane 0: tile records through the stage ring (bulk-copy
// engine).  A stage is refilled once every epilogue warp and every group's
// MMAs are done with its tile.
__device__ __forceinline__ void producer(const TcArgs& a, const Smem& sm, size_t t0, int T) {
    for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        if (t >= kStages) mbar_wait(&sm.bempty[s], ((t / kStages) - 1) & 1);
        mbar_expect_tx(&sm.bfull[s], kRecBytes);
        bulk_load(sm.stage + s * kRecBytes, a.rec + (t0 + t) * kRecBytes, kRecBytes, &sm.bfull[s]);
    }
}

// MMA issuer, the control warp: parts in order, for each part the groups
// in order.  Group g's part u = (tile t, part h) needs the tile's stage
// (bfull), the group's A rows for t (afull) and its TMEM buffer u % kBufs
// released (tempty).  After the last part of a tile the MMAs' completion
// releases the stage (bempty counts one commit per group).  The whole warp
// runs the loop (warp-uniform addresses and descriptors live in uniform
// registers) and one elected lane issues: sub-partition 0 also hosts three
// epilogue warps, and every group has a warp there, so the issuer's
// instruction count paces the CTA.  (Measured alternatives, no gain or
// worse: the refill wait inside this loop, one issuer warp per group on
// sub-partitions 1-3, a non-blocking per-group issue loop — 30 % slower:
// its polling takes issue slots from sub-partition 0's epilogue warps.)
__device__ __forceinline__ void issuer(const Smem& sm, uint32_t tbase, int T) {
    constexpr uint32_t idesc = idesc_tf32(128, kN);
    const uint64_t desc0 = smem_desc(0, kKChunkBytes, kRowGroupBytes);
    const uint32_t stage0 = smem_u32(sm.stage), abuf0 = smem_u32(sm.abuf);
#if AIDW_TC_TRACE
    long long wb = 0, wa = 0, we[kGroups] = {}, tall = clock64();
#endif
    for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        TRACE_T0(c0);
        mbar_wait(&sm.bfull[s], (t / kStages) & 1);
        TRACE_ADD(wb, c0);
        TRACE_T0(c1);
        for (int g = 0; g < kGroups; ++g) mbar_wait(&sm.afull[g * 2 + (t & 1)], (t >> 1) & 1);
        TRACE_ADD(wa, c1);
        tc_fence_after();
        const uint32_t b0 = stage0 + s * kRecBytes;
#pragma unroll
        for (int h = 0; h < kParts; ++h) {
            const uint32_t bh = b0 + h * (kN / 8) * kRowGroupBytes;
            const int u = t * kParts + h, b = u % kBufs;
#pragma unroll
            for (int g = 0; g < kGroups; ++g) {
                TRACE_T0(c2);
                if (u >= kBufs) mbar_wait(&sm.tempty[g * kBufs + b], ((u / kBufs) - 1) & 1);
                TRACE_ADD(we[g], c2);
                tc_fence_after();
                const uint32_t a0 = abuf0 + (g * 2 + (t & 1)) * kABytes;
                const uint32_t d = tbase + (g * kBufs + b) * kN;
                if (elect_one()) {
                    mma_tf32(d, smem_desc_at(desc0, a0), smem_desc_at(desc0, bh), idesc, false);
                    mma_tf32(d, smem_desc_at(desc0, a0 + 2 * kKChunkBytes),
                             smem_desc_at(desc0, bh + 2 * kKChunkBytes), idesc, true);
                    mma_commit(&sm.tfull[g * kBufs + b]);
                }
                __syncwarp();
            }
        }
        if (elect_one())
            for (int g = 0; g < kGroups; ++g) mma_commit(&sm.bempty[s]);
        __syncwarp();
    }
#if AIDW_TC_TRACE
    if (TRACE_CTA && (threadIdx.x & 31) == 0)
        printf("issuer: total %lld  wait bfull %lld afull %lld tempty g0 %lld g1 %lld g2 %lld (T %d)\n",
               clock64() - tall, wb, wa, we[0], we[1], we[kGroups - 1], T);
#endif
}

// Epilogue warp: the tile loop for one weight form (MODE = a class, or
// kClsMixed: each lane its own class).
template <int MODE>
__device__ __forceinline__ void epilogue(const TcArgs& a, const Smem& sm, uint32_t tbase,
                                         size_t t0, int T, int g, int quarter, int lane, bool valid,
                                         float4 q, int cls, const QConst& qc, double m0,
                                         double& SW, double& SWZ) {
    const int r = quarter * 32 + lane;
    char* myabuf = sm.abuf + g * 2 * kABytes;
#if AIDW_TC_TRACE
    long long wf = 0, tpart = 0, ttile = 0, tbuild = 0, tall = clock64();
#endif
    for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        const char* st = sm.stage + s * kRecBytes;
        const float* nf = reinterpret_cast<const float*>(st + kBBytes);
        const float4 tb = __ldg(a.tile_box + t0 + t);
        const float4 tg = __ldg(a.tile_geo + t0 + t);
        const float ex = fmaxf(0.0f, fmaxf(tb.x - q.x, q.x - tb.z));
        const float ey = fmaxf(0.0f, fmaxf(tb.y - q.y, q.y - tb.w));
        const bool nq = fmaf(ex, ex, ey * ey) <= tg.z;
        f2 sw0 = 0ull, swz0 = 0ull, sw1 = 0ull, swz1 = 0ull;
#pragma unroll 1
        for (int h = 0; h < kParts; ++h) {
            const int u = t * kParts + h, b = u % kBufs;
            TRACE_T0(c0);
            mbar_wait(&sm.tfull[g * kBufs + b], (u / kBufs) & 1);
            TRACE_ADD(wf, c0);
            TRACE_T0(c1);
            tc_fence_after();
            const uint32_t ta = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + (g * kBufs + b) * kN;
            far_tmem_part<MODE>(ta, nf + kNZH * kWeightTile + h * kN, cls, qc,
                                &sm.tempty[g * kBufs + b], lane, sw0, swz0, sw1, swz1);
#if AIDW_TC_TRACE
            tmem_hold_f2(sw0, swz0, sw1, swz1);
#endif
            TRACE_ADD(tpart, c1);
        }
        TRACE_T0(c3);
        if (!nq) {
            float w0, w1, z0, z1;
            up2(add2(sw0, sw1), w0, w1);
            up2(add2(swz0, swz1), z0, z1);
            SW += (static_cast<double>(w0) + static_cast<double>(w1)) * m0;
            SWZ += (static_cast<double>(z0) + static_cast<double>(z1)) * m0;
        }
        if (!AIDW_TC_NONEAR_DEBUG && __any_sync(0xFFFFFFFFu, valid && nq)) {
            double nw = 0.0, nz = 0.0;
            if (MODE == kClsMixed) near_tile_any(cls, nf, q, qc, nw, nz);
            else near_tile<MODE>(nf, q, qc, nw, nz);
            if (nq) SW += nw, SWZ += nz;
        }
        // every lane releases the stage after its own reads (an arrival by
        // lane 0 after __syncwarp is as correct — the release is cumulative —
        // but racecheck does not see it; same K4 time,
        // profiles/r02/tc_release_s47.txt)
        mbar_arrive(&sm.bempty[s]);
        if (t + 2 < T) {  // A(t + 2): the MMAs of tile t (its last readers) are complete
            TRACE_T0(c4);
            build_a(myabuf + (t & 1) * kABytes, r, q, __ldg(a.tile_geo + t0 + t + 2));
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.afull[g * 2 + (t & 1)]);
            TRACE_ADD(tbuild, c4);
        }
        TRACE_ADD(ttile, c3);
    }
#if AIDW_TC_TRACE
    if (TRACE_CTA && lane == 0)
        printf("epi g%d q%d: total %lld  wait tfull %lld  parts %lld  tile tail %lld (A rows %lld)\n",
               g, quarter, clock64() - tall, wf, tpart, ttile, tbuild);
#endif
}

__global__ void __launch_bounds__(kTcThreads, 1) weight_tc_kernel(TcArgs a) {
    extern __shared__ __align__(1024) char smem_raw[];
    const unsigned chunk = blockIdx.y;
    const size_t t0 = static_cast<size_t>(chunk) * a.tiles_per_chunk;
    const size_t t1 = t0 + a.tiles_per_chunk < a.tiles ? t0 + a.tiles_per_chunk : a.tiles;
    const int T = t1 > t0 ? static_cast<int>(t1 - t0) : 0;
    // class regions of the slab (device counts, no host sync): CTAs
    // [0, ctas_g) take the general queries, the rest the recipe queries
    const size_t num_a = static_cast<size_t>(a.scan_a[a.n - 1]) + a.flag_a[a.n - 1];
    const size_t num_g = a.n - num_a;
    const size_t g0 = a.s0, g1 = a.s1 < num_g ? a.s1 : num_g;
    const size_t r0 = a.s0 > num_g ? a.s0 : num_g, r1 = a.s1;
    const size_t ctas_g = g1 > g0 ? (g1 - g0 + kCtaQ - 1) / kCtaQ : 0;
    const size_t bx = blockIdx.x;
    if (bx >= ctas_g && (r1 <= r0 || (bx - ctas_g) * kCtaQ >= r1 - r0)) return;
    const bool recipe = bx >= ctas_g;
    if (!(a.classes & (recipe ? 2u : 1u))) return;  // that region runs on the other engine
    const size_t q0 = recipe ? r0 + (bx - ctas_g) * kCtaQ : g0 + bx * kCtaQ;
    const size_t q1 = recipe ? r1 : g1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp >> 2, quarter = warp & 3;
    const size_t pos = q0 + static_cast<size_t>(g) * 128 + quarter * 32 + lane;
    const bool valid = warp < kEpiWarps && pos < q1;
    const size_t ldp = a.s1 - a.s0;
    if (T == 0) {  // a chunk past the data: zero partials
        if (valid) a.part[static_cast<size_t>(chunk) * ldp + (pos - a.s0)] = make_double2(0.0, 0.0);
        return;
    }

    Smem sm = carve(smem_raw);
    if (warp == kCtlWarp) tmem_alloc<kTmemCols>(sm.tmem_slot);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.bfull[s], 1);
            mbar_init(&sm.bempty[s], kGroups + kEpiWarps * 32);
        }
        for (int i = 0; i < 2 * kGroups; ++i) mbar_init(&sm.afull[i], 4);
        for (int i = 0; i < kBufs * kGroups; ++i) {
            mbar_init(&sm.tfull[i], 1);
            mbar_init(&sm.tempty[i], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *sm.tmem_slot;

    if (warp == kCtlWarp) {
        issuer(sm, tbase, T);
    } else if (warp == kProdWarp) {
        if (lane == 0) producer(a, sm, t0, T);
    } else {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 par = make_float4(recipe ? kCodeA4 : -1.0f, 0.f, 1.f, recipe ? kCodeA4 : 0.f);
        if (valid) q = a.qhl[pos], par = a.qpar[pos];
        int cls;
        if (recipe) {
            cls = par.w == kCodeA2 ? kClsA2 : par.w == kCodeA1 ? kClsA1 : par.w == kCodeA3 ? kClsA3
                                                                                       : kClsA4;
        } else {
            cls = kClsG;  // (the CUDA-core engine's G1 / G2 query split does not apply)
        }
        QConst qc;
        qc.c = bc2(recipe ? 0.0f : par.x);
        qc.b = bc2(recipe ? 0.0f : par.y);
        qc.s = bc2(par.z);
        // far alpha = 4 sums are s-free: rescale by s^-2 (a power of two: exact)
        const double m0 = cls == kClsA4 ? 1.0 / (static_cast<double>(par.z) * par.z) : 1.0;
        const unsigned present = __reduce_or_sync(0xFFFFFFFFu, valid ? 1u << cls : 0u);
        const int mode = present == 0u ? (recipe ? kClsA4 : kClsG)
                       : (present & (present - 1u)) ? kClsMixed
                                                     : __ffs(present) - 1;
        // A rows of the first two tiles
        char* myabuf = sm.abuf + g * 2 * kABytes;
        const int r = quarter * 32 + lane;
        for (int t = 0; t < 2 && t < T; ++t) {
            build_a(myabuf + t * kABytes, r, q, __ldg(a.tile_geo + t0 + t));
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.afull[g * 2 + t]);
        }
        double SW = 0.0, SWZ = 0.0;
        switch (mode) {
            case kClsA4: epilogue<kClsA4>(a, sm, tbase, t0, T, g, quarter, lane, valid, q, cls, qc, m0, SW, SWZ); break;
            case kClsA2: epilogue<kClsA2>(a, sm, tbase, t0, T, g, quarter, lane, valid, q, cls, qc, m0, SW, SWZ); break;
            case kClsA1: epilogue<kClsA1>(a, sm, tbase, t0, T, g, quarter, lane, valid, q, cls, qc, m0, SW, SWZ); break;
            case kClsA3: epilogue<kClsA3>(a, sm, tbase, t0, T, g, quarter, lane, valid, q, cls, qc, m0, SW, SWZ); break;
            case kClsG: epilogue<kClsG>(a, sm, tbase, t0, T, g, quarter, lane, valid, q, cls, qc, m0, SW, SWZ); break;
            default: epilogue<kClsMixed>(a, sm, tbase, t0, T, g, quarter, lane, valid, q, cls, qc, m0, SW, SWZ); break;
        }
        if (valid) a.part[static_cast<size_t>(chunk) * ldp + (pos - a.s0)] = make_double2(SW, SWZ);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kCtlWarp) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tbase);
    }
}

}  // namespace

// ------------------------------------------------------------ host side
size_t weight_tc_record_bytes(size_t tiles) { return tiles * kRecBytes; }

void weight_tc_records(const float* rec, const float4* tile_geo, size_t tiles, size_t m,
                       char* tc_rec, cudaStream_t s) {
    LAUNCH(tc_records_kernel, tiles, kWeightTile, 0, s, rec, tile_geo, m, tc_rec);
}

void weight_tc_launch(const WeightTcLaunch& l, cudaStream_t s) {
    CK(cudaFuncSetAttribute(weight_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(kSmemBytes)));
    TcArgs a{l.tc_rec, l.tiles, l.tiles_per_chunk, l.qhl, l.qpar, l.n, l.flag_a, l.scan_a,
             l.s0, l.s1, l.part, l.tile_box, l.tile_geo, l.classes};
    dim3 grid(ceil_div(l.s1 - l.s0, static_cast<size_t>(kCtaQ)) + 1, l.chunks);
    LAUNCH(weight_tc_kernel, grid, kTcThreads, kSmemBytes, s, a);
}

}  // namespace aidwb
