// weight_ops.cuh — arithmetic shared by the FP32 weighting engines (K4 on
// the CUDA cores, weight.cu, and K4 with the far-form d2 on the tensor cores,
// weight_tc.cu): MUFU wrappers, packed f32x2 operations, the FMA-pipe exp2,
// the data-tile record layout and the recipe class codes.  Each query's
// arithmetic is written once here, so both engines evaluate a (query, point)
// pair with the same roundings for a given form.
#pragma once

#include <cstdint>

#include "weight.cuh"

namespace aidwb {
namespace wops {

constexpr int kTileFloats = 9 * kWeightTile;  // SoA tile, 9 components (see kComps)

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

// SoA components of a 256-record data tile:
//   near form  x_hi y_hi x_lo y_lo z_hi z_lo   (unit-box coordinates, hi/lo)
//   far form   px2 = -2 p'x, py2 = -2 p'y, pp = |p'|^2 with p' = p - c, c the
//              tile's centre — d2 = |q'|^2 + px2 q'x + py2 q'y + pp in 3 FP32
//              ops per pair; z_hi is shared with the near form
enum : int { kXH, kYH, kXL, kYL, kZH, kZL, kPX, kPY, kPP, kComps };
static_assert(kComps * kWeightTile == kTileFloats, "tile layout");


// Recipe class codes (qpar.x / qpar.w of a recipe query; general classes: 0, 2).
constexpr float kCodeA4 = 1.0f, kCodeA2 = 3.0f, kCodeA1 = 4.0f, kCodeA3 = 5.0f;

// ---- packed f32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2): two queries per
// 64-bit register pair; each lane rounds exactly like the scalar op, so a
// query's result does not depend on which lane / pair it occupies.
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2 bc2(float v) { return pk2(v, v); }
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
__device__ __forceinline__ f2 rcp2(f2 v) {
    float lo, hi;
    up2(v, lo, hi);
    return pk2(mufu_rcp(lo), mufu_rcp(hi));
}

__device__ __forceinline__ float mufu_rsq(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ f2 rsq2(f2 v) {
    float lo, hi;
    up2(v, lo, hi);
    return pk2(mufu_rsq(lo), mufu_rsq(hi));
}

__device__ __forceinline__ f2 cube2(f2 r) { return mul2(mul2(r, r), r); }

// exp2 on the FMA pipe for class-G2 queries (x <= ~0 after ratio scaling):
// Cody-Waite split x = n + f, n = rint(x) via the 1.5 * 2^23 magic add,
// f in [-0.5, 0.5], 2^f by a degree-5 near-minimax fit (max rel. error
// 1.9e-7 incl. FP32 Horner rounding, on par with MUFU.EX2; the degree-6 fit
// (9.7e-8) cost 2.5 % of the general path for no measurable accuracy),
// 2^n added into the exponent.
// Arguments clamp at -125 (results < 2^-125 are ~0 relative to the leading
// weight, which is 1).  Scalar and packed forms round identically.
constexpr float kExpMagic = 12582912.0f;  // 1.5 * 2^23
constexpr float kE0 = 1.0f, kD1 = 0.6931470036506653f, kD2 = 0.24022242426872253f,
                kD3 = 0.05550733581185341f, kD4 = 0.009671512991189957f,
                kD5 = 0.001326472731307149f;

__device__ __forceinline__ float exp2_fma(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + kExpMagic;
    const float f = x - (t - kExpMagic);
    float p = fmaf(kD5, f, kD4);
    p = fmaf(p, f, kD3);
    p = fmaf(p, f, kD2);
    p = fmaf(p, f, kD1);
    p = fmaf(p, f, kE0);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ f2 exp2_fma2(f2 x) {
    float lo, hi;
    up2(x, lo, hi);
    const f2 xc = pk2(fmaxf(lo, -125.0f), fmaxf(hi, -125.0f));
    const f2 m = bc2(kExpMagic);
    const f2 t = add2(xc, m);
    const f2 f = sub2(xc, sub2(t, m));
    f2 p = fma2(bc2(kD5), f, bc2(kD4));
    p = fma2(p, f, bc2(kD3));
    p = fma2(p, f, bc2(kD2));
    p = fma2(p, f, bc2(kD1));
    p = fma2(p, f, bc2(kE0));
    float plo, phi, tlo, thi;
    up2(p, plo, phi);
    up2(t, tlo, thi);
    return pk2(__int_as_float(__float_as_int(plo) + (__float_as_int(tlo) << 23)),
               __int_as_float(__float_as_int(phi) + (__float_as_int(thi) << 23)));
}

}  // namespace wops
}  // namespace aidwb
