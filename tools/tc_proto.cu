// tc_proto.cu — prototype / microbenchmark of K4's far form on the 5th-gen
// tensor cores: d2 = |q'|^2 - 2 q'.p' + |p'|^2 (tile-centred) as one
// kind::tf32 tcgen05 MMA per (128 queries x 128 points) with exact hi/mid/lo
// TF32 pieces (K = 16), accumulator in TMEM; the epilogue warps read d2 with
// tcgen05.ld and run the alpha = 4 paired-reciprocal sums.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I paper_1601_05904_b200/csrc tools/tc_proto.cu -o /tmp/tc_proto
//   /tmp/tc_proto [n_queries] [tiles]
//
// Reports: d2 accuracy against FP64 on far pairs, sums against an FP64
// reference on sampled queries, pairs / SM-clock.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace aidwb::tc;

#define CKP(x)                                                                               \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                         \
        }                                                                                    \
    } while (0)

constexpr int kTilePts = 256;
#ifndef PROTO_N
#define PROTO_N 128
#endif
#ifndef PROTO_GROUPS
#define PROTO_GROUPS 2
#endif
constexpr int kN = PROTO_N;          // MMA N (tile part)
constexpr int kParts = 256 / kN;     // MMA parts per tile
constexpr int kM = 128;              // MMA M (queries per group)
constexpr int kGroups = PROTO_GROUPS;  // query groups per CTA (same B operand)
constexpr int kStages = 4;
constexpr uint32_t kBBytes = kTilePts * kK * 4;   // 16 KB
constexpr uint32_t kZBytes = kTilePts * 4;        // 1 KB
constexpr uint32_t kRecBytes = kBBytes + kZBytes;
constexpr uint32_t kABytes = kM * kK * 4;         // 8 KB
constexpr int kEpiWarps = 4 * kGroups;
#ifndef PROTO_CTRL
#define PROTO_CTRL 2
#endif
constexpr int kCtrlWarps = PROTO_CTRL;  // 2: producer + MMA warps; 1: one warp does both
constexpr int kThreads = (kEpiWarps + kCtrlWarps) * 32;
constexpr int kMmaWarp = kEpiWarps + kCtrlWarps - 1;
constexpr int kCtaQ = kM * kGroups;

typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void up2(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
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
__device__ __forceinline__ float mufu_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ f2 rcp2(f2 v) {
    float lo, hi;
    up2(v, lo, hi);
    return pk2(mufu_rcp(lo), mufu_rcp(hi));
}

// A row (query side) for one tile centre: 16 tf32 values in operand layout.
__device__ __forceinline__ void build_a(char* abuf, int r, float4 q, float2 c) {
    const float fx = (q.x - c.x) + q.z;
    const float fy = (q.y - c.y) + q.w;
    const float fq = fmaf(fx, fx, fy * fy);
    const float xh = tf32_hi(fx), xr = fx - xh, xm = tf32_hi(xr), xl = xr - xm;
    const float yh = tf32_hi(fy), yr = fy - yh, ym = tf32_hi(yr), yl = yr - ym;
    const float qh = tf32_hi(fq), qr = fq - qh, qm = tf32_hi(qr), ql = qr - qm;
    const float a[16] = {xh, xh, xm, xm, xl, yh, yh, ym, ym, yl, qh, qm, ql, 1.0f, 1.0f, 0.0f};
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
        float4* p = reinterpret_cast<float4*>(abuf + operand_offset(r, 4 * c4));
        *p = make_float4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
    }
}

struct Args {
    const char* rec;
    const float2* cgeo;
    const float4* qhl;
    int n, tiles;
    double2* out;
    float* dump;  // d2 of tile 0, n x 256 (or null)
    int mode;     // 0 full, 1 TMEM loads only
};

#ifndef PROTO_SINGLE
#define PROTO_SINGLE 0
#endif
#ifndef PROTO_C
#define PROTO_C 32
#endif
constexpr int kC = PROTO_C;  // TMEM columns per load
template <int C>
__device__ __forceinline__ void ldc(uint32_t ta, uint32_t (&v)[C]) {
    if constexpr (C == 128) tmem_ld128(ta, v);
    else if constexpr (C == 64) tmem_ld64(ta, v);
    else if constexpr (C == 32) tmem_ld32(ta, v);
    else tmem_ld16(ta, v);
}
template <int C>
__device__ __forceinline__ void ldc_after(uint32_t ta, uint32_t (&w)[C], uint32_t (&v)[C]) {
    if constexpr (C == 32) tmem_ld32_after(ta, w, v);
    else if constexpr (C == 16) tmem_ld16_after(ta, w, v);
}
// alpha = 4 far sums of C columns: w0 + w2 = (a0 + a2) rcp(a0 a2), ...
template <int C>
__device__ __forceinline__ void epi32(const uint32_t (&v)[C], const float* zz, f2& sw0, f2& swz0,
                                      f2& sw1, f2& swz1) {
#pragma unroll
    for (int j = 0; j < C; j += 8) {
        const float4 Za = *reinterpret_cast<const float4*>(zz + j);
        const float4 Zb = *reinterpret_cast<const float4*>(zz + j + 4);
        {
            const f2 d01 = pk2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
            const f2 d23 = pk2(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
            const f2 A = mul2(d01, d01), B = mul2(d23, d23);
            const f2 rr = rcp2(mul2(A, B));
            sw0 = fma2(rr, add2(A, B), sw0);
            swz0 = fma2(rr, fma2(B, pk2(Za.x, Za.y), mul2(A, pk2(Za.z, Za.w))), swz0);
        }
        {
            const f2 d01 = pk2(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
            const f2 d23 = pk2(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
            const f2 A = mul2(d01, d01), B = mul2(d23, d23);
            const f2 rr = rcp2(mul2(A, B));
            sw1 = fma2(rr, add2(A, B), sw1);
            swz1 = fma2(rr, fma2(B, pk2(Zb.x, Zb.y), mul2(A, pk2(Zb.z, Zb.w))), swz1);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 1) far_tc_kernel(Args a) {
    extern __shared__ __align__(1024) char smem[];
    char* stage = smem;                                   // kStages x kRecBytes
    char* abuf = smem + kStages * kRecBytes;              // [group][2] x kABytes
    uint64_t* bar = reinterpret_cast<uint64_t*>(abuf + 2 * kGroups * kABytes);
    uint64_t *bfull = bar, *bempty = bar + kStages;
    uint64_t* afull = bar + 2 * kStages;                  // [group][2]
    uint64_t* tfull = afull + 2 * kGroups;                // [group][half]
    uint64_t* tempty = tfull + 2 * kGroups;               // [group][half]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2 * kGroups);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kMmaWarp) tmem_alloc<512>(s_tmem);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bfull[s], 1), mbar_init(&bempty[s], 1 + kEpiWarps);
        for (int i = 0; i < 2 * kGroups; ++i) {
            mbar_init(&afull[i], 4);
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *s_tmem;
    const int T = a.tiles;

    if (kCtrlWarps == 2 && warp == kEpiWarps) {  // ---- producer
        if (lane == 0) {
            for (int t = 0; t < T; ++t) {
                const int s = t % kStages;
                if (t >= kStages) mbar_wait(&bempty[s], ((t / kStages) - 1) & 1);
                mbar_expect_tx(&bfull[s], kRecBytes);
                bulk_load(stage + s * kRecBytes, a.rec + static_cast<size_t>(t) * kRecBytes, kRecBytes,
                          &bfull[s]);
            }
        }
    } else if (warp == kMmaWarp) {  // ---- MMA issuer (and producer with one control warp)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(kM, kN);
            if (kCtrlWarps == 1)
                for (int t = 0; t < kStages && t < T; ++t) {
                    mbar_expect_tx(&bfull[t], kRecBytes);
                    bulk_load(stage + t * kRecBytes, a.rec + static_cast<size_t>(t) * kRecBytes, kRecBytes,
                              &bfull[t]);
                }
            for (int t = 0; t < T; ++t) {
                const int s = t % kStages;
                mbar_wait(&bfull[s], (t / kStages) & 1);
                for (int g = 0; g < kGroups; ++g) mbar_wait(&afull[g * 2 + (t & 1)], (t >> 1) & 1);
                tc_fence_after();
                const uint32_t b0 = smem_u32(stage + s * kRecBytes);
                for (int h = 0; h < kParts; ++h) {
                    if (kCtrlWarps == 1 && h == kParts / 2 && t >= 1 && t - 1 + kStages < T) {
                        // tile t - 1 consumed by every warp: refill its stage
                        const int tp = t - 1, sp = tp % kStages;
                        mbar_wait(&bempty[sp], (tp / kStages) & 1);
                        mbar_expect_tx(&bfull[sp], kRecBytes);
                        bulk_load(stage + sp * kRecBytes, a.rec + static_cast<size_t>(tp + kStages) * kRecBytes,
                                  kRecBytes, &bfull[sp]);
                    }
                    const uint32_t bh = b0 + h * (kN / 8) * kRowGroupBytes;
                    const int u = t * kParts + h, b = u & 1;
                    for (int g = 0; g < kGroups; ++g) {
                        if (u >= 2) mbar_wait(&tempty[g * 2 + b], ((u >> 1) - 1) & 1);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(abuf + (g * 2 + (t & 1)) * kABytes);
                        const uint32_t d = tbase + (g * 2 + b) * kN;
                        mma_tf32(d, smem_desc(a0, kKChunkBytes, kRowGroupBytes),
                                 smem_desc(bh, kKChunkBytes, kRowGroupBytes), idesc, false);
                        mma_tf32(d, smem_desc(a0 + 2 * kKChunkBytes, kKChunkBytes, kRowGroupBytes),
                                 smem_desc(bh + 2 * kKChunkBytes, kKChunkBytes, kRowGroupBytes), idesc,
                                 true);
                        mma_commit(&tfull[g * 2 + b]);
                    }
                }
                mma_commit(&bempty[s]);
            }
        }
    } else {  // ---- epilogue: one query per thread (TMEM lane)
        const int g = warp >> 2, quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const int qi = blockIdx.x * kCtaQ + g * kM + r;
        const float4 q = qi < a.n ? a.qhl[qi] : make_float4(0.f, 0.f, 0.f, 0.f);
        char* myabuf = abuf + g * 2 * kABytes;
        for (int t = 0; t < 2 && t < T; ++t) {
            build_a(myabuf + t * kABytes, r, q, a.cgeo[t]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&afull[g * 2 + t]);
        }
        double SW = 0.0, SWZ = 0.0;
        for (int t = 0; t < T; ++t) {
            const int s = t % kStages;
            const float* z = reinterpret_cast<const float*>(stage + s * kRecBytes + kBBytes);
            f2 sw0 = 0ull, swz0 = 0ull, sw1 = 0ull, swz1 = 0ull;
            for (int h = 0; h < kParts; ++h) {
                const int u = t * kParts + h, b = u & 1;
                mbar_wait(&tfull[g * 2 + b], (u >> 1) & 1);
                tc_fence_after();
                const uint32_t ta =
                    tbase + (static_cast<uint32_t>(quarter * 32) << 16) + (g * 2 + b) * kN;
                const float* zh = z + h * kN;
#if PROTO_SINGLE
                {
                    uint32_t v[kN];
                    ldc<kN>(ta, v);
                    tmem_wait_ld();
                    tmem_hold(v);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[g * 2 + b]);
                    epi32<kN>(v, zh, sw0, swz0, sw1, swz1);
                }
                continue;
#endif
                uint32_t v[kC], w[kC];
                ldc<kC>(ta, v);
                tmem_wait_ld();
                tmem_hold(v);
                if (a.dump && t == 0 && qi < a.n) {
                    for (int c = 0; c < kN / 32; ++c) {
                        uint32_t uu[32];
                        tmem_ld32(ta + 32 * c, uu);
                        tmem_wait_ld();
                        tmem_hold(uu);
                        for (int j = 0; j < 32; ++j)
                            a.dump[static_cast<size_t>(qi) * kTilePts + h * kN + c * 32 + j] =
                                __uint_as_float(uu[j]);
                    }
                }
                // kC-column chunks, the next load in flight during each chunk's sums
#pragma unroll
                for (int c = 0; c + 2 < kN / kC; c += 2) {
                    ldc_after<kC>(ta + kC * (c + 1), w, v);
                    epi32<kC>(v, zh + kC * c, sw0, swz0, sw1, swz1);
                    tmem_wait_ld_after(sw0, swz0, sw1, swz1);
                    tmem_hold(w);
                    ldc_after<kC>(ta + kC * (c + 2), v, w);
                    epi32<kC>(w, zh + kC * (c + 1), sw0, swz0, sw1, swz1);
                    tmem_wait_ld_after(sw0, swz0, sw1, swz1);
                    tmem_hold(v);
                }
                ldc_after<kC>(ta + kN - kC, w, v);
                epi32<kC>(v, zh + kN - 2 * kC, sw0, swz0, sw1, swz1);
                tmem_wait_ld_after(sw0, swz0, sw1, swz1);
                tmem_hold(w);
                // TMEM reads of this part are complete: release it to the MMA
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[g * 2 + b]);
                epi32<kC>(w, zh + kN - kC, sw0, swz0, sw1, swz1);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bempty[s]);
            float a0, a1, b0, b1;
            up2(add2(sw0, sw1), a0, a1);
            up2(add2(swz0, swz1), b0, b1);
            SW += static_cast<double>(a0) + a1;
            SWZ += static_cast<double>(b0) + b1;
            if (t + 2 < T) {
                build_a(myabuf + (t & 1) * kABytes, r, q, a.cgeo[t + 2]);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[g * 2 + (t & 1)]);
            }
        }
        if (qi < a.n) a.out[qi] = make_double2(SW, SWZ);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<512>(tbase);
    }
}

// ---------------------------------------------------------------- host
static float tf32_hi_h(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}
static void split2(double v, float& h, float& l) {
    h = tf32_hi_h(static_cast<float>(v));
    l = tf32_hi_h(static_cast<float>(v - h));
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 148 * 2 * 128 * 4;
    const int T = argc > 2 ? atoi(argv[2]) : 1024;
    const int G = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(T))));
    std::mt19937_64 rng(42);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<double> px(static_cast<size_t>(T) * kTilePts), py(px.size()), pz(px.size());
    std::vector<char> rec(static_cast<size_t>(T) * kRecBytes, 0);
    std::vector<float2> cgeo(T);
    for (int t = 0; t < T; ++t) {
        const double x0 = (t % G) / static_cast<double>(G), y0 = (t / G) / static_cast<double>(G);
        float bx0 = 1e30f, by0 = 1e30f, bx1 = -1e30f, by1 = -1e30f;
        for (int j = 0; j < kTilePts; ++j) {
            const size_t i = static_cast<size_t>(t) * kTilePts + j;
            px[i] = x0 + U(rng) / G, py[i] = y0 + U(rng) / G, pz[i] = U(rng) * 2.0 - 1.0;
            bx0 = std::min(bx0, static_cast<float>(px[i])), bx1 = std::max(bx1, static_cast<float>(px[i]));
            by0 = std::min(by0, static_cast<float>(py[i])), by1 = std::max(by1, static_cast<float>(py[i]));
        }
        const float cx = 0.5f * (bx0 + bx1), cy = 0.5f * (by0 + by1);
        cgeo[t] = make_float2(cx, cy);
        char* R = rec.data() + static_cast<size_t>(t) * kRecBytes;
        for (int j = 0; j < kTilePts; ++j) {
            const size_t i = static_cast<size_t>(t) * kTilePts + j;
            const double ppx = px[i] - cx, ppy = py[i] - cy;
            float xh, xl, yh, yl, ph, pl;
            split2(-2.0 * ppx, xh, xl);
            split2(-2.0 * ppy, yh, yl);
            split2(ppx * ppx + ppy * ppy, ph, pl);
            const float b[16] = {xh, xl, xh, xl, xh, yh, yl, yh, yl, yh, 1.f, 1.f, 1.f, ph, pl, 0.f};
            for (int k = 0; k < 16; ++k) memcpy(R + operand_offset(j, k), &b[k], 4);
            const float zf = static_cast<float>(pz[i]);
            memcpy(R + kBBytes + 4 * j, &zf, 4);
        }
    }
    std::vector<float4> qhl(n);
    std::vector<double> qx(n), qy(n);
    for (int i = 0; i < n; ++i) {
        qx[i] = U(rng), qy[i] = U(rng);
        const float xh = static_cast<float>(qx[i]), yh = static_cast<float>(qy[i]);
        qhl[i] = make_float4(xh, yh, static_cast<float>(qx[i] - xh), static_cast<float>(qy[i] - yh));
    }
    char* d_rec;
    float2* d_c;
    float4* d_q;
    double2* d_out;
    float* d_dump;
    CKP(cudaMalloc(&d_rec, rec.size()));
    CKP(cudaMalloc(&d_c, T * sizeof(float2)));
    CKP(cudaMalloc(&d_q, n * sizeof(float4)));
    CKP(cudaMalloc(&d_out, n * sizeof(double2)));
    CKP(cudaMalloc(&d_dump, static_cast<size_t>(n) * kTilePts * 4));
    CKP(cudaMemcpy(d_rec, rec.data(), rec.size(), cudaMemcpyHostToDevice));
    CKP(cudaMemcpy(d_c, cgeo.data(), T * sizeof(float2), cudaMemcpyHostToDevice));
    CKP(cudaMemcpy(d_q, qhl.data(), n * sizeof(float4), cudaMemcpyHostToDevice));
    const size_t smem = kStages * kRecBytes + 2 * kGroups * kABytes + 32 * 8 + 16;
    CKP(cudaFuncSetAttribute(far_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int ctas = (n + kCtaQ - 1) / kCtaQ;
    Args args{d_rec, d_c, d_q, n, T, d_out, d_dump, 0};
    far_tc_kernel<<<ctas, kThreads, smem>>>(args);
    CKP(cudaGetLastError());
    CKP(cudaDeviceSynchronize());
    // d2 accuracy on tile 0, far pairs (box distance > 0.3 diag)
    std::vector<float> dump(static_cast<size_t>(n) * kTilePts);
    CKP(cudaMemcpy(dump.data(), d_dump, dump.size() * 4, cudaMemcpyDeviceToHost));
    {
        double bx0 = 1e30, by0 = 1e30, bx1 = -1e30, by1 = -1e30;
        for (int j = 0; j < kTilePts; ++j)
            bx0 = std::min(bx0, px[j]), bx1 = std::max(bx1, px[j]), by0 = std::min(by0, py[j]), by1 = std::max(by1, py[j]);
        const double diag = std::hypot(bx1 - bx0, by1 - by0);
        double emax = 0.0, esum = 0.0;
        long cnt = 0, bad = 0;
        for (int i = 0; i < n; ++i) {
            const double ex = std::max(0.0, std::max(bx0 - qx[i], qx[i] - bx1));
            const double ey = std::max(0.0, std::max(by0 - qy[i], qy[i] - by1));
            if (std::hypot(ex, ey) <= 0.3 * diag) continue;
            for (int j = 0; j < kTilePts; ++j) {
                const double dx = px[j] - qx[i], dy = py[j] - qy[i];
                const double d2 = dx * dx + dy * dy;
                const double e = std::fabs(dump[static_cast<size_t>(i) * kTilePts + j] - d2) / d2;
                if (!(e < 1e-3)) ++bad;
                emax = std::max(emax, e), esum += e, ++cnt;
            }
        }
        printf("d2 (tile 0, %ld far pairs): max rel err %.3e, mean %.3e, %ld bad\n", cnt, emax,
               esum / std::max(1L, cnt), bad);
    }
    // sums on sampled queries vs FP64 (far form for every pair: near pairs
    // are excluded from the check by sampling queries inside tile-free space
    // is not possible here, so compare with the same FP64 all-pairs sum and
    // report the relative difference of sum w)
    std::vector<double2> out(n);
    CKP(cudaMemcpy(out.data(), d_out, n * sizeof(double2), cudaMemcpyDeviceToHost));
    {
        double emax = 0.0;
        for (int s = 0; s < 64; ++s) {
            const int i = (s * 7919) % n;
            double sw = 0.0, swz = 0.0;
            for (size_t j = 0; j < px.size(); ++j) {
                const double dx = px[j] - qx[i], dy = py[j] - qy[i];
                const double d2 = dx * dx + dy * dy;
                const double w = 1.0 / (d2 * d2);
                sw += w, swz += w * pz[j];
            }
            const double e = std::fabs(out[i].y / out[i].x - swz / sw);
            emax = std::max(emax, e);
        }
        printf("prediction (64 queries, all pairs far form): max abs err %.3e\n", emax);
    }
    args.dump = nullptr;
    for (int mode = 0; mode < 1; ++mode) {
    args.mode = mode;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    far_tc_kernel<<<ctas, kThreads, smem>>>(args);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) far_tc_kernel<<<ctas, kThreads, smem>>>(args);
    cudaEventRecord(e1);
    CKP(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double pairs = static_cast<double>(ctas) * kCtaQ * T * kTilePts;
    printf("mode %d n %d tiles %d: %.3f ms, %.1f Gpair/s, %.2f pairs/SM-clk at %d MHz\n", mode, n, T, ms,
           pairs / ms * 1e-6, pairs / (ms * 1e-3) / (148.0 * clk * 1e3), clk / 1000);
    }
    return 0;
}
