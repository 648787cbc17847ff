// ldtm_probe.cu — what limits the tensor-core K4 epilogue: does a
// tcgen05.ld stream overlap with FP32 (FMA pipe) and MUFU (XU) math, or do
// they serialise?  One CTA per SM, W warps, TMEM filled once; every mode
// reads / computes C values per warp-iteration.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1601_05904_b200/csrc tools/ldtm_probe.cu -o /tmp/ldtm_probe
//
// Modes (values = TMEM columns read per thread, i.e. (query, point) pairs):
//   fma     : 4 FP32 lane-ops per value (2 FFMA2 per 2 values)
//   mufu    : 0.5 MUFU.RCP per value
//   a4      : the alpha = 4 paired form (4 FP32 + 0.5 MUFU per value)
//   ld+X    : tcgen05.ld x64 (+ wait) feeding X
//   lds+X   : X fed from shared memory (16 LDS.128 per 64 values) instead
#include <cuda_runtime.h>

#include <cstdio>

#include "tc.cuh"

using namespace aidwb::tc;
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
__device__ __forceinline__ float rcp(float x) {
    float r;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ f2 rcp2(f2 v) {
    float lo, hi;
    up2(v, lo, hi);
    return pk2(rcp(lo), rcp(hi));
}

enum { kLd = 0, kFma = 1, kMufu = 2, kA4 = 3, kFmaInd = 4, kFmaSc = 5, kA4S = 6, kA4Q = 7 };

// consumers of 64 values
template <int OP>
__device__ __forceinline__ void consume(const uint32_t (&v)[64], const float* z, f2 (&acc)[4]) {
#pragma unroll
    for (int j = 0; j < 64; j += 4) {
        const f2 d01 = pk2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
        const f2 d23 = pk2(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        f2& s0 = acc[(j >> 2) & 1];
        f2& s1 = acc[2 + ((j >> 2) & 1)];
        if (OP == kLd) {
            s0 ^= d01 ^ d23;  // integer (ALU), 2 ops / 4 values
        } else if (OP == kFma) {  // 16 lane-ops / 4 values
            s0 = fma2(d01, d01, s0);
            s1 = fma2(d23, d23, s1);
            s0 = fma2(d01, d23, s0);
            s1 = fma2(d23, d01, s1);
            s0 = fma2(s1, d01, s0);
            s1 = fma2(s0, d23, s1);
            s0 = fma2(d01, s1, s0);
            s1 = fma2(d23, s0, s1);
        } else if (OP == kMufu) {  // 2 MUFU / 4 values (+1 FADD2 to consume)
            const float4 Z = *reinterpret_cast<const float4*>(z + j);
            s0 = add2(s0, pk2(rcp(__uint_as_float(v[j]) + Z.x), rcp(__uint_as_float(v[j + 2]) + Z.y)));
        } else if (OP == kFmaInd) {  // 8 FFMA2 / 4 values, register operands, 4 chains
            acc[0] = fma2(d01, d23, acc[0]);
            acc[1] = fma2(d23, d01, acc[1]);
            acc[2] = fma2(d01, d01, acc[2]);
            acc[3] = fma2(d23, d23, acc[3]);
            acc[0] = fma2(acc[1], d01, acc[0]);
            acc[1] = fma2(acc[2], d23, acc[1]);
            acc[2] = fma2(acc[3], d01, acc[2]);
            acc[3] = fma2(acc[0], d23, acc[3]);
        } else if (OP == kFmaSc) {  // the same lane-ops as scalar FFMA
            float a[8], x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) up2(acc[i], a[2 * i], a[2 * i + 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = __uint_as_float(v[j + i]);
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = fmaf(x[(i + r) & 3], x[(i + 2 * r + 1) & 3], a[i]);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = pk2(a[2 * i], a[2 * i + 1]);
        } else if (OP == kA4S) {  // alpha = 4 paired form in scalar ops
            const float4 Z = *reinterpret_cast<const float4*>(z + j);
            float w[4], zz[4] = {Z.x, Z.y, Z.z, Z.w}, a[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) up2(acc[i], a[2 * i], a[2 * i + 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = __uint_as_float(v[j + i]) * __uint_as_float(v[j + i]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float A = w[h], B = w[h + 2];
                const float R = rcp(A * B);
                const int o = ((j >> 2) & 1) * 2 + h;
                a[o] = fmaf(R, A + B, a[o]);
                a[4 + o] = fmaf(R, fmaf(B, zz[h], A * zz[h + 2]), a[4 + o]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = pk2(a[2 * i], a[2 * i + 1]);
        } else if (OP == kA4Q) {  // four points on one reciprocal (8 values per step)
            if (j & 4) continue;
            const float4 Za = *reinterpret_cast<const float4*>(z + j);
            const float4 Zb = *reinterpret_cast<const float4*>(z + j + 4);
            const f2 d45 = pk2(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
            const f2 d67 = pk2(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
            const f2 A0 = mul2(d01, d01), A1 = mul2(d23, d23), A2 = mul2(d45, d45), A3 = mul2(d67, d67);
            const f2 p01 = mul2(A0, A1), p23 = mul2(A2, A3);
            const f2 r = rcp2(mul2(p01, p23));
            const f2 S = fma2(add2(A0, A1), p23, mul2(add2(A2, A3), p01));
            const f2 t01 = fma2(A1, pk2(Za.x, Za.y), mul2(A0, pk2(Za.z, Za.w)));
            const f2 t23 = fma2(A3, pk2(Zb.x, Zb.y), mul2(A2, pk2(Zb.z, Zb.w)));
            const f2 T = fma2(p23, t01, mul2(p01, t23));
            s0 = fma2(S, r, s0);
            s1 = fma2(T, r, s1);
        } else {  // alpha = 4 paired reciprocal, the K4 far form
            const float4 Z = *reinterpret_cast<const float4*>(z + j);
            const f2 A = mul2(d01, d01), B = mul2(d23, d23);
            const f2 R = rcp2(mul2(A, B));
            s0 = fma2(R, add2(A, B), s0);
            s1 = fma2(R, fma2(B, pk2(Z.x, Z.y), mul2(A, pk2(Z.z, Z.w))), s1);
        }
    }
}

// SRC: 0 = registers perturbed per iteration (no load), 1 = TMEM (tcgen05.ld x64),
// 2 = shared memory (LDS.128)
template <int SRC, int OP>
__global__ void __launch_bounds__(512, 1) probe(int iters, float* out) {
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) float z[1024];
    __shared__ __align__(16) uint32_t sv[16][64 * 8];  // per-warp LDS source
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) z[i] = 0.001f * i;
    for (int i = lane; i < 64 * 8; i += 32)
        sv[warp][i] = __float_as_uint(1.0f + 0.001f * i);
    if (SRC == 1 && warp == 0) tmem_alloc<512>(&s_tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = SRC == 1 ? s_tmem : 0u;
    const uint32_t ta = tb + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    if (SRC == 1 && warp < 4) {
        for (int c = 0; c < 512; ++c) {
            const uint32_t val = __float_as_uint(1.0f + 0.001f * (c + lane));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(val)
                         : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    f2 acc[4] = {0ull, 0ull, 0ull, 0ull};
    uint32_t v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = __float_as_uint(1.0f + 0.01f * (j + lane));
    const uint32_t base = ((warp >> 2) & 3) * 128;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        if (SRC == 1) {
            tmem_ld64(ta + base + ((it * 64) & 127), v);
            tmem_wait_ld();
            tmem_hold(v);
        } else if (SRC == 2) {
            const uint32_t* p = &sv[warp][(it & 7) * 64];
#pragma unroll
            for (int j = 0; j < 64; j += 4) {
                const uint4 u = *reinterpret_cast<const uint4*>(p + j);
                v[j] = u.x, v[j + 1] = u.y, v[j + 2] = u.z, v[j + 3] = u.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 64; j += 16) v[j] ^= static_cast<uint32_t>(it);  // 4 ALU / 64 values
            tmem_hold(v);
        }
        consume<OP>(v, z + ((it * 64) & 511), acc);
    }
    float a, b, s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) up2(acc[i], a, b), s += a + b;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    tc_fence_before();
    __syncthreads();
    if (SRC == 1 && warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tb);
    }
}

template <int SRC, int OP>
void run(const char* name, int warps, int iters, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    probe<SRC, OP><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(e0);
    probe<SRC, OP><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double clk_hz = 1965e6;
    const double vals = 148.0 * warps * 32 * 64.0 * iters;
    printf("%-10s warps/SM %2d: %8.3f ms, %6.2f values/SM-clk\n", name, warps, ms,
           vals / (ms * 1e-3) / (148.0 * clk_hz));
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    const int iters = 4000;
    for (int w : {8, 12, 16}) {
        run<1, kFma>("ld+fma", w, iters, out);
        run<2, kFma>("lds+fma", w, iters, out);
        run<2, kMufu>("lds+mufu", w, iters, out);
        run<1, kMufu>("ld+mufu", w, iters, out);
        run<1, kA4>("ld+a4", w, iters, out);
        run<2, kA4>("lds+a4", w, iters, out);
        run<2, kFmaInd>("lds+fmaind", w, iters, out);
        run<2, kFmaSc>("lds+fmasc", w, iters, out);
        run<1, kA4S>("ld+a4s", w, iters, out);
        run<1, kA4Q>("ld+a4q", w, iters, out);
    }
    return 0;
}
