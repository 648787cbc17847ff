// tmem_bench.cu — microbenchmarks behind K4's tensor-core far form:
//   ld   : tcgen05.ld (32x32b.xN) throughput, W warps per SM, one CTA per SM
//   math : the alpha = 4 paired-reciprocal epilogue on register values
//          (8 f32x2 ops + 2 MUFU.RCP per 4 pairs), W warps per SM
//   both : tcgen05.ld feeding the epilogue (no MMA), loads double-buffered
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1601_05904_b200/csrc tools/tmem_bench.cu -o /tmp/tmem_bench
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

__device__ __forceinline__ void epi32(const uint32_t (&v)[32], const float* zz, f2& sw0, f2& swz0,
                                      f2& sw1, f2& swz1) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
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

// quad form: four points on one reciprocal (far pairs: d2 >= 1e-4, so the
// product of four d2^2 stays inside FP32); lanes = two quads, TMEM column
// pairs (2c, 2c + 1) = point c of quad 0 / of quad 1
__device__ __forceinline__ void epi32q(const uint32_t (&v)[32], const float* zz, f2& sw0, f2& swz0,
                                       f2& sw1, f2& swz1) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const float4 Za = *reinterpret_cast<const float4*>(zz + j);
        const float4 Zb = *reinterpret_cast<const float4*>(zz + j + 4);
        f2 A[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const f2 d = pk2(__uint_as_float(v[j + 2 * i]), __uint_as_float(v[j + 2 * i + 1]));
            A[i] = mul2(d, d);
        }
        const f2 p01 = mul2(A[0], A[1]), p23 = mul2(A[2], A[3]);
        const f2 r = rcp2(mul2(p01, p23));
        const f2 S = fma2(add2(A[0], A[1]), p23, mul2(add2(A[2], A[3]), p01));
        const f2 t01 = fma2(A[1], pk2(Za.x, Za.y), mul2(A[0], pk2(Za.z, Za.w)));
        const f2 t23 = fma2(A[3], pk2(Zb.x, Zb.y), mul2(A[2], pk2(Zb.z, Zb.w)));
        const f2 T = fma2(p23, t01, mul2(p01, t23));
        if (j & 8) {
            sw1 = fma2(S, r, sw1);
            swz1 = fma2(T, r, swz1);
        } else {
            sw0 = fma2(S, r, sw0);
            swz0 = fma2(T, r, swz0);
        }
    }
}

// tcgen05.ld into w, ordered after every prior use of v (v passes through
// the asm), so work on v can be scheduled between this load and its wait
__device__ __forceinline__ void tmem_ld32_after(uint32_t taddr, uint32_t (&w)[32], uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%64];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
          "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]),
          "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]),
          "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31]),
          "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
          "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
          "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
          "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_after(f2& a, f2& b, f2& c, f2& d) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+l"(a), "+l"(b), "+l"(c), "+l"(d)::"memory");
}

// pipe microbenchmarks: 8 independent chains per thread, 32 ops per chain per iteration
template <int OP>
__global__ void pipe_kernel(int iters, float* out) {
    float x[8];
    f2 y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1.0f + 0.01f * (threadIdx.x + i), y[i] = pk2(x[i], x[i] + 0.5f);
    const f2 c = pk2(0.999f, 0.998f), d = pk2(1e-4f, 2e-4f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 32; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) x[i] = __int_as_float(__float_as_int(mufu_rcp(x[i])) ^ 1);
                else if (OP == 1) y[i] = fma2(y[i], c, d);
                else if (OP == 3) y[i] = mul2(y[i], c);
                else if (OP == 4) y[i] = add2(y[i], d);
                else if (OP == 5) x[i] = __int_as_float(__float_as_int(x[i]) ^ 1);
                else x[i] = fmaf(x[i], 0.999f, 1e-4f);
            }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float a, b;
        up2(y[i], a, b);
        s += x[i] + a + b;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void runp(const char* name, int warps, int iters, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    pipe_kernel<OP><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(e0);
    pipe_kernel<OP><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = 148.0 * warps * 32 * 256.0 * iters;  // thread-instructions
    printf("%-6s warps/SM %2d: %.3f ms, %.2f thread-instr/SM-clk (%.2f warp-instr/SM-clk)\n", name, warps,
           ms, ops / (ms * 1e-3) / (148.0 * clk * 1e3), ops / 32 / (ms * 1e-3) / (148.0 * clk * 1e3));
}

// MODE 0: ld only (tree XOR), 1: math only, 2: ld + math (double-buffered);
// +10: quad-reciprocal math
template <int MODE_>
__global__ void bench_kernel(int iters, float* out) {
    constexpr int MODE = MODE_ % 10;
    constexpr bool QUAD = MODE_ >= 10;
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) float z[512];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 512; i += blockDim.x) z[i] = 0.001f * i;
    if (MODE != 1 && warp == 0) tmem_alloc<512>(&s_tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = MODE != 1 ? s_tmem : 0u;
    const uint32_t ta = tb + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    // initialise this warp's TMEM lanes (4 warps per lane quarter share; fine)
    if (MODE != 1) {
        for (int c = 0; c < 512; c += 1) {
            const uint32_t val = __float_as_uint(1.0f + 0.001f * (c + lane));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(val)
                         : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    f2 sw0 = 0ull, swz0 = 0ull, sw1 = 0ull, swz1 = 0ull;
    uint32_t acc = 0;
    uint32_t v[32], w[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = w[j] = __float_as_uint(1.0f + 0.01f * (j + lane));
    const int base = (warp >> 2) * 128;  // warps sharing a lane quarter read different columns
    if (MODE == 2 || MODE == 3) {
        tmem_ld32(ta + base, v);
        tmem_wait_ld();
        tmem_hold(v);
    }
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = base + ((it * 32) & 127);
        if (MODE == 0) {
            tmem_ld32(ta + col, v);
            tmem_wait_ld();
            tmem_hold(v);
#pragma unroll
            for (int s = 16; s > 0; s >>= 1)
#pragma unroll
                for (int j = 0; j < s; ++j) v[j] ^= v[j + s];
            acc += v[0];
        } else if (MODE == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] ^= (it & 1);
            if (QUAD) epi32q(v, z + ((it * 32) & 255), sw0, swz0, sw1, swz1); else epi32(v, z + ((it * 32) & 255), sw0, swz0, sw1, swz1);
        } else if (MODE == 3) {
            // forced overlap: ping-pong buffers, load of the next chunk issued
            // before this chunk's math, waited after it
            tmem_ld32_after(ta + base + (((it + 1) * 32) & 127), w, v);
            if (QUAD) epi32q(v, z + ((it * 32) & 255), sw0, swz0, sw1, swz1); else epi32(v, z + ((it * 32) & 255), sw0, swz0, sw1, swz1);
            tmem_wait_after(sw0, swz0, sw1, swz1);
            tmem_hold(w);
            ++it;
            tmem_ld32_after(ta + base + (((it + 1) * 32) & 127), v, w);
            if (QUAD) epi32q(w, z + ((it * 32) & 255), sw0, swz0, sw1, swz1); else epi32(w, z + ((it * 32) & 255), sw0, swz0, sw1, swz1);
            tmem_wait_after(sw0, swz0, sw1, swz1);
            tmem_hold(v);
        } else {
            // next chunk in flight while this one is processed
            tmem_ld32(ta + base + (((it + 1) * 32) & 127), w);
            if (QUAD) epi32q(v, z + ((it * 32) & 255), sw0, swz0, sw1, swz1); else epi32(v, z + ((it * 32) & 255), sw0, swz0, sw1, swz1);
            tmem_wait_ld();
            tmem_hold(w);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = w[j];
        }
    }
    float a0, a1, b0, b1, c0, c1, d0, d1;
    up2(sw0, a0, a1), up2(swz0, b0, b1), up2(sw1, c0, c1), up2(swz1, d0, d1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + b0 + b1 + c0 + c1 + d0 + d1 + acc;
    tc_fence_before();
    __syncthreads();
    if (MODE != 1 && warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tb);
    }
}

template <int MODE>
void run(const char* name, int warps, int iters, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    bench_kernel<MODE><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(e0);
    bench_kernel<MODE><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double vals = 148.0 * warps * 32 * 32.0 * iters;  // one value = one pair
    printf("%-5s warps/SM %2d: %.3f ms, %.2f values(pairs)/SM-clk, %.1f B/SM-clk\n", name, warps, ms,
           vals / (ms * 1e-3) / (148.0 * clk * 1e3), 4.0 * vals / (ms * 1e-3) / (148.0 * clk * 1e3));
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    const int iters = 20000;
    for (int w : {8, 16, 32}) runp<0>("rcp", w, 2000, out);
    for (int w : {8, 16, 32}) runp<1>("ffma2", w, 2000, out);
    for (int w : {8, 16, 32}) runp<2>("ffma", w, 2000, out);
    for (int w : {8, 16, 32}) runp<3>("fmul2", w, 2000, out);
    for (int w : {8, 16, 32}) runp<4>("fadd2", w, 2000, out);
    for (int w : {8, 16, 32}) runp<5>("lop3", w, 2000, out);
    for (int w : {4, 8, 16}) run<0>("ld", w, iters, out);
    for (int w : {4, 8, 16}) run<1>("math", w, iters, out);
    for (int w : {4, 8, 16}) run<2>("both", w, iters, out);
    for (int w : {4, 8, 16}) run<3>("both2", w, iters, out);
    for (int w : {4, 8}) run<11>("mathq", w, iters, out);
    for (int w : {4, 8, 16}) run<12>("bothq", w, iters, out);
    return 0;
}
