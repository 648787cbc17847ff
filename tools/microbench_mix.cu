// Issue-mix probe for K4's far loop on sm_100a: how close to the FMA-pipe
// bound does an instruction stream with R packed FP32 ops (FFMA2) per
// MUFU.RCP get, at 2 / 3 / 4 CTAs (16 / 24 / 32 warps) per SM?  K4's alpha = 4
// far loop issues 104 packed FP32 + 24 MUFU per 32 pairs (R = 4.33; FMA pipe
// 208 cycles vs XU 192 per warp-iteration).  Also re-measures MUFU.RCP alone
// (round 1's figure came from a launch that never ran).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbmix microbench_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 2048
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float rcp(float x) {
    float r;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// Per iteration and chain: F packed FMAs then one MUFU.RCP on each lane of
// the chain's pair, 8 independent chains.  F = 0: MUFU only.
template <int F, int M>
__global__ void mix(float* out, float s) {
    u64 p[8];
    float a[8];
    for (int i = 0; i < 8; ++i) {
        const float v = 1.0f + threadIdx.x * 1e-6f + i * 1e-3f;
        p[i] = __float_as_uint(v) | (static_cast<u64>(__float_as_uint(v + 0.5f)) << 32);
        a[i] = v;
    }
    const u64 ps = __float_as_uint(s) | (static_cast<u64>(__float_as_uint(s)) << 32);
    const u64 pc = __float_as_uint(0.25f) | (static_cast<u64>(__float_as_uint(0.25f)) << 32);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int f = 0; f < F; ++f) p[i] = ffma2(p[i], ps, pc);
#pragma unroll
            for (int mm = 0; mm < M; ++mm) a[i] = rcp(a[i] + 1.0f);
        }
    }
    float r = 0;
    for (int i = 0; i < 8; ++i) r += a[i] + __uint_as_float(static_cast<unsigned>(p[i]));
    if (r == 12345.f) out[0] = r;
}
template <int F, int M>
void run(const char* name, int ctas_per_sm, int sms, float* o) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // resident CTAs per SM limited to ctas_per_sm through dynamic shared memory
    const int smem = (220 * 1024) / ctas_per_sm;
    cudaFuncSetAttribute(mix<F, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        mix<F, M><<<sms * ctas_per_sm * 4, 256, smem>>>(o, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        const cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(err));
            return;
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warps = static_cast<double>(sms) * ctas_per_sm * 4 * 8;
        const double fma_cycles_per_warp = static_cast<double>(N_ITER) * 8 * (F * 2 + M);  // FFMA2: 2 cycles, FADD: 1
        const double mufu_cycles_per_warp = static_cast<double>(N_ITER) * 8 * M * 8;  // 8 cycles / warp-instr
        const double cycles = ms * 1e-3 * 1965e6;
        // per SMSP: warps / (4 * sms) warps share the pipes
        const double wps = warps / (4.0 * sms);
        if (rep)
            printf("%-24s ctas/SM %d  %.3f ms  FMA pipe %.2f  XU %.2f  (bound %s)\n", name, ctas_per_sm, ms,
                   wps * fma_cycles_per_warp / cycles, wps * mufu_cycles_per_warp / cycles,
                   F * 2 > M * 8 ? "FMA" : "XU");
    }
}
int main() {
    float* o;
    cudaMalloc(&o, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int c : {2, 3, 4}) {
        run<0, 1>("MUFU.RCP only", c, sms, o);
        run<4, 1>("4 FFMA2 : 1 RCP", c, sms, o);
        run<13, 3>("13 FFMA2 : 3 RCP (K4)", c, sms, o);
        run<5, 1>("5 FFMA2 : 1 RCP", c, sms, o);
        run<8, 1>("8 FFMA2 : 1 RCP", c, sms, o);
        run<16, 0>("FFMA2 only", c, sms, o);
    }
    return 0;
}
