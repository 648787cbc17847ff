// mma_latency.cu — issue-to-completion latency of K4's tensor-core step (one
// M128 N64 K16 kind::tf32 tcgen05.mma pair + tcgen05.commit -> mbarrier),
// alone and while W epilogue-like warps stream tcgen05.ld.x64 (+ optional
// FP32 math) from other TMEM columns of the same CTA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1601_05904_b200/csrc tools/mma_latency.cu -o /tmp/mma_latency
#include <cuda_runtime.h>

#include <cstdio>

#include "tc.cuh"

using namespace aidwb::tc;

constexpr int kReps = 2000;

template <int LOADERS, bool MATH>
__global__ void __launch_bounds__(512, 1) lat_kernel(unsigned long long* out, float* sink) {
    __shared__ __align__(1024) char ops[8192 + 4096];
    __shared__ uint64_t bar;
    __shared__ uint32_t s_tmem;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (8192 + 4096) / 4; i += blockDim.x)
        reinterpret_cast<float*>(ops)[i] = 0.0f;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        stop = 0;
    }
    if (warp == 0) tmem_alloc<512>(&s_tmem);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = s_tmem;
    if (warp == 0) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, 64);
            const uint32_t a0 = smem_u32(ops), b0 = smem_u32(ops + 8192);
            unsigned long long total = 0, mx = 0;
            for (int r = 0; r < kReps; ++r) {
                const unsigned long long c0 = clock64();
                mma_tf32(tb, smem_desc(a0, kKChunkBytes, kRowGroupBytes),
                         smem_desc(b0, kKChunkBytes, kRowGroupBytes), idesc, false);
                mma_tf32(tb, smem_desc(a0 + 2 * kKChunkBytes, kKChunkBytes, kRowGroupBytes),
                         smem_desc(b0 + 2 * kKChunkBytes, kKChunkBytes, kRowGroupBytes), idesc, true);
                mma_commit(&bar);
                mbar_wait(&bar, r & 1);
                const unsigned long long dt = clock64() - c0;
                total += dt;
                mx = dt > mx ? dt : mx;
            }
            stop = 1;
            if (blockIdx.x == 0) out[0] = total / kReps, out[1] = mx;
        }
    } else if (warp <= LOADERS) {
        // streamers: TMEM columns 64..511 of their lane quarter
        const uint32_t ta = tb + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        float acc = 0.f;
        int it = 0;
        while (!stop) {
            uint32_t v[64];
            tmem_ld64(ta + 64 + ((it * 64) % 448), v);
            tmem_wait_ld();
            tmem_hold(v);
            if (MATH) {
#pragma unroll
                for (int j = 0; j < 64; j += 2)
                    acc = fmaf(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), acc);
            } else {
                acc += __uint_as_float(v[0] ^ v[63]);
            }
            ++it;
        }
        sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tb);
    }
}

template <int L, bool M>
void run(const char* name, unsigned long long* d, float* sink) {
    lat_kernel<L, M><<<148, 512>>>(d, sink);
    cudaDeviceSynchronize();
    lat_kernel<L, M><<<148, 512>>>(d, sink);
    unsigned long long h[2];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("%-28s mean %llu cycles, max %llu %s\n", name, h[0], h[1],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 16);
    cudaMalloc(&sink, 148 * 512 * 4);
    run<0, false>("alone", d, sink);
    run<4, false>("4 ld warps", d, sink);
    run<12, false>("12 ld warps", d, sink);
    run<12, true>("12 ld+math warps", d, sink);
    run<15, true>("15 ld+math warps", d, sink);
    return 0;
}
