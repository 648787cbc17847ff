// Pipe-throughput probe for K4 design decisions on sm_100a: scalar FFMA vs
// packed FFMA2 (f32x2), FADD2, MUFU.EX2 / RCP / LG2, and mixes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define N_ITER 4096
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float ex2(float x) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rcp(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float lg2(float x) { float r; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

__device__ __forceinline__ double rcp64(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

template <int MODE> __global__ void k(float* out, float s) {
  float a[8]; u64 p[8]; double dd[8]; const double ds = s;
  __half2 hh[8]; const __half2 hs = __float2half2_rn(s);
  for (int i = 0; i < 8; ++i) hh[i] = __float2half2_rn(threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 8; ++i) dd[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; p[i] = __float_as_uint(a[i]) | ((u64)__float_as_uint(a[i] + 1.f) << 32); }
  u64 ps = __float_as_uint(s) | ((u64)__float_as_uint(s) << 32);
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fmaf(a[i], s, 0.5f);                    // FFMA
      if (MODE == 1) p[i] = ffma2(p[i], ps, ps);                     // FFMA2
      if (MODE == 2) p[i] = fadd2(p[i], ps);                         // FADD2
      if (MODE == 3) a[i] = ex2(a[i]);                               // MUFU.EX2
      if (MODE == 4) a[i] = __int_as_float(__float_as_int(rcp(a[i])) ^ 1);  // MUFU.RCP (+ LOP3: rcp(rcp(x)) folds away)
      if (MODE == 5) a[i] = lg2(a[i]);                               // MUFU.LG2
      if (MODE == 6) { p[i] = ffma2(p[i], ps, ps); a[i] = ex2(a[i]); }  // FFMA2 + EX2 mix
      if (MODE == 7) { a[i] = fmaf(a[i], s, 0.5f); a[i] = a[i] + s; }   // FFMA + FADD
      if (MODE == 8) dd[i] = fma(dd[i], ds, 0.5);                    // DFMA
      if (MODE == 9) dd[i] = dd[i] + ds;                             // DADD
      if (MODE == 10) dd[i] = rcp64(dd[i]);                          // MUFU.RCP64H (+ fixup)
      if (MODE == 11) { dd[i] = fma(dd[i], ds, 0.5); p[i] = ffma2(p[i], ps, ps); }  // DFMA + FFMA2
      if (MODE == 12) hh[i] = __hfma2(hh[i], hs, hs);                // HFMA2
      if (MODE == 13) { hh[i] = __hfma2(hh[i], hs, hs); p[i] = ffma2(p[i], ps, ps); }  // HFMA2 + FFMA2
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i] + __uint_as_float((unsigned)p[i]) + (float)dd[i] + __low2float(hh[i]);
  if (r == 12345.f) out[0] = r;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"FFMA", "FFMA2", "FADD2", "MUFU.EX2", "MUFU.RCP", "MUFU.LG2", "FFMA2+EX2", "FFMA+FADD",
                         "DFMA", "DADD", "RCP.F64", "DFMA+FFMA2", "HFMA2", "HFMA2+FFMA2"};
  const int ops[] = {1, 1, 1, 1, 1, 1, 2, 2, 1, 1, 1, 2, 1, 2};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 14; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      dim3 g(sms * 8), b(256);
      cudaEventRecord(e0);
      switch (mode) { case 0: k<0><<<g,b>>>(o,1.0001f); break; case 1: k<1><<<g,b>>>(o,1.0001f); break; case 2: k<2><<<g,b>>>(o,1.0001f); break; case 3: k<3><<<g,b>>>(o,0.5f); break;
        case 4: k<4><<<g,b>>>(o,1.f); break; case 5: k<5><<<g,b>>>(o,1.f); break; case 6: k<6><<<g,b>>>(o,1.0001f); break; case 7: k<7><<<g,b>>>(o,1.0001f); break;
        case 8: k<8><<<g,b>>>(o,1.0001f); break; case 9: k<9><<<g,b>>>(o,1.0001f); break; case 10: k<10><<<g,b>>>(o,1.f); break; case 11: k<11><<<g,b>>>(o,1.0001f); break; case 12: k<12><<<g,b>>>(o,1.0001f); break; case 13: k<13><<<g,b>>>(o,1.0001f); break; }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_instr = (double)sms * 8 * 8 * N_ITER * 8 * ops[mode];  // warps * iters * unroll * ops
      double cycles = ms * 1e-3 * 1965e6;  // assumes max clock
      if (rep) printf("%-10s %8.3f ms  %.2f warp-instr/clk/SM (thread-ops/clk/SM %.1f)\n", names[mode], ms, warp_instr / cycles / sms, 32 * warp_instr / cycles / sms);
    }
  }
  return 0;
}
