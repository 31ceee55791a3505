// Throughput microbenchmark of the XU (MUFU) pipe vs FMA-pipe alternatives on sm_100a.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>

template <int MODE>
__global__ void bench(float *out, int iters, long long *cyc) {
  float a0 = threadIdx.x * 1e-3f - 3.f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 - 0.1f, a5 = a0 - 0.2f, a6 = a0 - 0.3f, a7 = a0 - 0.4f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // ex2.approx.ftz.f32
#define EX(x) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x))
      EX(a0); EX(a1); EX(a2); EX(a3); EX(a4); EX(a5); EX(a6); EX(a7);
    } else if (MODE == 1) {  // cvt.rn.bf16x2.f32
      uint32_t r;
#define CV(x, y) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x), "f"(y)); acc ^= r
      CV(a0, a1); CV(a2, a3); CV(a4, a5); CV(a6, a7); CV(a1, a0); CV(a3, a2); CV(a5, a4); CV(a7, a6);
    } else if (MODE == 2) {  // ex2.approx.f16x2
      uint32_t h0 = __float_as_uint(a0), h1 = __float_as_uint(a1), h2 = __float_as_uint(a2), h3 = __float_as_uint(a3);
#define EH(x) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x))
      EH(h0); EH(h1); EH(h2); EH(h3); EH(h0); EH(h1); EH(h2); EH(h3);
      acc ^= h0 ^ h1 ^ h2 ^ h3;
    } else if (MODE == 3) {  // FFMA throughput reference (8 independent chains)
#define FM(x) asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0f3A800000;" : "+f"(x))
      FM(a0); FM(a1); FM(a2); FM(a3); FM(a4); FM(a5); FM(a6); FM(a7);
    } else if (MODE == 4) {  // packed fma.rn.f32x2 (sm_100)
      uint64_t p0, p1, p2, p3;
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p0) : "f"(a0), "f"(a1));
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p1) : "f"(a2), "f"(a3));
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p2) : "f"(a4), "f"(a5));
      asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p3) : "f"(a6), "f"(a7));
#define F2(x) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x))
      F2(p0); F2(p1); F2(p2); F2(p3); F2(p0); F2(p1); F2(p2); F2(p3);
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(p0));
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a2), "=f"(a3) : "l"(p1));
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a4), "=f"(a5) : "l"(p2));
      asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a6), "=f"(a7) : "l"(p3));
    } else if (MODE == 5) {  // F2F f32 -> bf16 single (cvt.rn.bf16.f32)
      uint16_t r;
#define C1(x) asm volatile("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(x)); acc ^= r
      C1(a0); C1(a1); C1(a2); C1(a3); C1(a4); C1(a5); C1(a6); C1(a7);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + acc;
}

int main() {
  float *out;
  long long *cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMallocManaged(&cyc, 148 * 8);
  const char *names[] = {"ex2.approx.ftz.f32", "cvt.rn.bf16x2.f32", "ex2.approx.f16x2", "fma.rn.f32", "fma.rn.f32x2",
                         "cvt.rn.bf16.f32"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int threads : {256, 1024}) {
      int iters = 2000;
      void (*k)(float *, int, long long *) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : mode == 3 ? bench<3> : mode == 4 ? bench<4> : bench<5>;
      k<<<148, threads>>>(out, iters, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      double ops = 8.0 * iters * threads;  // per SM (one block per SM)
      printf("%-22s threads %4d: %.2f ops/clk/SM (%s)\n", names[mode], threads, ops / (double)cyc[0], cudaGetErrorString(e));
    }
  }
  return 0;
}
