// Microbenchmark of B2's elementwise body per element pair (no memory): x = s*c + t;
// P = ex2(l*k + x); dS = P*(dp - D); pack P and dS to bf16x2.  Variants:
//   0: scalar FFMA/FADD/FMUL, ALU pack (IADD + PRMT)     1: scalar, cvt.rn.bf16x2 pack
//   2: f32x2 FFMA/FADD/FMUL, cvt pack                     3: f32x2, ALU pack
// Reports cycles per element pair per warp (8 independent pairs per iteration).
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void uf2(uint64_t r, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pk_alu(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t pk_cvt(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

template <int MODE>
__global__ void bench(uint32_t *out, int iters, long long *cyc) {
  float s[16], dp[16];
  for (int z = 0; z < 16; ++z) {
    s[z] = threadIdx.x * 1e-4f + z * 0.01f;
    dp[z] = 0.5f - z * 0.02f;
  }
  const float c = 0.25f, k = -1.4426950408889634f;
  float t = 0.125f, l = 1.5f, D = 0.3f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pp[8], dd[8];
    if (MODE <= 1) {
#pragma unroll
      for (int z = 0; z < 16; z += 2) {
        float P[2], S[2];
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const float x = fmaf(s[z + w], c, t);
          P[w] = ex2(fmaf(l, k, x));
          S[w] = P[w] * (dp[z + w] - D);
        }
        pp[z / 2] = MODE == 0 ? pk_alu(P[0], P[1]) : pk_cvt(P[0], P[1]);
        dd[z / 2] = MODE == 0 ? pk_alu(S[0], S[1]) : pk_cvt(S[0], S[1]);
      }
    } else {
      const uint64_t c2 = f2(c, c), t2 = f2(t, t), l2 = f2(l, l), k2 = f2(k, k), D2 = f2(D, D);
#pragma unroll
      for (int z = 0; z < 16; z += 2) {
        const uint64_t x = fma2(f2(s[z], s[z + 1]), c2, t2);
        uint64_t a = fma2(l2, k2, x);
        float a0, a1;
        uf2(a, a0, a1);
        const uint64_t P = f2(ex2(a0), ex2(a1));
        const uint64_t S = mul2(P, sub2(f2(dp[z], dp[z + 1]), D2));
        float p0, p1, s0, s1;
        uf2(P, p0, p1);
        uf2(S, s0, s1);
        pp[z / 2] = MODE == 2 ? pk_cvt(p0, p1) : pk_alu(p0, p1);
        dd[z / 2] = MODE == 2 ? pk_cvt(s0, s1) : pk_alu(s0, s1);
      }
    }
#pragma unroll
    for (int z = 0; z < 8; ++z) acc ^= pp[z] + dd[z];
    // perturb inputs so nothing is loop invariant
#pragma unroll
    for (int z = 0; z < 16; ++z) s[z] = __uint_as_float(__float_as_uint(s[z]) ^ (acc & 1));
    t += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t *out;
  long long *cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMallocManaged(&cyc, 148 * 8);
  const char *names[] = {"scalar + alu pack", "scalar + cvt pack", "f32x2 + cvt pack", "f32x2 + alu pack"};
  for (int mode = 0; mode < 4; ++mode)
    for (int threads : {128, 256}) {
      const int iters = 4000;
      void (*kf)(uint32_t *, int, long long *) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : bench<3>;
      kf<<<148, threads>>>(out, iters, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      // per SMSP: threads/128 warps, 8 pairs per iteration each
      const double pairs_per_smsp = 8.0 * iters * (threads / 128.0);
      printf("%-20s threads %4d: %.2f cycles per element pair per SMSP (%s)\n", names[mode], threads,
             (double)cyc[0] / pairs_per_smsp, cudaGetErrorString(e));
    }
  return 0;
}
