// The forward's real per-tile tensor-core sequence at L = 7 (one CTA per SM, one issuing thread):
//   QK: 4 SS MMAs (M=64, N=240, K=16; two sub-tiles at TMEM lane offsets 0 / 16) into S [0, 240)
//   PV: 30 K-steps x 2 sub-tiles TS MMAs (M=64, N=32, K=16; A = P at [240, 360)) into OACC chains
// Reports cycles per tile for QK only, PV only and both, for OACC = 1, 2, 4.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2204_07143_b200/csrc -I include
#include <stdint.h>
#include <stdio.h>

#include "na2d_sm100.cuh"
using namespace na2d::sm100;

template <bool QK, bool PV, int OACC, int KSTEPS>
__global__ void seq(int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t &bar = *(uint64_t *)(smem + 100 * 1024);
  uint32_t &slot = *(uint32_t *)(smem + 100 * 1024 + 8);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u;
    x ^= x >> 13;
    ((uint32_t *)smem)[i] = (x & 0x807f807fu) | 0x3f003f00u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t iqk = idesc_bf16(64, 240, false), ipv = idesc_bf16(64, 32, true);
    const uint32_t q = smem_u32(smem), k = q + 8192, v = q + 8192 + 21504 + 1024;
    const uint64_t dq = sdesc_sw64(q), dk = sdesc_sw64(k), dv = sdesc_sw64(v);
    const uint32_t d0 = tmem, d1 = d0 + (16u << 16);
    const uint32_t b0 = tmem + 240, b1 = b0 + (16u << 16);
    const uint32_t o0 = tmem + 360, o1 = o0 + (16u << 16);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        if (QK) {
          mma_ss(d0, dq, dk, iqk, 0);
          mma_ss(d1, dq + (4096 >> 4), dk + ((4 * 24 * 64) >> 4), iqk, 0);
          mma_ss(d0, dq + 2, dk + 2, iqk, 1);
          mma_ss(d1, dq + ((4096 + 32) >> 4), dk + ((4 * 24 * 64 + 32) >> 4), iqk, 1);
        }
        if (PV) {
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const uint32_t voff = (ks * 16 * 64) >> 4, oc = (ks % OACC) * 32;
            const uint32_t a = ks >= OACC ? 1u : 0u;
            mma_ts(o0 + oc, b0 + ks * 4, dv + voff, ipv, a);
            mma_ts(o1 + oc, b1 + ks * 4, dv + ((4 * 24 * 64) >> 4) + voff, ipv, a);
          }
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <bool QK, bool PV, int OACC, int KSTEPS = 30>
void run(const char *name) {
  long long *cyc, host[148];
  cudaMalloc(&cyc, 148 * 8);
  auto kf = seq<QK, PV, OACC, KSTEPS>;
  cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  const int iters = 400;
  kf<<<148, 128, 110 * 1024>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, cyc, sizeof(host), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += host[i];
  printf("%-34s %7.1f cyc/tile (%s)\n", name, m / 148 / iters, cudaGetErrorString(e));
}

int main() {
  run<true, false, 1>("QK only");
  run<false, true, 1>("PV only, OACC 1");
  run<false, true, 2>("PV only, OACC 2");
  run<false, true, 4>("PV only, OACC 4");
  run<true, true, 1>("QK + PV, OACC 1");
  run<true, true, 4>("QK + PV, OACC 4");
  run<false, true, 4, 15>("PV 15 K-steps, OACC 4");
  return 0;
}
