// Does a tcgen05.mma kind::f16 with an f16 accumulator (instruction-descriptor D format 0) pack two
// results per 32-bit TMEM column?  M = 128, N = 64, K = 16: A = ones, B[n][k] = (n + 1) / 64 for k = 0
// and 0 otherwise, so D[m][n] = (n + 1) / 64.  TMEM columns [0, 64) of lane 0 are printed raw: fp32
// results fill 64 columns; packed fp16 pairs would fill 32 columns and leave [32, 64) untouched (0).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdio.h>

#include "na2d_sm100.cuh"
using namespace na2d::sm100;

__device__ void store_sw32(uint8_t *base, int row, int col, __half v) {  // 16 halves per row, SW32
  const int chunk = (col * 2) / 16, within = (col * 2) % 16;
  const int pos = chunk ^ ((row >> 2) & 1);
  *(__half *)(base + row * 32 + pos * 16 + within) = v;
}

__global__ void k(uint32_t *out, int dfmt) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[64 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * 16; i += blockDim.x) store_sw32(sa, i / 16, i % 16, __float2half(1.f));
  for (int i = tid; i < 64 * 16; i += blockDim.x)
    store_sw32(sb, i / 16, i % 16, __float2half((i % 16) == 0 ? (i / 16 + 1) / 64.f : 0.f));
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  {
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 128; c += 32) tmem_st32_zero(addr + c);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      // kind::f16: D format bits [4,6): 0 = f16, 1 = f32; A/B fp16 (format 0); N / 8, M / 16
      const uint32_t id = ((uint32_t)dfmt << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      mma_ss(tmem, sdesc_sw<32>(smem_u32(sa)), sdesc_sw<32>(smem_u32(sb)), id, 0);
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t r[32];
    tmem_ld32(tmem, r);
    tc_wait_ld();
    if (tid == 0)
      for (int z = 0; z < 32; ++z) out[z] = r[z];
    tmem_ld32(tmem + 32, r);
    tc_wait_ld();
    if (tid == 0)
      for (int z = 0; z < 32; ++z) out[32 + z] = r[z];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

int main() {
  uint32_t *d, h[64];
  cudaMalloc(&d, 64 * 4);
  for (int dfmt = 1; dfmt >= 0; --dfmt) {
    cudaMemset(d, 0, 64 * 4);
    k<<<1, 128>>>(d, dfmt);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("D format %s (%s): ", dfmt ? "f32" : "f16", cudaGetErrorString(e));
    for (int z = 0; z < 64; ++z) {
      if (dfmt) printf("%.4f ", *(float *)&h[z]);
      else {
        __half lo, hi;
        *(uint16_t *)&lo = h[z] & 0xffff;
        *(uint16_t *)&hi = h[z] >> 16;
        printf("[%.4f %.4f] ", __half2float(lo), __half2float(hi));
      }
    }
    printf("\n");
  }
  return 0;
}
