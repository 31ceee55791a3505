// TMEM access latency: cycles from tcgen05.ld / st issue to tcgen05.wait completion (one warp per
// quarter, everything else idle), and with 16 warps hammering.
#include <stdint.h>
#include <stdio.h>
#include "na2d_sm100.cuh"
using namespace na2d::sm100;

__global__ void k(long long *out, int busy) {
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) done = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  if (warp < 4) {
    uint32_t r[16];
    long long tl = 0, ts = 0, tl2 = 0;
    for (int it = 0; it < 64; ++it) {
      long long t0 = clock64();
      tmem_ld16(la + (it % 8) * 16, r);
      tc_wait_ld();
      long long t1 = clock64();
      r[0] += it;
      tmem_st16(la + 256 + (it % 8) * 16, r);
      tc_wait_st();
      long long t2 = clock64();
      uint32_t h[8];
      tmem_ld_h8<6>(la + (it % 8) * 16, h);
      tc_wait_ld();
      long long t3 = clock64();
      r[1] += h[3];
      tl += t1 - t0;
      ts += t2 - t1;
      tl2 += t3 - t2;
    }
    if (lane == 0) {
      out[warp * 3] = tl / 64;
      out[warp * 3 + 1] = ts / 64;
      out[warp * 3 + 2] = tl2 / 64;
    }
    if (r[0] == 12345) out[100] = r[1];
    __syncwarp();
    if (warp == 0 && lane == 0) done = 1;
  } else if (busy) {
    uint32_t r[16];
    uint32_t acc = 0;
    while (!done) {
      tmem_ld16(la + 128 + (warp % 8) * 16, r);
      tc_wait_ld();
      acc += r[2];
      tmem_st16(la + 384 + (warp % 8) * 16, r);
    }
    tc_wait_st();
    if (acc == 77) out[101] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  long long *d, h[16];
  cudaMalloc(&d, 1024 * 8);
  for (int busy = 0; busy < 2; ++busy) {
    k<<<148, busy ? 640 : 128>>>(d, busy);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("busy=%d (%s): ld.x16 %lld cyc, st.x16 %lld cyc, ld.16x32bx2.x8 %lld cyc\n", busy, cudaGetErrorString(e), h[0],
           h[1], h[2]);
  }
  return 0;
}
