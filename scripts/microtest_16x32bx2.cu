// Layout check of tcgen05.ld / st .16x32bx2 (16 TMEM lanes x 2 column blocks per warp).
#include <stdint.h>
#include <stdio.h>

#include "na2d_sm100.cuh"
using namespace na2d::sm100;

__global__ void k(uint32_t *out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // warp w writes its quarter: value = lane_global * 1000 + col for cols [0, 64)
  const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < 64; c += 4) {
    uint32_t v[4];
    for (int z = 0; z < 4; ++z) v[z] = (warp * 32 + lane) * 1000 + c + z;
    tmem_st4(la + c, v);
  }
  tc_wait_st();
  __syncwarp();
  // 16x32bx2 loads: lane base 0 and 16 of the quarter, 4 columns, half split offset 8, from col 2
  uint32_t r0[4], r1[4];
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 8;"
               : "=r"(r0[0]), "=r"(r0[1]), "=r"(r0[2]), "=r"(r0[3]) : "r"(la + 2));
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 8;"
               : "=r"(r1[0]), "=r"(r1[1]), "=r"(r1[2]), "=r"(r1[3]) : "r"(la + ((uint32_t)16 << 16) + 2));
  tc_wait_ld();
  for (int z = 0; z < 4; ++z) {
    out[(warp * 32 + lane) * 8 + z] = r0[z];
    out[(warp * 32 + lane) * 8 + 4 + z] = r1[z];
  }
  // store test: thread writes 7000000 + tid into 16x32bx2.x1 at col 100 (split 4) from lane base 16
  uint32_t sv[1] = {7000000u + threadIdx.x};
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x1.b32 [%0], 4, {%1};" ::"r"(la + ((uint32_t)16 << 16) + 100), "r"(sv[0]) : "memory");
  tc_wait_st();
  uint32_t a[8];
  tmem_ld8(la + 100, a);
  tc_wait_ld();
  for (int z = 0; z < 8; ++z) out[4096 + (warp * 32 + lane) * 8 + z] = a[z];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  uint32_t *d, h[8192];
  cudaMalloc(&d, sizeof(h));
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(e));
  for (int t : {0, 1, 15, 16, 17, 31, 32, 48}) {
    printf("thread %2d ld base0:", t);
    for (int z = 0; z < 4; ++z) printf(" %u", h[t * 8 + z]);
    printf(" | base16:");
    for (int z = 0; z < 4; ++z) printf(" %u", h[t * 8 + 4 + z]);
    printf("\n");
  }
  for (int t : {0, 15, 16, 17, 31}) {
    printf("tmem lane %2d cols 100..107 after st:", t);
    for (int z = 0; z < 8; ++z) printf(" %u", h[4096 + t * 8 + z]);
    printf("\n");
  }
  return 0;
}
