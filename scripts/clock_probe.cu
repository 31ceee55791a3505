// clock_probe: SM clock seen by clock64 vs %globaltimer, (a) one spinning warp on an idle GPU,
// (b) one warp per SM spinning while every other warp of the CTA runs FFMA (load).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(long long spin, long long *out, int load) {
  long long c0 = clock64(), g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (threadIdx.x < 32) {
    while (clock64() - c0 < spin) {}
  } else if (load) {
    float a = threadIdx.x, b = 1.0001f;
    for (long long i = 0; i < spin / 8; ++i) a = a * b + 0.5f;
    if (a == 0.f) out[2] = 1;
  }
  __syncthreads();
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = c1 - c0; out[1] = g1 - g0; }
}
int main() {
  long long *d, h[3];
  cudaMalloc(&d, 3 * sizeof(long long));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int load = 0; load < 2; ++load) {
    for (int rep = 0; rep < 3; ++rep) {
      probe<<<load ? sms : 1, load ? 1024 : 32>>>(200000000LL, d, load);
      cudaMemcpy(h, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
      printf("%s: %lld cycles in %lld ns -> %.3f GHz\n", load ? "all SMs, FFMA load" : "one warp, idle", h[0], h[1],
             (double)h[0] / h[1]);
    }
  }
  return 0;
}
