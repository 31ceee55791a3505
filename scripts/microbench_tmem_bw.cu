// TMEM load / store throughput on every SM: W warps (W/4 per sub-partition) loop tcgen05.ld or
// tcgen05.st over their lane quarter.  Reported per sub-partition: cycles per instruction and bytes
// per cycle, to tell a per-instruction cost from a per-byte cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2204_07143_b200/csrc -I include
#include <stdint.h>
#include <stdio.h>

#include "na2d_sm100.cuh"
using namespace na2d::sm100;

constexpr int kIters = 512;

template <int N>
__device__ __forceinline__ void ldN(uint32_t a, uint32_t (&r)[32]) {
  if constexpr (N == 32) tmem_ld32(a, r);
  if constexpr (N == 16) tmem_ld16(a, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
  if constexpr (N == 8) tmem_ld8(a, *reinterpret_cast<uint32_t(*)[8]>(&r[0]));
  if constexpr (N == 4) tmem_ld4(a, *reinterpret_cast<uint32_t(*)[4]>(&r[0]));
  if constexpr (N == 2) tmem_ld2(a, *reinterpret_cast<uint32_t(*)[2]>(&r[0]));
  if constexpr (N == -8) tmem_ld_h8<6>(a, *reinterpret_cast<uint32_t(*)[8]>(&r[0]));
  if constexpr (N == -4) tmem_ld_h4<6>(a, *reinterpret_cast<uint32_t(*)[4]>(&r[0]));
  if constexpr (N == -2) tmem_ld_h2<6>(a, *reinterpret_cast<uint32_t(*)[2]>(&r[0]));
}
template <int N>
__device__ __forceinline__ void stN(uint32_t a, const uint32_t (&r)[32]) {
  if constexpr (N == 16) tmem_st16(a, *reinterpret_cast<const uint32_t(*)[16]>(&r[0]));
  if constexpr (N == 8) tmem_st8(a, *reinterpret_cast<const uint32_t(*)[8]>(&r[0]));
  if constexpr (N == 4) tmem_st4(a, *reinterpret_cast<const uint32_t(*)[4]>(&r[0]));
  if constexpr (N == 2) tmem_st2(a, *reinterpret_cast<const uint32_t(*)[2]>(&r[0]));
  if constexpr (N == 1) tmem_st1(a, r[0]);
  if constexpr (N == -4) tmem_st_h4<6>(a, *reinterpret_cast<const uint32_t(*)[4]>(&r[0]));
  if constexpr (N == -2) tmem_st_h2<6>(a, *reinterpret_cast<const uint32_t(*)[2]>(&r[0]));
  if constexpr (N == -1) tmem_st_h1<6>(a, r[0]);
}

// ST: 0 = loads, 1 = stores.  DEPTH instructions per wait.
template <int ST, int N, int DEPTH>
__global__ void k(long long *out, int nwarps) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4) * 128;
  uint32_t r[32];
#pragma unroll
  for (int z = 0; z < 32; ++z) r[z] = threadIdx.x + z;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        if constexpr (ST) stN<N>(la + d * 32, r);
        else ldN<N>(la + d * 32, r);
      }
      if constexpr (ST) {
        tc_wait_st();
        r[0] += 1;
      } else {
        tc_wait_ld();
        acc += r[0] ^ r[1];
      }
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x % 32 == 0 && warp < nwarps) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 0x12345) out[100000] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int ST, int N, int DEPTH>
void run(long long *d) {
  const int cols = N < 0 ? -N : N;
  const int bytes = 32 * cols * 4;  // per warp instruction (.16x32bx2: 32 threads x cols regs)
  for (int nw : {4, 8, 16}) {
    k<ST, N, DEPTH><<<148, 512>>>(d, nw);
    cudaError_t e = cudaDeviceSynchronize();
    static long long h[148 * 32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < nw; ++w) cyc = cyc > h[b * 32 + w] ? cyc : h[b * 32 + w];
    const double instr_per_smsp = (double)(nw / 4) * DEPTH * kIters;
    printf("%s %-10s x%-2d depth %2d warps %2d: %6.2f cyc/instr/SMSP, %6.1f B/cyc/SM (%s)\n", ST ? "st" : "ld",
           N < 0 ? "16x32bx2" : "32x32b", cols, DEPTH, nw, cyc / instr_per_smsp, 4 * instr_per_smsp * bytes / cyc,
           cudaGetErrorString(e));
  }
}

int main() {
  long long *d;
  cudaMalloc(&d, 200000 * 8);
  run<0, 2, 4>(d);
  run<0, 4, 4>(d);
  run<0, 8, 4>(d);
  run<0, 16, 4>(d);
  run<0, 32, 2>(d);
  run<0, -2, 4>(d);
  run<0, -4, 4>(d);
  run<0, -8, 4>(d);
  run<1, 1, 4>(d);
  run<1, 2, 4>(d);
  run<1, 4, 4>(d);
  run<1, 8, 4>(d);
  run<1, 16, 4>(d);
  run<1, 16, 1>(d);
  run<1, 4, 16>(d);
  run<1, -1, 4>(d);
  run<1, -2, 4>(d);
  run<1, -4, 4>(d);
  return 0;
}
