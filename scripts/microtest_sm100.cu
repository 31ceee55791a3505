// Microtests of sm_100a behaviour the NA2D kernels rely on (run on the GPU box):
//  1. M=64 tcgen05.mma (SS) D layout: row m -> TMEM lane (m%16) + 32*(m/16) (+16 with a lane
//     offset of 16 in the D address), column n.
//  2. M=64 TS MMA with A (bf16) read from TMEM lanes at offset 16.
//  3. tcgen05.ld .x8/.x4/.x2 at odd/even unaligned column offsets.
//  4. shared-memory fp32 atomic add throughput (distinct addresses per lane, same address).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2204_07143_b200/csrc microtest_sm100.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include "na2d_sm100.cuh"

using namespace na2d::sm100;

// A: 64 x 32 bf16 (K-major, SW64), B: N x 32 bf16 (K-major SW64), D = A B^T (64 x N fp32).
// Write A and B swizzled manually: row r, 16B chunk c stored at chunk c ^ ((r >> 1) & 3).
__device__ void store_sw64(uint8_t *base, int row, int col, __nv_bfloat16 v) {
  int chunk = (col * 2) / 16, within = (col * 2) % 16;
  int pos = chunk ^ ((row >> 1) & 3);
  *(__nv_bfloat16 *)(base + row * 64 + pos * 16 + within) = v;
}

constexpr int N = 64;

__global__ void test_m64(float *outD, float *outD2, const float *A, const float *B, float *outTS, int *ld_ok) {
  __shared__ __align__(1024) uint8_t sa[64 * 64];
  __shared__ __align__(1024) uint8_t sb[N * 64];
  __shared__ __align__(1024) uint8_t sv[64 * 64];  // V: 64 keys x 32 dims (MN-major for TS MMA)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 64 * 32; i += blockDim.x) store_sw64(sa, i / 32, i % 32, __float2bfloat16(A[i]));
  for (int i = tid; i < N * 32; i += blockDim.x) store_sw64(sb, i / 32, i % 32, __float2bfloat16(B[i]));
  // V[key][d] = B[key][d] reused (keys = rows of B), 64 keys
  for (int i = tid; i < 64 * 32; i += blockDim.x) store_sw64(sv, i / 32, i % 32, __float2bfloat16(B[i]));
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // zero columns [0, 256) of all lanes
  {
    uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 256; c += 32) tmem_st32_zero(addr + c);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // 1. two M=64 MMAs: D0 at lane 0 (cols 0..N), D1 at lane 16 (same cols) with A rows permuted? use same A,B
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t id = ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(64 >> 4) << 24));
      for (int k = 0; k < 2; ++k) mma_ss(tmem + 0, sdesc_sw64(smem_u32(sa) + k * 32), sdesc_sw64(smem_u32(sb) + k * 32), id, k);
      // second: B rows shifted by 8 (start at row 8 -> + 512 B), D at lane 16
      for (int k = 0; k < 2; ++k)
        mma_ss(tmem + (16u << 16), sdesc_sw64(smem_u32(sa) + k * 32), sdesc_sw64(smem_u32(sb) + 8 * 64 + k * 32), id, k);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
    tc_wait_ld();
    for (int c = 0; c < 32; ++c) outD[(warp * 32 + lane) * 64 + c] = __uint_as_float(r[c]);
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 32, r);
    tc_wait_ld();
    for (int c = 0; c < 32; ++c) outD[(warp * 32 + lane) * 64 + 32 + c] = __uint_as_float(r[c]);
  }
  // 3. unaligned ld: compare x8 at col 3 / x4 at col 5 / x2 at col 7 with x32 values
  {
    uint32_t full[32], a8[8], a4[4];
    const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16);
    tmem_ld32(base, full);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a8[0]), "=r"(a8[1]), "=r"(a8[2]), "=r"(a8[3]), "=r"(a8[4]), "=r"(a8[5]), "=r"(a8[6]), "=r"(a8[7])
                 : "r"(base + 3));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a4[0]), "=r"(a4[1]), "=r"(a4[2]), "=r"(a4[3])
                 : "r"(base + 21));
    tc_wait_ld();
    int ok = 1;
    for (int c = 0; c < 8; ++c) ok &= a8[c] == full[3 + c];
    for (int c = 0; c < 4; ++c) ok &= a4[c] == full[21 + c];
    ld_ok[warp * 32 + lane] = ok;
  }
  // 2. TS MMA: A = bf16(D) rows from TMEM lanes (offset 16) packed into cols [128, 160):
  //    each thread packs its lane's D[0..63] -> 32 packed cols; then O = A(64x64) * V(64 keys x 32)
  {
    const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16);
    uint32_t r[32];
    tmem_ld32(base, r);
    tc_wait_ld();
    uint32_t pk[8];
    for (int g = 0; g < 2; ++g) {
      for (int c = 0; c < 8; ++c) pk[c] = pack_bf16(__uint_as_float(r[g * 16 + 2 * c]), __uint_as_float(r[g * 16 + 2 * c + 1]));
      tmem_st8(base + 128 + g * 8, pk);
    }
    tmem_ld32(base + 32, r);
    tc_wait_ld();
    for (int g = 0; g < 2; ++g) {
      for (int c = 0; c < 8; ++c) pk[c] = pack_bf16(__uint_as_float(r[g * 16 + 2 * c]), __uint_as_float(r[g * 16 + 2 * c + 1]));
      tmem_st8(base + 144 + g * 8, pk);
    }
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t id = ((1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(64 >> 4) << 24));
      // sub-tile at lane offset 16: O1 at cols 192.. lanes +16, A from lanes +16 cols 128..160
      for (int ks = 0; ks < 4; ++ks)
        mma_ts(tmem + (16u << 16) + 192, tmem + (16u << 16) + 128 + ks * 8, sdesc_sw64(smem_u32(sv) + ks * 1024), id, ks);
      for (int ks = 0; ks < 4; ++ks)
        mma_ts(tmem + 192, tmem + 128 + ks * 8, sdesc_sw64(smem_u32(sv) + ks * 1024), id, ks);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 1);
  tc_fence_after();
  {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 192, r);
    tc_wait_ld();
    for (int c = 0; c < 32; ++c) outTS[(warp * 32 + lane) * 32 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// A (fp16 pairs) from TMEM x B (bf16, smem MN-major): can kind::f16 mix operand types?
__global__ void test_mixed(const float *A, const float *B, float *out, int a_fmt) {
  __shared__ __align__(1024) uint8_t sv[64 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 64 * 32; i += blockDim.x) store_sw64(sv, i / 32, i % 32, __float2bfloat16(B[i]));
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  // row m = lane of quarter: A[m][k] for k < 64, packed fp16 (a_fmt 0) or bf16 (a_fmt 1)
  {
    const int m = warp * 32 + lane;
    uint32_t pk[8];
    for (int g = 0; g < 4; ++g) {
      for (int c = 0; c < 8; ++c) {
        float lo = A[(m % 64) * 64 + g * 16 + 2 * c], hi = A[(m % 64) * 64 + g * 16 + 2 * c + 1];
        if (a_fmt == 0) {
          __half2 h = __floats2half2_rn(lo, hi);
          pk[c] = *(uint32_t *)&h;
        } else pk[c] = pack_bf16(lo, hi);
      }
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + g * 8, pk);
    }
    tc_wait_st();
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t id = ((1u << 4) | ((uint32_t)a_fmt << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(32 >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24));
      for (int ks = 0; ks < 4; ++ks) mma_ts(tmem + 128, tmem + ks * 8, sdesc_sw64(smem_u32(sv) + ks * 1024), id, ks);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 128, r);
  tc_wait_ld();
  for (int c = 0; c < 32; ++c) out[(warp * 32 + lane) * 32 + c] = __uint_as_float(r[c]);
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

__global__ void atom_bench(float *out, int mode, int iters, long long *cycles) {
  __shared__ float acc[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  for (int it = 0; it < iters; ++it) {
    int addr;
    if (mode == 0) addr = (warp * 32 + lane + it * 7) & 4095;        // distinct banks
    else if (mode == 1) addr = (warp * 64 + (it & 63)) & 4095;      // same address per warp
    else addr = ((lane * 40) + warp * 8 + it) & 4095;               // strided
    atomicAdd(&acc[addr], 1.0f);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) atomicAdd(&out[i], acc[i]);
}

int main() {
  float *A, *B, *D, *TS;
  int *ok;
  cudaMallocManaged(&A, 64 * 32 * 4);
  cudaMallocManaged(&B, N * 32 * 4);
  cudaMallocManaged(&D, 128 * 64 * 4);
  cudaMallocManaged(&TS, 128 * 32 * 4);
  cudaMallocManaged(&ok, 128 * 4);
  srand(1);
  for (int i = 0; i < 64 * 32; ++i) A[i] = (float)((rand() % 17) - 8) / 8.f;
  for (int i = 0; i < N * 32; ++i) B[i] = (float)((rand() % 17) - 8) / 8.f;
  test_m64<<<1, 128>>>(D, nullptr, A, B, TS, ok);
  cudaError_t e = cudaDeviceSynchronize();
  printf("test_m64: %s\n", cudaGetErrorString(e));
  // expected D0[m][n] = sum_k A[m][k] B[n][k]; D1[m][n] = sum_k A[m][k] B[n+8][k]
  int bad0 = 0, bad1 = 0, badz = 0;
  for (int lane = 0; lane < 128; ++lane) {
    int q = lane / 32, l = lane % 32;
    for (int n = 0; n < 64; ++n) {
      float got = D[lane * 64 + n];
      if (l < 16) {
        int m = q * 16 + l;
        float ex = 0;
        for (int k = 0; k < 32; ++k) ex += A[m * 32 + k] * B[n * 32 + k];
        if (n < N && fabsf(got - ex) > 1e-3) bad0++;
      } else {
        int m = q * 16 + (l - 16);
        float ex = 0;
        if (n + 8 < N) {
          for (int k = 0; k < 32; ++k) ex += A[m * 32 + k] * B[(n + 8) * 32 + k];
          if (fabsf(got - ex) > 1e-3) bad1++;
        }
      }
    }
  }
  int okc = 0;
  for (int i = 0; i < 128; ++i) okc += ok[i];
  printf("M64 lane0 half mismatches %d, lane16 half mismatches %d (zero-check %d); unaligned ld ok lanes %d/128\n", bad0, bad1,
         badz, okc);
  // TS check: O[m][d] = sum_key bf16(D_half[m][key]) * B[key][d] for key < 64 (lane offset 16 uses D1 half)
  int badts = 0;
  for (int lane = 0; lane < 128; ++lane) {
    int q = lane / 32, l = lane % 32;
    for (int d = 0; d < 32; ++d) {
      double ex = 0;
      for (int key = 0; key < 64; ++key) {
        float dv = D[lane * 64 + key];
        float pb = __bfloat162float(__float2bfloat16(dv));
        ex += pb * __bfloat162float(__float2bfloat16(B[key * 32 + d]));
      }
      float got = TS[lane * 32 + d];
      if (fabs(got - ex) > 1e-2 * (1 + fabs(ex))) badts++;
    }
  }
  printf("TS MMA mismatches %d\n", badts);
  {
    float *A2, *B2, *O2;
    cudaMallocManaged(&A2, 64 * 64 * 4);
    cudaMallocManaged(&B2, 64 * 32 * 4);
    cudaMallocManaged(&O2, 128 * 32 * 4);
    for (int i = 0; i < 64 * 64; ++i) A2[i] = (float)(rand() % 20001 - 10000) * 1.2345e-5f;  // fine-grained values
    for (int i = 0; i < 64 * 32; ++i) B2[i] = (float)((rand() % 17) - 8) / 8.f;
    for (int fmt = 0; fmt < 2; ++fmt) {
      test_mixed<<<1, 128>>>(A2, B2, O2, fmt);
      cudaError_t e = cudaDeviceSynchronize();
      printf("test_mixed fmt %d: %s\n", fmt, cudaGetErrorString(e));
      fflush(stdout);
      if (e != cudaSuccess) return 1;
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int d = 0; d < 32; ++d) {
          double ex = 0;
          for (int k = 0; k < 64; ++k) ex += (double)A2[(m % 64) * 64 + k] * B2[k * 32 + d];
          maxerr = fmax(maxerr, fabs(ex - O2[m * 32 + d]));
        }
      printf("TS A=%s (TMEM) x B=bf16: %s, max abs err vs fp64 %.3e\n", fmt == 0 ? "fp16" : "bf16", cudaGetErrorString(e), maxerr);
    }
  }
  float *out;
  long long *cyc;
  cudaMallocManaged(&out, 4096 * 4);
  cudaMallocManaged(&cyc, 148 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    int iters = 4096;
    atom_bench<<<148, 256>>>(out, mode, iters, cyc);
    cudaDeviceSynchronize();
    double per = (double)cyc[0] / iters;
    printf("smem atomicAdd mode %d: %.1f cycles per iteration of 8 warps (%.2f cycles per warp-instr)\n", mode, per, per / 8);
  }
  return 0;
}
