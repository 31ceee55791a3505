#include <string>
// tcgen05.mma throughput for the shapes the NA2D kernels use (one CTA per SM, 148 CTAs).
#include <stdint.h>
#include <stdio.h>

#include "na2d_sm100.cuh"

using namespace na2d::sm100;

template <int M, int N, bool TS, int CHAINS>
__global__ void mma_bench(int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
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
    constexpr uint32_t id = idesc_bf16(M, N, TS);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
          const uint32_t d = tmem + (TS ? 256 : 0) + c * (TS ? 32 : N) % 256;
          if (TS)
            mma_ts(tmem + 256 + c * 32, tmem + 0 + (it % 8) * 8, sdesc_sw64(b + (it % 8) * 1024), id, it > 0);
          else
            mma_ss(tmem + (c % 2) * 256, sdesc_sw64(a + (it % 2) * 32), sdesc_sw64(b + (it % 2) * 32), id, it > 0);
          (void)d;
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

template <int M, int N, bool TS, int CHAINS>
void run(const char *name) {
  long long *cyc;
  cudaMallocManaged(&cyc, 148 * 8);
  auto k = mma_bench<M, N, TS, CHAINS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  k<<<148, 128, 100 * 1024>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  double per = (double)cyc[0] / (iters * CHAINS);
  double macs = (double)M * N * 16;
  printf("%-34s %7.1f cyc/MMA  %6.0f MAC/clk/SM  (%s)\n", name, per, macs / per, cudaGetErrorString(e));
}


// B2's per-chunk tensor sequence: S^T/dP^T (8 SS, M=64 N=96, sub-tiles at TMEM lane offsets 0 / 16)
// into slot x, then dV/dK (24 TS, M=64 N=32, A = bf16 P^T / dS^T from the slot) into 8 chains.
// MODE 1: S only, 2: dV/dK only, 3: both.  Reports cycles per chunk and the issue time per chunk.
template <int MODE>
__global__ void chunk_bench(int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
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
    constexpr uint32_t ids = idesc_bf16(64, 96, false), ido = idesc_bf16(64, 32, true);
    const uint32_t q = smem_u32(smem), dO = q + 24576, k = q + 49152, v = k + 8192;
    long long t0 = clock64(), tiss = 0;
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        const uint32_t x = (it & 1) * 192;
        const int row = (it % 3) * 4;
        long long a = clock64();
        if (MODE & 1) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {
              const uint32_t lo = ((uint32_t)(16 * sb) << 16) + x;
              mma_ss(tmem + lo, sdesc_sw64(k + sb * 4096 + kk * 32), sdesc_sw64(q + row * 24 * 64 + kk * 32), ids, kk);
              mma_ss(tmem + lo + 96, sdesc_sw64(v + sb * 4096 + kk * 32), sdesc_sw64(dO + row * 24 * 64 + kk * 32), ids, kk);
            }
        }
        if (MODE & 2) {
#pragma unroll
          for (int ks = 0; ks < 6; ++ks)
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {
              const uint32_t lo = (uint32_t)(16 * sb) << 16;
              const uint32_t boff = row * 24 * 64 + ks * 16 * 64;
              mma_ts(tmem + lo + 384 + (ks & 1) * 32, tmem + lo + x + ks * 8, sdesc_sw64(dO + boff), ido, it > 0 || ks >= 2);
              mma_ts(tmem + lo + 448 + (ks & 1) * 32, tmem + lo + x + 96 + ks * 8, sdesc_sw64(q + boff), ido, it > 0 || ks >= 2);
            }
        }
        tiss += clock64() - a;
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      cyc[2 * blockIdx.x] = t1 - t0;
      cyc[2 * blockIdx.x + 1] = tiss;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run_chunk(const char *name) {
  long long *cyc;
  cudaMallocManaged(&cyc, 2 * 148 * 8);
  auto kf = chunk_bench<MODE>;
  cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 1000;
  kf<<<148, 128, 100 * 1024>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-34s %7.1f cyc/chunk  issue %6.1f cyc/chunk (%s)\n", name, (double)cyc[0] / iters, (double)cyc[1] / iters,
         cudaGetErrorString(e));
}

int main_old() {
  run_chunk<1>("B2 chunk: S/dP only");
  run_chunk<2>("B2 chunk: dV/dK only");
  run_chunk<3>("B2 chunk: S/dP + dV/dK");
  run<128, 256, false, 1>("SS M=128 N=256 (1 chain)");
  run<128, 256, false, 2>("SS M=128 N=256 (2 chains)");
  run<64, 240, false, 1>("SS M=64 N=240 (1 chain)");
  run<64, 240, false, 2>("SS M=64 N=240 (2 chains)");
  run<128, 160, false, 2>("SS M=128 N=160 (2 chains)");
  run<64, 32, true, 1>("TS M=64 N=32 (1 chain)");
  run<64, 32, true, 4>("TS M=64 N=32 (4 chains)");
  run<128, 32, true, 1>("TS M=128 N=32 (1 chain)");
  run<128, 32, true, 4>("TS M=128 N=32 (4 chains)");
  run<128, 64, true, 4>("TS M=128 N=64 (4 chains)");
  run<64, 64, true, 4>("TS M=64 N=64 (4 chains)");
  run<64, 32, false, 4>("SS M=64 N=32 (4 chains)");
  run<128, 32, false, 4>("SS M=128 N=32 (4 chains)");
  run<64, 48, false, 4>("SS M=64 N=48 (4 chains)");
  run<128, 96, false, 2>("SS M=128 N=96 (2 chains)");
  run<64, 96, false, 2>("SS M=64 N=96 (2 chains)");
  return 0;
}

// TS M=64 N=32 MMA stream (warp 0, 3 chains, like the forward's PV) while NLD other warps hammer
// TMEM with tcgen05.ld/st x16 on disjoint columns (like the softmax warps of the other group).
template <int NLD, bool ST>
__global__ void contention_bench(int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t &bar = *(uint64_t *)(smem + 80 * 1024);
  uint32_t &slot = *(uint32_t *)(smem + 80 * 1024 + 8);
  volatile int &done = *(volatile int *)(smem + 80 * 1024 + 16);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t id = idesc_bf16(64, 32, true);
    const uint32_t b = smem_u32(smem + 16384);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 6; ++c)
          mma_ts(tmem + ((uint32_t)(16 * (c & 1)) << 16) + 128 + (c >> 1) * 32,
                 tmem + ((uint32_t)(16 * (c & 1)) << 16) + (it % 8) * 8,
                 sdesc_sw64(b + (it % 8) * 1024), id, it > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && warp < 4 + NLD) {
    const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 + (warp >= 8 ? 128 : 0);
    uint32_t r[16];
    float acc = 0.f;
    while (!done) {
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        tmem_ld16(la + k * 16, r);
        tc_wait_ld();
        acc += __uint_as_float(r[3]);
        if (ST) {
          tmem_st16(la + k * 16, r);
        }
      }
      if (ST) tc_wait_st();
    }
    if (acc == 1234.5f) cyc[1000] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int NLD, bool ST>
void run_cont(const char *name) {
  long long *cyc = nullptr, host[4] = {0, 0, 0, 0};
  cudaError_t e0 = cudaMalloc(&cyc, 2000 * 8);
  auto k = contention_bench<NLD, ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  k<<<148, 384, 100 * 1024>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %7.1f cyc/MMA (%s / %s)\n", name, (double)host[0] / (iters * 6), cudaGetErrorString(e0),
         cudaGetErrorString(e));
  cudaFree(cyc);
}

int main_old2() {
  run_cont<0, false>("TS M=64 N=32 x6 chains, idle");
  run_cont<4, false>("... + 4 warps tcgen05.ld");
  run_cont<8, false>("... + 8 warps tcgen05.ld");
  run_cont<4, true>("... + 4 warps ld+st");
  run_cont<8, true>("... + 8 warps ld+st");
  return 0;
}

// The forward's per-tile tensor sequence: QK (4 SS, M=64 N=240, sub-tiles at lane offsets 0/16)
// into slot t&1, then PV of the previous tile (30 TS, M=64 N=32, A = P at slot (t-1)&1 columns
// [0,120), D at [120,216) in 3 chains x 2 sub-tiles).  NLD other warps do TMEM ld/st.
template <int NLD, bool QK, bool PV, bool MODE_ST = true>
__global__ void fwd_seq_bench(int iters, long long *cyc, const uint8_t *gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t &bar = *(uint64_t *)(smem + 90 * 1024);
  uint32_t &slot = *(uint32_t *)(smem + 90 * 1024 + 8);
  volatile int &done = *(volatile int *)(smem + 90 * 1024 + 16);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 88 * 1024 / 4; i += blockDim.x) {  // random bf16 pairs in [-2, 2)
    uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    ((uint32_t *)smem)[i] = (x & 0x807f807fu) | 0x3f003f00u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t iqk = idesc_bf16(64, 240, false), ipv = idesc_bf16(64, 32, true);
    const uint32_t q = smem_u32(smem), k = q + 8192, v = q + 8192 + 21504;
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        const uint32_t s0 = tmem + (it & 1) * 256, p0 = tmem + ((it + 1) & 1) * 256;
        if (QK) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
#pragma unroll
            for (int sb = 0; sb < 2; ++sb)
              mma_ss(s0 + ((uint32_t)(16 * sb) << 16), sdesc_sw64(q + sb * 4096 + kk * 32),
                     sdesc_sw64(k + sb * 4 * 1536 + kk * 32), iqk, kk);
        }
        if (PV) {
          if (NLD >= 100) tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 15; ++ks)
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {
              const uint32_t b = p0 + ((uint32_t)(16 * sb) << 16);
              mma_ts(b + 120 + (ks % 3) * 32, b + ks * 8, sdesc_sw64(v + sb * 4 * 1536 + ks * 1024), ipv, ks >= 3);
            }
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && warp < 4 + NLD && MODE_ST == false && QK == false) {
  } else if (warp == 4 && NLD == 1) {
    const int lane = threadIdx.x % 32;
    // bulk-copy producer: 2 x 16 KB global -> smem [60 KB, 92 KB) per round, like the TMA halo loads
    uint64_t &tb = *(uint64_t *)(smem + 90 * 1024 + 32);
    if (lane == 0) {
      mbar_init(&tb, 1);
      fence_barrier_init();
      uint32_t ph = 0;
      size_t off = blockIdx.x * 65536;
      while (!done) {
        mbar_expect_tx(&tb, 32768);
        for (int h = 0; h < 2; ++h)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(smem + 52 * 1024 + h * 16384)), "l"(gsrc + off + h * 16384), "r"(16384),
                       "r"(smem_u32(&tb)) : "memory");
        mbar_wait(&tb, ph);
        ph ^= 1;
        off = (off + 32768) % (size_t)(148 * 65536 * 16);
      }
    }
  } else if (warp >= 4 && warp < 4 + NLD && (NLD == 6 || NLD == 5)) {
    // LDS with bank conflicts (NLD == 6: lanes stride 40 floats, 8-way; NLD == 5: stride 32, 32-way)
    const int stride = NLD == 6 ? 40 : 32;
    const float *sp = (const float *)(smem + 60 * 1024) + (threadIdx.x % 32) * stride;
    float acc2 = 0.f;
    while (!done) {
#pragma unroll 8
      for (int kk = 0; kk < 64; ++kk) acc2 += sp[kk & 15];
    }
    if (acc2 == 1234.5f) cyc[1000] = 1;
  } else if (warp >= 4 && warp < 4 + NLD && NLD == 7) {
    // pure ALU / MUFU / LDS load (no TMEM): FFMA2 + ex2 + LDS like the softmax warps
    float2 a = make_float2(threadIdx.x * 1e-3f, 0.5f), b2 = make_float2(1.0001f, 0.9999f);
    float e0 = 0.f, e1 = 0.f;
    const float *sp = (const float *)(smem + (threadIdx.x % 64) * 16);
    while (!done) {
#pragma unroll 8
      for (int kk = 0; kk < 64; ++kk) {
        a = __ffma2_rn(a, b2, make_float2(sp[kk & 7], sp[(kk + 3) & 7]));
        e0 += ex2(a.x * 1e-3f);
        e1 += ex2(a.y * 1e-3f);
      }
    }
    if (e0 + e1 == 1234.5f) cyc[1000] = 1;
  } else if (warp >= 4 && warp < 4 + (NLD >= 100 ? NLD - 100 : NLD)) {
    // like the softmax passes: both slots' lanes, two x16 loads in flight, a x16 + x8 store
    const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >= 8 ? 256 : 0);
    uint32_t r[16], r2[16];
    float acc = 0.f;
    while (!done) {
#pragma unroll 1
      for (int kk = 0; kk < 5; ++kk) {
        tmem_ld16(la + kk * 24, r);
        tmem_ld16(la + kk * 24 + 24, r2);
        tc_wait_ld();
        acc += __uint_as_float(r[3]) + __uint_as_float(r2[5]);
        if (MODE_ST) {
          tmem_st16(la + kk * 16 + 120, r);
          uint32_t r8[8] = {r2[0], r2[1], r2[2], r2[3], r2[4], r2[5], r2[6], r2[7]};
          tmem_st8(la + kk * 16 + 136, r8);
        }
      }
      tc_wait_st();
    }
    if (acc == 1234.5f) cyc[1000] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int NLD, bool QK, bool PV, bool MODE_ST = true>
void run_seq(const char *name) {
  long long *cyc = nullptr, host[4] = {0, 0, 0, 0};
  cudaMalloc(&cyc, 2000 * 8);
  auto k = fwd_seq_bench<NLD, QK, PV, MODE_ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 500;
  static uint8_t *gsrc = nullptr;
  if (!gsrc) cudaMalloc(&gsrc, (size_t)148 * 65536 * 16 + 65536);
  k<<<148, 384, 100 * 1024>>>(iters, cyc, gsrc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cyc/tile (%s)\n", name, (double)host[0] / iters, cudaGetErrorString(e));
  fflush(stdout);
  cudaFree(cyc);
}

int main_old4() {
  run_seq<0, true, false>("fwd seq: QK only");
  run_seq<0, false, true>("fwd seq: PV only");
  run_seq<0, true, true>("fwd seq: QK + PV");
  run_seq<8, true, true, false>("fwd seq: QK + PV, 8 ld warps");
  run_seq<8, true, true>("fwd seq: QK + PV, 8 ld/st warps");
  run_seq<4, true, true>("fwd seq: QK + PV, 4 ld/st warps");
  run_seq<7, true, true>("fwd seq: QK + PV, 7 ALU/MUFU/LDS warps");
  run_seq<6, true, true>("fwd seq: QK + PV, 6 LDS 8-way-conflict warps");
  run_seq<5, true, true>("fwd seq: QK + PV, 5 LDS 32-way-conflict warps");
  return 0;
}

// Issue mechanics: the forward's per-tile MMAs (4 QK + 30 PV) issued as
//   V=0: one elect block per tile;  V=1: QK block + 5 PV blocks of 6 (elect + syncwarp each);
//   V=2: V=1 + a tcgen05.commit after every block;  V=3: V=1 + mbarrier wait (already complete)
//   + tcgen05.fence::after_thread_sync before every block;  V=4: V=1 with precomputed descriptors.
template <int V>
__global__ void issue_bench(int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t &bar = *(uint64_t *)(smem + 90 * 1024);
  uint64_t &bar2 = *(uint64_t *)(smem + 90 * 1024 + 8);
  uint64_t &done_bar = *(uint64_t *)(smem + 90 * 1024 + 16);
  uint32_t &slot = *(uint32_t *)(smem + 90 * 1024 + 24);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 88 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&done_bar, 1);
    fence_barrier_init();
    mbar_arrive(&done_bar);
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t iqk = idesc_bf16(64, 240, false), ipv = idesc_bf16(64, 32, true);
    const uint32_t q = smem_u32(smem), k = q + 8192, v = q + 8192 + 21504;
    const uint64_t dv = sdesc_sw64(v);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t s0 = tmem + (it & 1) * 256, p0 = tmem + ((it + 1) & 1) * 256, p1 = p0 + ((uint32_t)16 << 16);
      if (V == 0) {
        if (elect_one()) {
          for (int kk = 0; kk < 2; ++kk)
            for (int sb = 0; sb < 2; ++sb)
              mma_ss(s0 + ((uint32_t)(16 * sb) << 16), sdesc_sw64(q + sb * 4096 + kk * 32),
                     sdesc_sw64(k + sb * 4 * 1536 + kk * 32), iqk, kk);
#pragma unroll
          for (int ks = 0; ks < 15; ++ks)
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {
              const uint32_t b = p0 + ((uint32_t)(16 * sb) << 16);
              mma_ts(b + 120 + (ks % 3) * 32, b + ks * 8, sdesc_sw64(v + sb * 4 * 1536 + ks * 1024), ipv, ks >= 3);
            }
        }
        __syncwarp();
      } else {
        if (elect_one()) {
          for (int kk = 0; kk < 2; ++kk)
            for (int sb = 0; sb < 2; ++sb)
              mma_ss(s0 + ((uint32_t)(16 * sb) << 16), sdesc_sw64(q + sb * 4096 + kk * 32),
                     sdesc_sw64(k + sb * 4 * 1536 + kk * 32), iqk, kk);
          if (V == 2) mma_commit(&bar2);
        }
        __syncwarp();
#pragma unroll
        for (int pk = 0; pk < 5; ++pk) {
          if (V == 3) {
            mbar_wait(&done_bar, 0);
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int k3 = 0; k3 < 3; ++k3) {
              const int ks = 3 * pk + k3;
              if (V == 4) {
                const uint32_t vo = (ks * 1024) >> 4;
                mma_ts(p0 + 120 + k3 * 32, p0 + ks * 8, dv + vo, ipv, pk > 0);
                mma_ts(p1 + 120 + k3 * 32, p1 + ks * 8, dv + (6144 >> 4) + vo, ipv, pk > 0);
              } else {
#pragma unroll
                for (int sb = 0; sb < 2; ++sb) {
                  const uint32_t b = p0 + ((uint32_t)(16 * sb) << 16);
                  mma_ts(b + 120 + k3 * 32, b + ks * 8, sdesc_sw64(v + sb * 4 * 1536 + ks * 1024), ipv, pk > 0);
                }
              }
            }
            if (V == 2) mma_commit(&bar2);
          }
          __syncwarp();
        }
      }
    }
    if (elect_one()) mma_commit(&bar);
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

template <int V>
void run_issue(const char *name) {
  long long *cyc = nullptr, host[4] = {0, 0, 0, 0};
  cudaMalloc(&cyc, 2000 * 8);
  auto k = issue_bench<V>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 500;
  k<<<148, 128, 100 * 1024>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-50s %7.1f cyc/tile (%s)\n", name, (double)host[0] / iters, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main_old5() {
  run_issue<0>("issue: one elect block per tile");
  run_issue<1>("issue: QK block + 5 PV blocks of 6");
  run_issue<2>("issue: ... + commit per block");
  run_issue<3>("issue: ... + mbar wait + fence per block");
  run_issue<4>("issue: 5 PV blocks, precomputed descriptors");
  return 0;
}

int main(int argc, char **argv) {
  // `microbench_mma all`: every section (MMA shapes / chains, TMEM contention, issue mechanics,
  // B2 chunk, forward sequence); default: the forward sequence only
  if (argc > 1 && std::string(argv[1]) == "all") {
    main_old();
    main_old2();
    main_old4();
    main_old5();
  }
  run_seq<8, true, true>("fwd seq: QK + PV, 8 ld/st warps");
  run_seq<108, true, true>("fwd seq: ... + fence::after_thread_sync per PV block");
  run_seq<100, true, true>("fwd seq: fence, no ld/st warps");
  return 0;
}
