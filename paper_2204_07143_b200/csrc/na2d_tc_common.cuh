// na2d_tc_common.cuh -- pieces shared by the tcgen05 NA2D kernels (forward, backward):
// tile geometry constants, TMEM row load/store helpers, reductions and the masked
// relative-positional-bias table.
#pragma once

#include <math.h>

#include "na2d_internal.cuh"
#include "na2d_sm100.cuh"

namespace na2d {
namespace tc {

using namespace sm100;

constexpr int kTQH = 8, kTQW = 16, kD = 32;  // tile: 8 x 16 queries (keys), head dim 32
constexpr int kHCP = 24;                    // halo row pitch (keys)
constexpr int kRowBytes = kD * 2;           // 64-byte rows (32 bf16)
constexpr int kTblStride = 40;              // floats per table row (8 mod 32: conflict-free 4x4 blocks)
constexpr int kTblOff = 8;                  // column offset for negative bias columns

// Masked, pre-scaled bias table for one head:
//   T[dc][a][kTblOff + b] = B[h][a][b] * mul   if b in [dc, dc + Lw)   (a < 2L-1)
//                          = -inf               otherwise, and for the extra row a = 2L-1
// dc = wstart(j) - j + L - 1 is the column-clamp class of the query, a/b the bias row/column
// (key - query + L - 1).  Row validity is applied by pointing at row 2L-1 instead.
template <int L>
struct BiasTable {
  static constexpr int TT = 2 * L - 1;
  static constexpr int TROWS = TT + 1;
  static constexpr int FLOATS = L * TROWS * kTblStride;
  // `copies` (1 or 2) parity copies of the table (copy x holds column b at kTblOff + x + b: a
  // reader whose first column has parity x uses copy x, so its element pairs are 8-byte aligned),
  // each with `extra` all -inf classes after the L real ones (copy x at
  // tbl + x * (L + extra) * TROWS * kTblStride), built from a staged, pre-scaled copy of the head's
  // (2L-1)^2 bias values in shared memory (rs, or null for no bias).  One table row per thread: no
  // global load latency and no per-element index arithmetic inside the build (the element-parallel
  // build straight from global memory it replaces took ~5.4 us per head in B1,
  // scripts/trace_fixed.py).  B1 uses it; B2 keeps build_rows (measured faster there).
  __device__ static void build_rows_smem(float *tbl, const float *rs, int Lw, int copies, int extra, int tid,
                                         int nthreads) {
    const int per_copy = (L + extra) * TROWS;
    for (int row = tid; row < copies * per_copy; row += nthreads) {
      const int x = row / per_copy, rc = row - x * per_copy;
      const int dc = rc / TROWS, rr = rc - dc * TROWS;
      float *dst = tbl + row * kTblStride;
      const bool live = dc < L && rr < TT;
      const float *src = rs + (live ? rr * TT : 0);
      const int lo = kTblOff + x + dc, hi = lo + Lw;  // entries holding columns [dc, dc + Lw)
#pragma unroll 8
      for (int e = 0; e < kTblStride; ++e)
        dst[e] = live && e >= lo && e < hi ? (rs ? src[e - kTblOff - x] : 0.f) : -INFINITY;
    }
  }
  // one table row per thread: the row's 2L-1 bias values are loaded together (independent loads),
  // then the row's kTblStride entries written
  __device__ static void build_rows(float *tbl, const float *rpb, int h, int Lw, float mul, int tid, int nthreads) {
    for (int row = tid; row < L * TROWS; row += nthreads) {
      const int dc = row / TROWS, rr = row % TROWS;
      float b[TT];
#pragma unroll
      for (int k = 0; k < TT; ++k) b[k] = (rpb && rr < TT) ? __ldg(&rpb[(h * TT + rr) * TT + k]) * mul : 0.f;
      float *dst = tbl + row * kTblStride;
#pragma unroll
      for (int e = 0; e < kTblStride; ++e) {
        const int cb = e - kTblOff;
        float v = -INFINITY;
#pragma unroll
        for (int k = 0; k < TT; ++k)
          if (cb == k && rr < TT && k >= dc && k < dc + Lw) v = b[k];
        dst[e] = v;
      }
    }
  }
};

// N consecutive TMEM columns of this warp's 32 lanes -> registers (N = 16a + 8b + 4c + 2d, the
// loads all issued before the caller's tcgen05.wait::ld)
template <int N>
__device__ __forceinline__ void ld_row(uint32_t addr, uint32_t (&v)[N]) {
  int o = 0;
#pragma unroll
  for (; o + 16 <= N; o += 16) {
    uint32_t a[16];
    tmem_ld16(addr + o, a);
#pragma unroll
    for (int z = 0; z < 16; ++z) v[o + z] = a[z];
  }
  if constexpr (N % 16 >= 8) {
    constexpr int B = N / 16 * 16;
    uint32_t a[8];
    tmem_ld8(addr + B, a);
#pragma unroll
    for (int z = 0; z < 8; ++z) v[B + z] = a[z];
  }
  if constexpr (N % 8 >= 4) {
    constexpr int B = N / 8 * 8;
    uint32_t a[4];
    tmem_ld4(addr + B, a);
#pragma unroll
    for (int z = 0; z < 4; ++z) v[B + z] = a[z];
  }
  if constexpr (N % 4 >= 2) {
    constexpr int B = N / 4 * 4;
    uint32_t a[2];
    tmem_ld2(addr + B, a);
    v[B] = a[0];
    v[B + 1] = a[1];
  }
  if constexpr (N % 2 == 1) tmem_ld1(addr + N - 1, v[N - 1]);
}
template <int N>
__device__ __forceinline__ void st_row(uint32_t addr, const uint32_t (&v)[N]) {
  int o = 0;
#pragma unroll
  for (; o + 16 <= N; o += 16) {
    uint32_t a[16];
#pragma unroll
    for (int z = 0; z < 16; ++z) a[z] = v[o + z];
    tmem_st16(addr + o, a);
  }
  if constexpr (N % 16 >= 8) {
    constexpr int B = N / 16 * 16;
    uint32_t a[8];
#pragma unroll
    for (int z = 0; z < 8; ++z) a[z] = v[B + z];
    tmem_st8(addr + B, a);
  }
  if constexpr (N % 8 >= 4) {
    constexpr int B = N / 8 * 8;
    uint32_t a[4] = {v[B], v[B + 1], v[B + 2], v[B + 3]};
    tmem_st4(addr + B, a);
  }
  if constexpr (N % 4 >= 2) {
    constexpr int B = N / 4 * 4;
    uint32_t a[2] = {v[B], v[B + 1]};
    tmem_st2(addr + B, a);
  }
  if constexpr (N % 2 == 1) tmem_st1(addr + N - 1, v[N - 1]);
}
// zeros into N consecutive TMEM columns of this warp's 32 lanes
template <int N>
__device__ __forceinline__ void st_zero(uint32_t addr) {
  const uint32_t z = 0;
  if constexpr (N >= 32) {
    tmem_st32_zero(addr);
    st_zero<N - 32>(addr + 32);
  } else if constexpr (N >= 16) {
    const uint32_t a[16] = {z, z, z, z, z, z, z, z, z, z, z, z, z, z, z, z};
    tmem_st16(addr, a);
    st_zero<N - 16>(addr + 16);
  } else if constexpr (N >= 8) {
    const uint32_t a[8] = {z, z, z, z, z, z, z, z};
    tmem_st8(addr, a);
    st_zero<N - 8>(addr + 8);
  } else if constexpr (N >= 4) {
    const uint32_t a[4] = {z, z, z, z};
    tmem_st4(addr, a);
    st_zero<N - 4>(addr + 4);
  } else if constexpr (N >= 2) {
    const uint32_t a[2] = {z, z};
    tmem_st2(addr, a);
    st_zero<N - 2>(addr + 2);
  } else if constexpr (N == 1) {
    tmem_st1(addr, z);
  }
}
__device__ __forceinline__ void st_zero12(uint32_t addr) {
  const uint32_t z8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint32_t z4[4] = {0, 0, 0, 0};
  tmem_st8(addr, z8);
  tmem_st4(addr + 8, z4);
}
template <int N>
__device__ __forceinline__ float tree_max(const float (&x)[N]) {
  float m[N];
#pragma unroll
  for (int z = 0; z < N; ++z) m[z] = x[z];
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int z = 0; z + w < N; z += 2 * w) m[z] = fmaxf(m[z], m[z + w]);
  return m[0];
}
template <int N>
__device__ __forceinline__ float tree_sum(const float (&x)[N]) {
  float m[N];
#pragma unroll
  for (int z = 0; z < N; ++z) m[z] = x[z];
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int z = 0; z + w < N; z += 2 * w) m[z] += m[z + w];
  return m[0];
}


int num_sms();  // of the current device

// Small-map pair mode: maps of at most one tile (H, W <= 8, whole map, no row band) and an even
// batch run two maps per 8 x 16 tile -- map (b, h) in tile columns 0-7 (TMEM lane quarters 0, 1)
// and map (b + 1, h) in columns 8-15 (quarters 2, 3) -- instead of one map in 49 of 128 query slots
// (NAT stage 4, 7 x 7).  K / V / Q halos come from make_tmap_e16_pair views; each map keeps its own
// clamped windows and bias cells.  NA2D_NO_PAIR=1 disables it (tests, A/B).
bool pair_mode(int B, int H, int W, int q_row0, int q_rows, int kv_row0, int kv_rows);
// raise kernel `func`'s dynamic shared-memory limit on the current device (once per device)
cudaError_t ensure_smem_attr(const void *func, int smem_bytes);

// Launch with programmatic stream serialization (see pdl_trigger / pdl_wait in na2d_sm100.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace tc
}  // namespace na2d
