// na2d_internal.cuh -- shared host/device definitions of libna2d (CUDA path only).
//
// Geometry of Eq. 2's neighbourhood rho: per axis the
// window of query i on an axis of n pixels starts at clamp(i - (L-1)/2, 0, n - L) and has
// length L; if L >= n it is the whole axis.  Bias cell = key - query + L - 1.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "na2d.h"

namespace na2d {

// Problem after validation; all row indices global (row bands).
struct Geo {
  int B, heads;
  int H;        // global map rows
  int W, d, L;
  int q_rows, q_row0;
  int kv_rows, kv_row0;
  float scale;  // multiplier on (q.k + B)
  int dtype;
};

__host__ __device__ __forceinline__ int wstart(int i, int n, int L) {
  if (L >= n) return 0;
  int s = i - (L - 1) / 2;
  s = s < 0 ? 0 : s;
  return s > n - L ? n - L : s;
}
__host__ __device__ __forceinline__ int wlen(int n, int L) { return L < n ? L : n; }

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f32(__half x) { return __half2float(x); }
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <> __device__ __forceinline__ __half from_f32<__half>(float x) { return __float2half_rn(x); }

// ---- launchers implemented per translation unit -------------------------------------------
// SIMT path (any even dim <= 128, any odd L <= 31, fp32 or bf16): na2d_simt.cu
cudaError_t simt_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                         void *out, float *lse, cudaStream_t st);
// ds_slots: scratch of simt_backward_scratch_bytes(g) (per-query window-slot dS, summed per dRPB
// cell in a fixed order: the SIMT dRPB is bitwise reproducible)
cudaError_t simt_backward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                          const void *out, const float *lse, const void *dout, void *dq, void *dk,
                          void *dv, float *drpb, float *D, float *ds_slots, cudaStream_t st);
size_t simt_backward_scratch_bytes(const Geo &g);
int simt_launches(const Geo &g, int which);
// SIMT dK/dV only (uses D and LSE already computed)
cudaError_t simt_backward_dkdv(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                               const float *lse, const void *dout, const float *D, void *dk, void *dv,
                               cudaStream_t st);

// The paper's unfused decomposition (QK+RPB -> softmax -> AV and gradients): na2d_unfused.cu
cudaError_t unfused_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                            float *lse, float *attn, cudaStream_t st);
cudaError_t unfused_backward(const Geo &g, const void *q, const void *k, const void *v, const void *dout,
                             const float *attn, float *dS, void *dq, void *dk, void *dv, float *drpb, cudaStream_t st);

// Debug timeline buffer set through na2d_debug_set_trace (null = tracing off).
void *debug_trace_buffer();

}  // namespace na2d
