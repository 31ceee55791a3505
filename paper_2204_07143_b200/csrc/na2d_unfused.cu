// na2d_unfused.cu -- the paper's own NA decomposition, as a comparison path.
//
// PAPER.md P:442 (App. A): NA runs as a QK kernel that adds the relative positional bias "as the
// attention weights are being computed" and writes the H x W x L^2 attention tensor, the softmax
// (left to the framework's kernel in the paper; here our own), and an AV kernel; training runs the
// backward of each.  Unlike the fused tcgen05 path this materialises the attention weights in HBM
// (4 L^2 bytes per query-head in fp32, ~4x the fused path's traffic at L = 7).  Kernels are plain
// CUDA-core code, one warp per query (or key) row:
//   qk_rpb   A[q][m] = scale (q . k_m + B[cell(q, m)])     m = window position, row-major
//   softmax  A[q][:] <- softmax(A[q][:]), LSE[q]          (exact, max-subtracted)
//   av       O[q] = sum_m A[q][m] v_m
//   backward dA[q][m] = dO_q . v_m; dV_p = sum_{q: p in rho(q)} A[q][m(q,p)] dO_q;
//            dS = A (dA - sum_m A dA); dQ = scale sum_m dS k_m; dK_p = scale sum dS q;
//            dB[cell] = scale sum dS (fp32 atomics)
#include <math.h>

#include "na2d_internal.cuh"
#include "na2d_profile.cuh"

namespace na2d {
namespace {

constexpr int kWarps = 8;  // warps per block; one row (query or key) per warp

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

struct Row {  // a query (or key) row of the flattened [B*heads][rows][W] index space
  long bh, t;
  int i, j;
};
__device__ __forceinline__ bool row_of(const Geo &g, long rows_per_bh, Row &r) {
  const long gw = (long)blockIdx.x * kWarps + threadIdx.x / 32;
  if (gw >= (long)g.B * g.heads * rows_per_bh) return false;
  r.bh = gw / rows_per_bh;
  r.t = gw - r.bh * rows_per_bh;
  r.i = (int)(r.t / g.W);
  r.j = (int)(r.t % g.W);
  return true;
}

// A[q][m], lanes over window positions m; q in registers of every lane (d <= 128 by chunks of 32)
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) qk_rpb_kernel(Geo g, const T *__restrict__ q, const T *__restrict__ k,
                                                            const float *__restrict__ rpb, float *__restrict__ A) {
  Row r;
  if (!row_of(g, (long)g.q_rows * g.W, r)) return;
  const int lane = threadIdx.x % 32, TT = 2 * g.L - 1;
  const int li = wlen(g.H, g.L), lj = wlen(g.W, g.L), nwin = li * lj;
  const int i = r.i + g.q_row0, j = r.j;
  const int si = wstart(i, g.H, g.L), sj = wstart(j, g.W, g.L);
  const T *qr = q + ((size_t)r.bh * g.q_rows * g.W + r.t) * g.d;
  const T *kb = k + (size_t)r.bh * g.kv_rows * g.W * g.d;
  float *ar = A + ((size_t)r.bh * g.q_rows * g.W + r.t) * nwin;
  for (int m = lane; m < nwin; m += 32) {
    const int p = si + m / lj, qq = sj + m % lj;
    const T *kr = kb + ((size_t)(p - g.kv_row0) * g.W + qq) * g.d;
    float dot = 0.f;
    for (int c = 0; c < g.d; ++c) dot = fmaf(to_f32(qr[c]), to_f32(kr[c]), dot);
    const float bias = rpb ? __ldg(&rpb[((size_t)(r.bh % g.heads) * TT + (p - i + g.L - 1)) * TT + (qq - j + g.L - 1)]) : 0.f;
    ar[m] = g.scale * (dot + bias);
  }
}

__global__ void __launch_bounds__(kWarps * 32) softmax_kernel(Geo g, float *__restrict__ A, float *__restrict__ lse) {
  Row r;
  if (!row_of(g, (long)g.q_rows * g.W, r)) return;
  const int lane = threadIdx.x % 32, nwin = wlen(g.H, g.L) * wlen(g.W, g.L);
  const size_t qi = (size_t)r.bh * g.q_rows * g.W + r.t;
  float *ar = A + qi * nwin;
  float mx = -INFINITY;
  for (int m = lane; m < nwin; m += 32) mx = fmaxf(mx, ar[m]);
  mx = warp_max(mx);
  float sum = 0.f;
  for (int m = lane; m < nwin; m += 32) sum += expf(ar[m] - mx);
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  for (int m = lane; m < nwin; m += 32) ar[m] = expf(ar[m] - mx) * inv;
  if (lane == 0 && lse) lse[qi] = mx + logf(sum);
}

// O[q][c] = sum_m A[q][m] v_m[c]; lanes over channels
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) av_kernel(Geo g, const float *__restrict__ A, const T *__restrict__ v,
                                                        T *__restrict__ out) {
  Row r;
  if (!row_of(g, (long)g.q_rows * g.W, r)) return;
  const int lane = threadIdx.x % 32, lj = wlen(g.W, g.L), nwin = wlen(g.H, g.L) * lj;
  const int i = r.i + g.q_row0, si = wstart(i, g.H, g.L), sj = wstart(r.j, g.W, g.L);
  const size_t qi = (size_t)r.bh * g.q_rows * g.W + r.t;
  const float *ar = A + qi * nwin;
  const T *vb = v + (size_t)r.bh * g.kv_rows * g.W * g.d;
  for (int c = lane; c < g.d; c += 32) {
    float acc = 0.f;
    for (int m = 0; m < nwin; ++m) {
      const int p = si + m / lj, qq = sj + m % lj;
      acc = fmaf(ar[m], to_f32(vb[((size_t)(p - g.kv_row0) * g.W + qq) * g.d + c]), acc);
    }
    out[qi * g.d + c] = from_f32<T>(acc);
  }
}

// dA[q][m] = dO_q . v_m (lanes over m), then in place dS = A (dA - sum_m A dA)
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) dattn_kernel(Geo g, const float *__restrict__ A, const T *__restrict__ v,
                                                           const T *__restrict__ dout, float *__restrict__ dS) {
  Row r;
  if (!row_of(g, (long)g.q_rows * g.W, r)) return;
  const int lane = threadIdx.x % 32, lj = wlen(g.W, g.L), nwin = wlen(g.H, g.L) * lj;
  const int i = r.i + g.q_row0, si = wstart(i, g.H, g.L), sj = wstart(r.j, g.W, g.L);
  const size_t qi = (size_t)r.bh * g.q_rows * g.W + r.t;
  const T *dor = dout + qi * g.d;
  const T *vb = v + (size_t)r.bh * g.kv_rows * g.W * g.d;
  const float *ar = A + qi * nwin;
  float *dr = dS + qi * nwin;
  float dot_ad = 0.f;
  for (int m = lane; m < nwin; m += 32) {
    const int p = si + m / lj, qq = sj + m % lj;
    const T *vr = vb + ((size_t)(p - g.kv_row0) * g.W + qq) * g.d;
    float da = 0.f;
    for (int c = 0; c < g.d; ++c) da = fmaf(to_f32(dor[c]), to_f32(vr[c]), da);
    dr[m] = da;
    dot_ad = fmaf(ar[m], da, dot_ad);
  }
  dot_ad = warp_sum(dot_ad);
  for (int m = lane; m < nwin; m += 32) dr[m] = ar[m] * (dr[m] - dot_ad);
}

// dQ[q][c] = scale sum_m dS[q][m] k_m[c]; dB[cell] += scale dS (atomics); lanes over channels
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) dq_kernel(Geo g, const float *__restrict__ dS, const T *__restrict__ k,
                                                        T *__restrict__ dq, float *__restrict__ drpb) {
  Row r;
  if (!row_of(g, (long)g.q_rows * g.W, r)) return;
  const int lane = threadIdx.x % 32, lj = wlen(g.W, g.L), nwin = wlen(g.H, g.L) * lj, TT = 2 * g.L - 1;
  const int i = r.i + g.q_row0, j = r.j, si = wstart(i, g.H, g.L), sj = wstart(j, g.W, g.L);
  const size_t qi = (size_t)r.bh * g.q_rows * g.W + r.t;
  const float *dr = dS + qi * nwin;
  const T *kb = k + (size_t)r.bh * g.kv_rows * g.W * g.d;
  for (int c = lane; c < g.d; c += 32) {
    float acc = 0.f;
    for (int m = 0; m < nwin; ++m) {
      const int p = si + m / lj, qq = sj + m % lj;
      acc = fmaf(dr[m], to_f32(kb[((size_t)(p - g.kv_row0) * g.W + qq) * g.d + c]), acc);
    }
    dq[qi * g.d + c] = from_f32<T>(g.scale * acc);
  }
  if (drpb)
    for (int m = lane; m < nwin; m += 32) {
      const int p = si + m / lj, qq = sj + m % lj;
      atomicAdd(&drpb[((size_t)(r.bh % g.heads) * TT + (p - i + g.L - 1)) * TT + (qq - j + g.L - 1)], g.scale * dr[m]);
    }
}

// dK_p = scale sum dS[q][m(q,p)] q_q, dV_p = sum A[q][m(q,p)] dO_q over the queries whose window
// holds key p (scanned over the (2L-1)^2 candidates); lanes over channels
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) dkdv_kernel(Geo g, const float *__restrict__ A,
                                                          const float *__restrict__ dS, const T *__restrict__ q,
                                                          const T *__restrict__ dout, T *__restrict__ dk,
                                                          T *__restrict__ dv) {
  Row r;
  if (!row_of(g, (long)g.kv_rows * g.W, r)) return;
  const int lane = threadIdx.x % 32, li = wlen(g.H, g.L), lj = wlen(g.W, g.L), nwin = li * lj;
  const int p = r.i + g.kv_row0, pc = r.j;
  const size_t kvi = (size_t)r.bh * g.kv_rows * g.W + r.t;
  const int q_end = g.q_row0 + g.q_rows;
  for (int c = lane; c < g.d; c += 32) {
    float ak = 0.f, av = 0.f;
    for (int i = max(g.q_row0, p - g.L + 1); i <= min(q_end - 1, p + g.L - 1); ++i) {
      const int si = wstart(i, g.H, g.L);
      if (p < si || p >= si + li) continue;
      for (int j = max(0, pc - g.L + 1); j <= min(g.W - 1, pc + g.L - 1); ++j) {
        const int sj = wstart(j, g.W, g.L);
        if (pc < sj || pc >= sj + lj) continue;
        const size_t qi = (size_t)r.bh * g.q_rows * g.W + (size_t)(i - g.q_row0) * g.W + j;
        const int m = (p - si) * lj + (pc - sj);
        ak = fmaf(dS[qi * nwin + m], to_f32(q[qi * g.d + c]), ak);
        av = fmaf(A[qi * nwin + m], to_f32(dout[qi * g.d + c]), av);
      }
    }
    dk[kvi * g.d + c] = from_f32<T>(g.scale * ak);
    dv[kvi * g.d + c] = from_f32<T>(av);
  }
}

unsigned blocks_for(long rows) { return (unsigned)((rows + kWarps - 1) / kWarps); }

template <typename T>
cudaError_t unfused_forward_t(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                              float *lse, float *attn, cudaStream_t st) {
  const long nq = (long)g.B * g.heads * g.q_rows * g.W;
  {
    ProfScope ps("na2d_paper_qk_rpb", st);
    qk_rpb_kernel<T><<<blocks_for(nq), kWarps * 32, 0, st>>>(g, (const T *)q, (const T *)k, rpb, attn);
  }
  {
    ProfScope ps("na2d_paper_softmax", st);
    softmax_kernel<<<blocks_for(nq), kWarps * 32, 0, st>>>(g, attn, lse);
  }
  {
    ProfScope ps("na2d_paper_av", st);
    av_kernel<T><<<blocks_for(nq), kWarps * 32, 0, st>>>(g, attn, (const T *)v, (T *)out);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t unfused_backward_t(const Geo &g, const void *q, const void *k, const void *v, const void *dout,
                               const float *attn, float *dS, void *dq, void *dk, void *dv, float *drpb, cudaStream_t st) {
  const long nq = (long)g.B * g.heads * g.q_rows * g.W, nk = (long)g.B * g.heads * g.kv_rows * g.W;
  if (drpb) {
    const cudaError_t e = cudaMemsetAsync(drpb, 0, sizeof(float) * g.heads * (2 * g.L - 1) * (2 * g.L - 1), st);
    if (e != cudaSuccess) return e;
  }
  {
    ProfScope ps("na2d_paper_dattn", st);
    dattn_kernel<T><<<blocks_for(nq), kWarps * 32, 0, st>>>(g, attn, (const T *)v, (const T *)dout, dS);
  }
  {
    ProfScope ps("na2d_paper_dq", st);
    dq_kernel<T><<<blocks_for(nq), kWarps * 32, 0, st>>>(g, dS, (const T *)k, (T *)dq, drpb);
  }
  {
    ProfScope ps("na2d_paper_dkdv", st);
    dkdv_kernel<T><<<blocks_for(nk), kWarps * 32, 0, st>>>(g, attn, dS, (const T *)q, (const T *)dout, (T *)dk,
                                                           (T *)dv);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t unfused_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                            float *lse, float *attn, cudaStream_t st) {
  if (g.dtype == NA2D_F16) return unfused_forward_t<__half>(g, q, k, v, rpb, out, lse, attn, st);
  return g.dtype == NA2D_F32 ? unfused_forward_t<float>(g, q, k, v, rpb, out, lse, attn, st)
                             : unfused_forward_t<__nv_bfloat16>(g, q, k, v, rpb, out, lse, attn, st);
}

cudaError_t unfused_backward(const Geo &g, const void *q, const void *k, const void *v, const void *dout,
                             const float *attn, float *dS, void *dq, void *dk, void *dv, float *drpb, cudaStream_t st) {
  if (g.dtype == NA2D_F16) return unfused_backward_t<__half>(g, q, k, v, dout, attn, dS, dq, dk, dv, drpb, st);
  return g.dtype == NA2D_F32 ? unfused_backward_t<float>(g, q, k, v, dout, attn, dS, dq, dk, dv, drpb, st)
                             : unfused_backward_t<__nv_bfloat16>(g, q, k, v, dout, attn, dS, dq, dk, dv, drpb, st);
}

}  // namespace na2d
