// na2d_simt.cu -- SIMT (CUDA-core FFMA) NA2D kernels.
//
// Used for the fp32 path (1e-4 relative parity forbids TF32 tensor cores) and for bf16 shapes
// the tcgen05 kernels do not cover (dim != 32, L > 7, ...).  One thread per query (forward,
// dQ) or per key (dK/dV); operands stream through L1/L2.  Every step is Eq. 2 and its
// analytic gradient, in fp32:
//   forward  s_m = scale (q.k_m + B[cell_m]); online max/sum; O = sum P_m v_m; LSE = m + log l
//   D        = dO . O                                       (a6)
//   dQ, dB   dS_m = P_m (dO.v_m - D); dQ = scale sum dS_m k_m; dB[cell_m] += scale dS_m (a7,a9,a10)
//   dK, dV   over the inverse neighbourhood of each key (a8)
#include <math.h>

#include "na2d_internal.cuh"
#include "na2d_profile.cuh"

namespace na2d {
namespace {

constexpr int kThreads = 128;

template <typename T, int DMAX>
__global__ void __launch_bounds__(kThreads) fwd_simt(Geo g, const T *__restrict__ q,
                                                     const T *__restrict__ k,
                                                     const T *__restrict__ v,
                                                     const float *__restrict__ rpb,
                                                     T *__restrict__ out, float *__restrict__ lse) {
  const int TT = 2 * g.L - 1;
  const long nq = (long)g.q_rows * g.W;
  const int li = wlen(g.H, g.L), lj = wlen(g.W, g.L);
  for (int bh = blockIdx.y; bh < g.B * g.heads; bh += gridDim.y) {
    const int h = bh % g.heads;
    const T *kb = k + (size_t)bh * g.kv_rows * g.W * g.d;
    const T *vb = v + (size_t)bh * g.kv_rows * g.W * g.d;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += (long)gridDim.x * blockDim.x) {
      const int i = (int)(t / g.W) + g.q_row0, j = (int)(t % g.W);
      const size_t qi = (size_t)bh * nq + t;
      float qv[DMAX], acc[DMAX];
#pragma unroll
      for (int c = 0; c < DMAX; ++c) {
        qv[c] = c < g.d ? to_f32(q[qi * g.d + c]) : 0.f;
        acc[c] = 0.f;
      }
      const int si = wstart(i, g.H, g.L), sj = wstart(j, g.W, g.L);
      float m = -INFINITY, l = 0.f;
      for (int p = si; p < si + li; ++p) {
        for (int qq = sj; qq < sj + lj; ++qq) {
          const size_t kidx = ((size_t)(p - g.kv_row0) * g.W + qq) * g.d;
          float dot = 0.f;
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < g.d) dot = fmaf(qv[c], to_f32(kb[kidx + c]), dot);
          const float bias = rpb ? __ldg(&rpb[((size_t)h * TT + (p - i + g.L - 1)) * TT + (qq - j + g.L - 1)]) : 0.f;
          const float s = g.scale * (dot + bias);
          const float mn = fmaxf(m, s);
          const float corr = expf(m - mn);  // exp(-inf) = 0 on the first key
          const float e = expf(s - mn);
          l = l * corr + e;
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < g.d) acc[c] = acc[c] * corr + e * to_f32(vb[kidx + c]);
          m = mn;
        }
      }
      const float inv = 1.f / l;
#pragma unroll
      for (int c = 0; c < DMAX; ++c)
        if (c < g.d) out[qi * g.d + c] = from_f32<T>(acc[c] * inv);
      if (lse) lse[qi] = m + logf(l);
    }
  }
}

// a6: D = rowsum(dO * O) in fp32
template <typename T>
__global__ void __launch_bounds__(256) delta_simt(long nq, int d, const T *__restrict__ out,
                                                  const T *__restrict__ dout, float *__restrict__ D) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += (long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < d; ++c) s = fmaf(to_f32(dout[t * d + c]), to_f32(out[t * d + c]), s);
    D[t] = s;
  }
}

// a7, a9, a10: thread per query
template <typename T, int DMAX>
__global__ void __launch_bounds__(kThreads) dq_simt(Geo g, const T *__restrict__ q, const T *__restrict__ k,
                                                    const T *__restrict__ v, const float *__restrict__ rpb,
                                                    const float *__restrict__ lse, const T *__restrict__ dout,
                                                    const float *__restrict__ D, T *__restrict__ dq,
                                                    float *__restrict__ ds_slots) {
  // ds_slots (when the problem has a bias table): scale * dS of query qi, window slot (p - si, q - sj)
  // at [qi * L * L + slot]; drpb_reduce sums them per cell in a fixed order (no atomics)
  const int TT = 2 * g.L - 1;
  const long nq = (long)g.q_rows * g.W;
  const int li = wlen(g.H, g.L), lj = wlen(g.W, g.L);
  for (int bh = blockIdx.y; bh < g.B * g.heads; bh += gridDim.y) {
    const int h = bh % g.heads;
    const T *kb = k + (size_t)bh * g.kv_rows * g.W * g.d;
    const T *vb = v + (size_t)bh * g.kv_rows * g.W * g.d;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += (long)gridDim.x * blockDim.x) {
      const int i = (int)(t / g.W) + g.q_row0, j = (int)(t % g.W);
      const size_t qi = (size_t)bh * nq + t;
      float qv[DMAX], dov[DMAX], acc[DMAX];
#pragma unroll
      for (int c = 0; c < DMAX; ++c) {
        qv[c] = c < g.d ? to_f32(q[qi * g.d + c]) : 0.f;
        dov[c] = c < g.d ? to_f32(dout[qi * g.d + c]) : 0.f;
        acc[c] = 0.f;
      }
      const float L_ = lse[qi], Dq = D[qi];
      const int si = wstart(i, g.H, g.L), sj = wstart(j, g.W, g.L);
      for (int p = si; p < si + li; ++p) {
        for (int qq = sj; qq < sj + lj; ++qq) {
          const size_t kidx = ((size_t)(p - g.kv_row0) * g.W + qq) * g.d;
          float dot = 0.f, dp = 0.f;
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < g.d) {
              dot = fmaf(qv[c], to_f32(kb[kidx + c]), dot);
              dp = fmaf(dov[c], to_f32(vb[kidx + c]), dp);
            }
          const int cell = (p - i + g.L - 1) * TT + (qq - j + g.L - 1);
          const float bias = rpb ? __ldg(&rpb[(size_t)h * TT * TT + cell]) : 0.f;
          const float P = expf(g.scale * (dot + bias) - L_);
          const float dS = P * (dp - Dq);
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < g.d) acc[c] = fmaf(dS, to_f32(kb[kidx + c]), acc[c]);
          if (rpb) ds_slots[qi * g.L * g.L + (p - si) * g.L + (qq - sj)] = g.scale * dS;
        }
      }
#pragma unroll
      for (int c = 0; c < DMAX; ++c)
        if (c < g.d) dq[qi * g.d + c] = from_f32<T>(g.scale * acc[c]);
    }
  }
}

// a10: dB[h][a][c] = sum over (b, i, j) of scale * dS at the window slot whose key is
// (i + a - L + 1, j + c - L + 1), one block per (head, cell): strided partial sums in a fixed order,
// then a fixed shared-memory tree (bitwise reproducible for a given launch configuration)
__global__ void __launch_bounds__(256) drpb_reduce_simt(Geo g, const float *__restrict__ ds_slots,
                                                        float *__restrict__ drpb) {
  __shared__ float red[256];
  const int TT = 2 * g.L - 1;
  const int h = blockIdx.x / (TT * TT), cell = blockIdx.x % (TT * TT);
  const int ro = cell / TT - (g.L - 1), co = cell % TT - (g.L - 1);  // key - query offsets
  const int li = wlen(g.H, g.L), lj = wlen(g.W, g.L);
  const long nq = (long)g.q_rows * g.W;
  float acc = 0.f;
  for (long t = threadIdx.x; t < (long)g.B * nq; t += 256) {
    const int b = (int)(t / nq);
    const long r = t - (long)b * nq;
    const int i = (int)(r / g.W) + g.q_row0, j = (int)(r % g.W);
    const int p = i + ro, qq = j + co;
    const int si = wstart(i, g.H, g.L), sj = wstart(j, g.W, g.L);
    if (p >= si && p < si + li && qq >= sj && qq < sj + lj) {
      const size_t qi = ((size_t)b * g.heads + h) * nq + r;
      acc += ds_slots[qi * g.L * g.L + (p - si) * g.L + (qq - sj)];
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) drpb[(size_t)h * TT * TT + cell] = red[0];
}

// a8: thread per key, looping over the queries whose window contains it (|i - p| <= L - 1).
template <typename T, int DMAX>
__global__ void __launch_bounds__(kThreads) dkdv_simt(Geo g, const T *__restrict__ q, const T *__restrict__ k,
                                                      const T *__restrict__ v, const float *__restrict__ rpb,
                                                      const float *__restrict__ lse, const T *__restrict__ dout,
                                                      const float *__restrict__ D, T *__restrict__ dk,
                                                      T *__restrict__ dv) {
  const int TT = 2 * g.L - 1;
  const long nk = (long)g.kv_rows * g.W, nq = (long)g.q_rows * g.W;
  const int li = wlen(g.H, g.L), lj = wlen(g.W, g.L);
  for (int bh = blockIdx.y; bh < g.B * g.heads; bh += gridDim.y) {
    const int h = bh % g.heads;
    const T *qb = q + (size_t)bh * nq * g.d;
    const T *dob = dout + (size_t)bh * nq * g.d;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < nk; t += (long)gridDim.x * blockDim.x) {
      const int p = (int)(t / g.W) + g.kv_row0, qq = (int)(t % g.W);
      const size_t ki = (size_t)bh * nk + t;
      float kv[DMAX], vv[DMAX], ak[DMAX], av[DMAX];
#pragma unroll
      for (int c = 0; c < DMAX; ++c) {
        kv[c] = c < g.d ? to_f32(k[ki * g.d + c]) : 0.f;
        vv[c] = c < g.d ? to_f32(v[ki * g.d + c]) : 0.f;
        ak[c] = av[c] = 0.f;
      }
      const int i0 = max(g.q_row0, p - g.L + 1), i1 = min(g.q_row0 + g.q_rows - 1, p + g.L - 1);
      const int j0 = max(0, qq - g.L + 1), j1 = min(g.W - 1, qq + g.L - 1);
      for (int i = i0; i <= i1; ++i) {
        const int si = wstart(i, g.H, g.L);
        if (p < si || p >= si + li) continue;
        for (int j = j0; j <= j1; ++j) {
          const int sj = wstart(j, g.W, g.L);
          if (qq < sj || qq >= sj + lj) continue;
          const size_t qi = (size_t)(i - g.q_row0) * g.W + j;
          float dot = 0.f, dp = 0.f;
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < g.d) {
              dot = fmaf(to_f32(qb[qi * g.d + c]), kv[c], dot);
              dp = fmaf(to_f32(dob[qi * g.d + c]), vv[c], dp);
            }
          const float bias = rpb ? __ldg(&rpb[((size_t)h * TT + (p - i + g.L - 1)) * TT + (qq - j + g.L - 1)]) : 0.f;
          const size_t qg = (size_t)bh * nq + qi;
          const float P = expf(g.scale * (dot + bias) - lse[qg]);
          const float dS = P * (dp - D[qg]);
#pragma unroll
          for (int c = 0; c < DMAX; ++c)
            if (c < g.d) {
              av[c] = fmaf(P, to_f32(dob[qi * g.d + c]), av[c]);
              ak[c] = fmaf(dS, to_f32(qb[qi * g.d + c]), ak[c]);
            }
        }
      }
#pragma unroll
      for (int c = 0; c < DMAX; ++c)
        if (c < g.d) {
          dk[ki * g.d + c] = from_f32<T>(g.scale * ak[c]);
          dv[ki * g.d + c] = from_f32<T>(av[c]);
        }
    }
  }
}

dim3 grid_for(long n, int units) {
  long bx = (n + kThreads - 1) / kThreads;
  if (bx > 4096) bx = 4096;
  int by = units < 65535 ? units : 65535;
  return dim3((unsigned)bx, (unsigned)by);
}

template <typename T, int DMAX>
cudaError_t fwd_t(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                  float *lse, cudaStream_t st) {
  ProfScope ps("na2d_fwd_simt", st);
  fwd_simt<T, DMAX><<<grid_for((long)g.q_rows * g.W, g.B * g.heads), kThreads, 0, st>>>(
      g, (const T *)q, (const T *)k, (const T *)v, rpb, (T *)out, lse);
  return cudaGetLastError();
}

template <typename T, int DMAX>
cudaError_t bwd_t(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const void *out,
                  const float *lse, const void *dout, void *dq, void *dk, void *dv, float *drpb, float *D,
                  float *ds_slots, cudaStream_t st) {
  const long nq = (long)g.B * g.heads * g.q_rows * g.W;
  const int TT = 2 * g.L - 1;
  long nb = (nq + 255) / 256;
  {
  ProfScope ps("na2d_bwd_delta", st);
  delta_simt<T><<<(unsigned)(nb > 8192 ? 8192 : nb), 256, 0, st>>>(nq, g.d, (const T *)out, (const T *)dout, D);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  {
  ProfScope ps("na2d_bwd_dq_simt", st);
  dq_simt<T, DMAX><<<grid_for((long)g.q_rows * g.W, g.B * g.heads), kThreads, 0, st>>>(
      g, (const T *)q, (const T *)k, (const T *)v, rpb, lse, (const T *)dout, D, (T *)dq, ds_slots);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (rpb) {
    ProfScope ps("na2d_bwd_drpb_simt", st);
    drpb_reduce_simt<<<g.heads * TT * TT, 256, 0, st>>>(g, ds_slots, drpb);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  ProfScope ps("na2d_bwd_dkdv_simt", st);
  dkdv_simt<T, DMAX><<<grid_for((long)g.kv_rows * g.W, g.B * g.heads), kThreads, 0, st>>>(
      g, (const T *)q, (const T *)k, (const T *)v, rpb, lse, (const T *)dout, D, (T *)dk, (T *)dv);
  return cudaGetLastError();
}

template <typename T, int DMAX>
cudaError_t dkdv_t(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const float *lse,
                   const void *dout, const float *D, void *dk, void *dv, cudaStream_t st) {
  ProfScope ps("na2d_bwd_dkdv_simt", st);
  dkdv_simt<T, DMAX><<<grid_for((long)g.kv_rows * g.W, g.B * g.heads), kThreads, 0, st>>>(
      g, (const T *)q, (const T *)k, (const T *)v, rpb, lse, (const T *)dout, D, (T *)dk, (T *)dv);
  return cudaGetLastError();
}

}  // namespace

#define NA2D_DISPATCH_D(FN, T, ...)              \
  (g.d <= 16    ? FN<T, 16>(__VA_ARGS__)          \
   : g.d <= 32  ? FN<T, 32>(__VA_ARGS__)          \
   : g.d <= 64  ? FN<T, 64>(__VA_ARGS__)          \
                : FN<T, 128>(__VA_ARGS__))

cudaError_t simt_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                         float *lse, cudaStream_t st) {
  if (g.dtype == NA2D_F32) return NA2D_DISPATCH_D(fwd_t, float, g, q, k, v, rpb, out, lse, st);
  if (g.dtype == NA2D_F16) return NA2D_DISPATCH_D(fwd_t, __half, g, q, k, v, rpb, out, lse, st);
  return NA2D_DISPATCH_D(fwd_t, __nv_bfloat16, g, q, k, v, rpb, out, lse, st);
}

cudaError_t simt_backward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                          const void *out, const float *lse, const void *dout, void *dq, void *dk, void *dv,
                          float *drpb, float *D, float *ds_slots, cudaStream_t st) {
  if (g.dtype == NA2D_F32)
    return NA2D_DISPATCH_D(bwd_t, float, g, q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, D, ds_slots, st);
  if (g.dtype == NA2D_F16)
    return NA2D_DISPATCH_D(bwd_t, __half, g, q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, D, ds_slots, st);
  return NA2D_DISPATCH_D(bwd_t, __nv_bfloat16, g, q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, D, ds_slots, st);
}

size_t simt_backward_scratch_bytes(const Geo &g) {
  return sizeof(float) * (size_t)g.B * g.heads * g.q_rows * g.W * g.L * g.L;
}

int simt_launches(const Geo &, int which) { return which == 0 ? 1 : 4; }

cudaError_t simt_backward_dkdv(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                               const float *lse, const void *dout, const float *D, void *dk, void *dv,
                               cudaStream_t st) {
  if (g.dtype == NA2D_F32) return NA2D_DISPATCH_D(dkdv_t, float, g, q, k, v, rpb, lse, dout, D, dk, dv, st);
  if (g.dtype == NA2D_F16) return NA2D_DISPATCH_D(dkdv_t, __half, g, q, k, v, rpb, lse, dout, D, dk, dv, st);
  return NA2D_DISPATCH_D(dkdv_t, __nv_bfloat16, g, q, k, v, rpb, lse, dout, D, dk, dv, st);
}

}  // namespace na2d
