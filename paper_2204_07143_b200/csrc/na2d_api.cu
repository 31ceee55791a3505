// na2d_api.cu -- the C ABI declared in include/na2d.h: argument validation, workspace
// layout, kernel-family dispatch and the host-buffer end-to-end step.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "na2d_internal.cuh"
#include "na2d_tc.cuh"

namespace na2d {
namespace {

constexpr int kMaxKernel = 31;  // SIMT dRPB staging bound ((2L-1)^2 floats of shared memory)

bool aligned16(const void *p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

// Synchronous validation; fills g on success.
na2d_status make_geo(const na2d_problem *p, Geo *g) {
  if (!p) return NA2D_ERR_NULL_POINTER;
  if (p->dtype != NA2D_BF16 && p->dtype != NA2D_F32 && p->dtype != NA2D_F16) return NA2D_ERR_DTYPE;
  if (p->kernel_size < 3 || (p->kernel_size % 2) == 0) return NA2D_ERR_KERNEL_SIZE;
  if (p->batch <= 0 || p->heads <= 0 || p->height <= 0 || p->width <= 0 || p->dim <= 0) return NA2D_ERR_SHAPE;
  if (!(isfinite(p->scale) && p->scale > 0.f)) return NA2D_ERR_INVALID_ARG;
  if (p->dim > 128 || (p->dim % 2) != 0 || p->kernel_size > kMaxKernel) return NA2D_ERR_UNSUPPORTED;
  g->B = p->batch;
  g->heads = p->heads;
  g->W = p->width;
  g->d = p->dim;
  g->L = p->kernel_size;
  g->scale = p->scale;
  g->dtype = p->dtype;
  g->q_rows = p->height;
  g->q_row0 = p->q_row0;
  g->H = p->map_height > 0 ? p->map_height : p->height;
  g->kv_row0 = p->kv_row0;
  g->kv_rows = p->kv_rows > 0 ? p->kv_rows : p->height;
  if (p->map_height < 0 || p->kv_rows < 0) return NA2D_ERR_SHAPE;
  if (g->q_row0 < 0 || g->q_row0 + g->q_rows > g->H) return NA2D_ERR_SHAPE;
  if (g->kv_row0 < 0 || g->kv_row0 + g->kv_rows > g->H) return NA2D_ERR_SHAPE;
  // every held query row's window must lie inside the held K/V rows (monotone starts)
  const int s0 = wstart(g->q_row0, g->H, g->L);
  const int s1 = wstart(g->q_row0 + g->q_rows - 1, g->H, g->L) + wlen(g->H, g->L);
  if (s0 < g->kv_row0 || s1 > g->kv_row0 + g->kv_rows) return NA2D_ERR_SHAPE;
  // 64-bit element counts must stay far from overflow
  const double elems = (double)g->B * g->heads * (double)(g->q_rows > g->kv_rows ? g->q_rows : g->kv_rows) *
                       g->W * g->d;
  if (elems > 9.0e15 || (double)g->B * g->heads > 2147483647.0) return NA2D_ERR_SHAPE;
  return NA2D_OK;
}

size_t elem_size(const Geo &g) { return g.dtype == NA2D_F32 ? 4 : 2; }
size_t n_query(const Geo &g) { return (size_t)g.B * g.heads * g.q_rows * g.W; }
size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

bool force_simt() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("NA2D_FORCE_SIMT");
    v = (e && e[0] && e[0] != '0') ? 1 : 0;
  }
  return v == 1;
}

bool use_tc(const Geo &g, int which) {
  if (force_simt()) return false;
  return which == 0 ? tc_forward_supported(g) : tc_backward_supported(g);
}

// Workspace: [D fp32 per query | tensor-core backward scratch, or the SIMT path's per-query window-slot dS]
size_t bwd_ws(const Geo &g) {
  size_t b = align_up(n_query(g) * sizeof(float));
  b += align_up(use_tc(g, 1) ? tc_backward_scratch_bytes(g) : simt_backward_scratch_bytes(g));
  return b;
}

thread_local cudaError_t t_last_cuda_error = cudaSuccess;

na2d_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return NA2D_OK;
  t_last_cuda_error = e;
  return NA2D_ERR_CUDA;
}

}  // namespace
}  // namespace na2d

using namespace na2d;

extern "C" {

const char *na2d_status_string(na2d_status s) {
  switch (s) {
    case NA2D_OK: return "ok";
    case NA2D_ERR_NULL_POINTER: return "a required pointer is NULL";
    case NA2D_ERR_KERNEL_SIZE: return "kernel_size must be odd and >= 3 (PAPER App. A: odd number greater than 1)";
    case NA2D_ERR_SHAPE: return "invalid shape (dimension <= 0, overflow, or band misses needed K/V rows)";
    case NA2D_ERR_DTYPE: return "dtype must be NA2D_BF16, NA2D_F32 or NA2D_F16";
    case NA2D_ERR_UNSUPPORTED: return "unsupported problem (dim must be even and <= 128, kernel_size <= 31)";
    case NA2D_ERR_ALIGNMENT: return "tensor base pointers must be 16-byte aligned";
    case NA2D_ERR_WORKSPACE: return "workspace smaller than na2d_backward_workspace_bytes()";
    case NA2D_ERR_INVALID_ARG: return "invalid argument (scale must be finite and > 0; drpb must be NULL iff rpb is NULL)";
    case NA2D_ERR_CUDA: return "CUDA runtime error";
  }
  return "unknown status";
}

int na2d_version(void) { return NA2D_VERSION; }

const char *na2d_last_cuda_error(void) { return cudaGetErrorString(t_last_cuda_error); }

na2d_status na2d_forward(const na2d_problem *p, const void *q, const void *k, const void *v, const float *rpb,
                         void *out, float *lse, void *stream) {
  Geo g;
  na2d_status s = make_geo(p, &g);
  if (s != NA2D_OK) return s;
  if (!q || !k || !v || !out) return NA2D_ERR_NULL_POINTER;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out) || !aligned16(lse) || !aligned16(rpb))
    return NA2D_ERR_ALIGNMENT;
  cudaStream_t st = (cudaStream_t)stream;
  (void)cudaGetLastError();  // a non-sticky error left by an unrelated earlier runtime call is not ours
  if (use_tc(g, 0)) return cuda_status(tc_forward(g, q, k, v, rpb, out, lse, st));
  return cuda_status(simt_forward(g, q, k, v, rpb, out, lse, st));
}

size_t na2d_backward_workspace_bytes(const na2d_problem *p) {
  Geo g;
  if (make_geo(p, &g) != NA2D_OK) return 0;
  return bwd_ws(g);
}

na2d_status na2d_backward(const na2d_problem *p, const void *q, const void *k, const void *v, const float *rpb,
                          const void *out, const float *lse, const void *dout, void *dq, void *dk, void *dv,
                          float *drpb, void *workspace, size_t workspace_bytes, void *stream) {
  Geo g;
  na2d_status s = make_geo(p, &g);
  if (s != NA2D_OK) return s;
  if (!q || !k || !v || !out || !lse || !dout || !dq || !dk || !dv) return NA2D_ERR_NULL_POINTER;
  if ((rpb == nullptr) != (drpb == nullptr)) return NA2D_ERR_INVALID_ARG;
  const size_t need = bwd_ws(g);
  if (workspace_bytes < need) return NA2D_ERR_WORKSPACE;
  if (!workspace) return NA2D_ERR_NULL_POINTER;
  const void *ptrs[] = {q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, workspace};
  for (const void *ptr : ptrs)
    if (!aligned16(ptr)) return NA2D_ERR_ALIGNMENT;
  cudaStream_t st = (cudaStream_t)stream;
  (void)cudaGetLastError();  // a non-sticky error left by an unrelated earlier runtime call is not ours
  float *D = (float *)workspace;
  if (use_tc(g, 1)) {
    void *scratch = (char *)workspace + align_up(n_query(g) * sizeof(float));
    return cuda_status(tc_backward(g, q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, D, scratch, st));
  }
  float *ds_slots = (float *)((char *)workspace + align_up(n_query(g) * sizeof(float)));
  return cuda_status(simt_backward(g, q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, D, ds_slots, st));
}

size_t na2d_paper_attn_bytes(const na2d_problem *p) {
  Geo g;
  if (make_geo(p, &g) != NA2D_OK) return 0;
  return n_query(g) * (size_t)wlen(g.H, g.L) * wlen(g.W, g.L) * sizeof(float);
}

na2d_status na2d_paper_forward(const na2d_problem *p, const void *q, const void *k, const void *v, const float *rpb,
                               void *out, float *lse, float *attn, void *stream) {
  Geo g;
  na2d_status s = make_geo(p, &g);
  if (s != NA2D_OK) return s;
  if (!q || !k || !v || !out || !lse || !attn) return NA2D_ERR_NULL_POINTER;
  const void *ptrs[] = {q, k, v, rpb, out, lse, attn};
  for (const void *ptr : ptrs)
    if (!aligned16(ptr)) return NA2D_ERR_ALIGNMENT;
  (void)cudaGetLastError();
  return cuda_status(unfused_forward(g, q, k, v, rpb, out, lse, attn, (cudaStream_t)stream));
}

na2d_status na2d_paper_backward(const na2d_problem *p, const void *q, const void *k, const void *v, const void *dout,
                                const float *attn, float *dS, void *dq, void *dk, void *dv, float *drpb,
                                void *stream) {
  Geo g;
  na2d_status s = make_geo(p, &g);
  if (s != NA2D_OK) return s;
  if (!q || !k || !v || !dout || !attn || !dS || !dq || !dk || !dv) return NA2D_ERR_NULL_POINTER;
  const void *ptrs[] = {q, k, v, dout, attn, dS, dq, dk, dv, drpb};
  for (const void *ptr : ptrs)
    if (!aligned16(ptr)) return NA2D_ERR_ALIGNMENT;
  (void)cudaGetLastError();
  return cuda_status(unfused_backward(g, q, k, v, dout, attn, dS, dq, dk, dv, drpb, (cudaStream_t)stream));
}

}  // extern "C" (reopened below)

namespace na2d {
namespace {

#ifndef NA2D_HOST_CHUNKS
#define NA2D_HOST_CHUNKS 16
#endif
constexpr int kHostChunks = NA2D_HOST_CHUNKS;  // batch chunks of the pipelined host step

// Per (host thread, device): the three non-blocking streams of the pipelined host step and its
// events, created on first use and kept (no per-call allocation).
struct HostPipe {
  int dev = -1;
  cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
  cudaEvent_t start = nullptr, done = nullptr, drpb_ready = nullptr;
  cudaEvent_t in_ev[kHostChunks] = {}, comp_ev[kHostChunks] = {};
};
cudaError_t host_pipe(HostPipe **pp) {
  static thread_local HostPipe pipes[8];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  HostPipe &hp = pipes[dev & 7];
  if (hp.dev != dev) {
    const unsigned fl = cudaStreamNonBlocking, ef = cudaEventDisableTiming;
    if ((e = cudaStreamCreateWithFlags(&hp.in, fl)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&hp.comp, fl)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&hp.out, fl)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&hp.start, ef)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&hp.done, ef)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&hp.drpb_ready, ef)) != cudaSuccess) return e;
    for (int c = 0; c < kHostChunks; ++c) {
      if ((e = cudaEventCreateWithFlags(&hp.in_ev[c], ef)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&hp.comp_ev[c], ef)) != cudaSuccess) return e;
    }
    hp.dev = dev;
  }
  *pp = &hp;
  return cudaSuccess;
}

// drpb = sum over chunks of the per-chunk tables, in chunk order (deterministic)
__global__ void sum_tables_kernel(const float *__restrict__ parts, int nparts, size_t stride, int n,
                                  float *__restrict__ dst) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int c = 0; c < nparts; ++c) acc += parts[(size_t)c * stride + e];
    dst[e] = acc;
  }
}

// Chunks are whole groups of `gran` images, so every chunk's tensor and LSE offsets stay
// 16-byte aligned (the kernels' TMA descriptors need it).
int host_gran(const Geo &g) {
  const size_t per_img = (size_t)g.heads * g.q_rows * g.W, img_bytes = per_img * g.d * (g.dtype == NA2D_F32 ? 4 : 2);
  for (int gr = 1; gr < 4; gr *= 2)
    if ((gr * per_img) % 4 == 0 && (gr * img_bytes) % 16 == 0) return gr;
  return 4;
}
int host_chunks(const Geo &g) {
  const int units = (g.B + host_gran(g) - 1) / host_gran(g);
  return units < kHostChunks ? units : kHostChunks;
}
int host_chunk_b0(const Geo &g, int c) {  // first image of chunk c (c = host_chunks(g) -> B)
  const int gr = host_gran(g), units = (g.B + gr - 1) / gr, nc = host_chunks(g);
  const int b = gr * (int)((long)units * c / nc);
  return b < g.B ? b : g.B;
}
// per-chunk dRPB table stride in floats (16-byte aligned)
size_t host_tbl_stride(const Geo &g) { return ((size_t)g.heads * (2 * g.L - 1) * (2 * g.L - 1) + 3) & ~(size_t)3; }

}  // namespace
}  // namespace na2d

extern "C" {

size_t na2d_step_host_workspace_bytes(const na2d_problem *p) {
  Geo g;
  if (make_geo(p, &g) != NA2D_OK) return 0;
  if (g.q_rows != g.H || g.kv_rows != g.H) return 0;
  const size_t t = align_up(n_query(g) * g.d * elem_size(g));
  const size_t TT = 2 * g.L - 1;
  // q k v dout out dq dk dv | lse | rpb drpb | per-chunk drpb | backward workspace (one chunk at a time)
  return 8 * t + align_up(n_query(g) * sizeof(float)) + 2 * align_up(g.heads * TT * TT * sizeof(float)) +
         align_up(host_chunks(g) * host_tbl_stride(g) * sizeof(float)) + bwd_ws(g);
}

na2d_status na2d_step_host(const na2d_problem *p, const void *q, const void *k, const void *v, const float *rpb,
                           const void *dout, void *out, float *lse, void *dq, void *dk, void *dv, float *drpb,
                           void *device_workspace, size_t workspace_bytes, void *stream) {
  Geo g;
  na2d_status s = make_geo(p, &g);
  if (s != NA2D_OK) return s;
  if (g.q_rows != g.H || g.kv_rows != g.H || g.q_row0 || g.kv_row0) return NA2D_ERR_SHAPE;
  if (!q || !k || !v || !dout || !out || !lse || !dq || !dk || !dv || !device_workspace) return NA2D_ERR_NULL_POINTER;
  if ((rpb == nullptr) != (drpb == nullptr)) return NA2D_ERR_INVALID_ARG;
  const size_t need = na2d_step_host_workspace_bytes(p);
  if (workspace_bytes < need) return NA2D_ERR_WORKSPACE;
  if (!aligned16(device_workspace)) return NA2D_ERR_ALIGNMENT;
  cudaStream_t st = (cudaStream_t)stream;
  (void)cudaGetLastError();  // a non-sticky error left by an unrelated earlier runtime call is not ours
  const size_t bytes = n_query(g) * g.d * elem_size(g);
  const size_t t = align_up(bytes);
  const size_t TT = 2 * g.L - 1;
  const size_t tbl = g.heads * TT * TT;
  const size_t tb = tbl * sizeof(float);
  char *w = (char *)device_workspace;
  char *dq_ = w, *dk_ = w + t, *dv_ = w + 2 * t, *dout_ = w + 3 * t, *out_ = w + 4 * t;
  char *q_ = w + 5 * t, *k_ = w + 6 * t, *v_ = w + 7 * t;
  float *lse_ = (float *)(w + 8 * t);
  float *rpb_ = (float *)(w + 8 * t + align_up(n_query(g) * sizeof(float)));
  float *drpb_ = (float *)((char *)rpb_ + align_up(tb));
  const int nc = host_chunks(g);
  float *drpb_parts = (float *)((char *)drpb_ + align_up(tb));
  const size_t tstride = host_tbl_stride(g);
  char *ws = (char *)drpb_parts + align_up(nc * tstride * sizeof(float));
  HostPipe *hp = nullptr;
  cudaError_t e = host_pipe(&hp);
  if (e != cudaSuccess) return cuda_status(e);
#define NA2D_TRY(x)                              \
  do {                                           \
    e = (x);                                     \
    if (e != cudaSuccess) return cuda_status(e); \
  } while (0)
  // Pipelined over batch chunks on three streams: copies in (H2D) for chunk c + 1 and copies out
  // (D2H) for chunk c - 1 run on the copy engines while chunk c computes; ordered after the
  // caller's prior work on `stream`, and `stream` waits for the last copy.
  NA2D_TRY(cudaEventRecord(hp->start, st));
  NA2D_TRY(cudaStreamWaitEvent(hp->in, hp->start, 0));
  NA2D_TRY(cudaStreamWaitEvent(hp->comp, hp->start, 0));
  NA2D_TRY(cudaStreamWaitEvent(hp->out, hp->start, 0));
  if (rpb) NA2D_TRY(cudaMemcpyAsync(rpb_, rpb, tb, cudaMemcpyHostToDevice, hp->in));
  const size_t per_img = bytes / g.B, lse_per_img = (size_t)g.heads * g.q_rows * g.W * sizeof(float);
  for (int c = 0; c < nc; ++c) {
    const int b0 = host_chunk_b0(g, c), b1 = host_chunk_b0(g, c + 1);
    if (b1 <= b0) continue;
    const size_t off = (size_t)b0 * per_img, n = (size_t)(b1 - b0) * per_img;
    const size_t loff = (size_t)b0 * lse_per_img, ln = (size_t)(b1 - b0) * lse_per_img;
    NA2D_TRY(cudaMemcpyAsync(q_ + off, (const char *)q + off, n, cudaMemcpyHostToDevice, hp->in));
    NA2D_TRY(cudaMemcpyAsync(k_ + off, (const char *)k + off, n, cudaMemcpyHostToDevice, hp->in));
    NA2D_TRY(cudaMemcpyAsync(v_ + off, (const char *)v + off, n, cudaMemcpyHostToDevice, hp->in));
    NA2D_TRY(cudaMemcpyAsync(dout_ + off, (const char *)dout + off, n, cudaMemcpyHostToDevice, hp->in));
    NA2D_TRY(cudaEventRecord(hp->in_ev[c], hp->in));
    NA2D_TRY(cudaStreamWaitEvent(hp->comp, hp->in_ev[c], 0));
    na2d_problem pc = *p;
    pc.batch = b1 - b0;
    s = na2d_forward(&pc, q_ + off, k_ + off, v_ + off, rpb ? rpb_ : nullptr, out_ + off,
                     (float *)((char *)lse_ + loff), hp->comp);
    if (s != NA2D_OK) return s;
    s = na2d_backward(&pc, q_ + off, k_ + off, v_ + off, rpb ? rpb_ : nullptr, out_ + off,
                      (float *)((char *)lse_ + loff), dout_ + off, dq_ + off, dk_ + off, dv_ + off,
                      rpb ? drpb_parts + c * tstride : nullptr, ws, bwd_ws(g), hp->comp);
    if (s != NA2D_OK) return s;
    NA2D_TRY(cudaEventRecord(hp->comp_ev[c], hp->comp));
    NA2D_TRY(cudaStreamWaitEvent(hp->out, hp->comp_ev[c], 0));
    NA2D_TRY(cudaMemcpyAsync((char *)out + off, out_ + off, n, cudaMemcpyDeviceToHost, hp->out));
    NA2D_TRY(cudaMemcpyAsync((char *)lse + loff, (char *)lse_ + loff, ln, cudaMemcpyDeviceToHost, hp->out));
    NA2D_TRY(cudaMemcpyAsync((char *)dq + off, dq_ + off, n, cudaMemcpyDeviceToHost, hp->out));
    NA2D_TRY(cudaMemcpyAsync((char *)dk + off, dk_ + off, n, cudaMemcpyDeviceToHost, hp->out));
    NA2D_TRY(cudaMemcpyAsync((char *)dv + off, dv_ + off, n, cudaMemcpyDeviceToHost, hp->out));
  }
  if (drpb) {
    sum_tables_kernel<<<(unsigned)((tbl + 255) / 256), 256, 0, hp->comp>>>(drpb_parts, nc, tstride, (int)tbl, drpb_);
    NA2D_TRY(cudaGetLastError());
    NA2D_TRY(cudaEventRecord(hp->drpb_ready, hp->comp));
    NA2D_TRY(cudaStreamWaitEvent(hp->out, hp->drpb_ready, 0));
    NA2D_TRY(cudaMemcpyAsync(drpb, drpb_, tb, cudaMemcpyDeviceToHost, hp->out));
  }
  NA2D_TRY(cudaEventRecord(hp->done, hp->out));
  NA2D_TRY(cudaStreamWaitEvent(st, hp->done, 0));
#undef NA2D_TRY
  return NA2D_OK;
}

int na2d_launch_count(const na2d_problem *p, int which) {
  Geo g;
  if (make_geo(p, &g) != NA2D_OK || (which != 0 && which != 1)) return -1;
  return use_tc(g, which) ? tc_launches(g, which) : simt_launches(g, which);
}

const char *na2d_kernel_family(const na2d_problem *p, int which) {
  Geo g;
  if (make_geo(p, &g) != NA2D_OK || (which != 0 && which != 1)) return nullptr;
  return use_tc(g, which) ? "tcgen05" : "simt";
}

}  // extern "C"
