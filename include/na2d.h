/*
 * na2d.h -- C ABI of libna2d: 2D Neighborhood Attention (NA2D) forward + backward on
 * NVIDIA B200 (sm_100a).
 *
 * The operation (Hassani et al., "Neighborhood Attention Transformer", arXiv 2204.07143;
 * PAPER.md line numbers cited as P:<n>):
 *
 *   Eq. 2:  NA(X_ij) = softmax( (Q_ij K_rho(ij)^T + B_ij) / scale ) V_rho(ij)
 *
 *   rho(i,j): the L x L window of key pixels
 *       rows [si, si+Lh) x cols [sj, sj+Lw), si = clamp(i - (L-1)/2, 0, H - L), Lh = L
 *       (if L >= H the window is the whole axis: si = 0, Lh = H), same for columns.
 *       Corner queries keep L^2 neighbours: the window shifts, it never shrinks (Fig. 7).
 *   B_ij: relative positional bias, one table per head of (2L-1) x (2L-1) fp32
 *       values, indexed by key minus query: B[h][p - i + L - 1][q - j + L - 1].
 *   scale: this ABI takes the MULTIPLIER (1/sqrt(d) for Eq. 1's sqrt(d_k)), and the
 *       bias is inside it:  s = scale * (q . k + B)   (reading R1).
 *   softmax over exactly the Lh*Lw window entries; LSE = max + log(sum exp(s - max)), natural
 *       log (reading R6).
 *   Backward (the analytic gradient of Eq. 2; the paper is silent, reading R5):
 *       D = dO.O, dP = dO.v, dS = P (dP - D), dQ = scale sum dS k, dK = scale sum dS q,
 *       dV = sum P dO, dB[cell] = scale sum dS over all (b, query, key) mapping to the cell.
 *
 * Tensor layouts (all C-contiguous, caller-owned DEVICE memory, base pointers 16-byte aligned):
 *   q, out, dout, dq : [batch][heads][height][width][dim]        element type = dtype
 *   k, v, dk, dv     : [batch][heads][kv_rows][width][dim]       element type = dtype
 *   lse              : [batch][heads][height][width]             fp32
 *   rpb, drpb        : [heads][2L-1][2L-1]                       fp32 (rpb == NULL: no bias,
 *                                                                  Table 7 variant P:352-353)
 * Row bands (multi-GPU row split): q/out/lse/dout/dq hold global rows
 *   [q_row0, q_row0 + height) of a map with map_height rows; k/v/dk/dv hold global rows
 *   [kv_row0, kv_row0 + kv_rows).  Geometry always uses global coordinates.  In the backward
 *   pass dk/dv/drpb receive the contributions of the held query rows only (the caller sums
 *   the partials of neighbouring bands).  Whole map: map_height = 0 (= height), q_row0 =
 *   kv_row0 = 0, kv_rows = 0 (= height).
 *
 * Streams and synchronisation: every call validates its arguments synchronously (on error
 * nothing is launched and no output is touched), then enqueues all work on `stream` (a
 * cudaStream_t, NULL = legacy default stream) and returns without synchronising.
 * Asynchronous device faults surface at the caller's next synchronisation.  A non-sticky CUDA
 * error left pending on the calling thread by an earlier, unrelated runtime call is cleared on
 * entry (NA2D_ERR_CUDA reports only errors of this call's own launches).  The library
 * allocates no device memory and keeps no per-call state; it is thread-safe.
 *
 * Precision: NA2D_BF16 = bf16 in/out, fp32 accumulation (tcgen05 tensor cores), fp32 LSE and
 * dRPB.  NA2D_F32 = fp32 in/out, fp32 SIMT FMA (no TF32), for 1e-4 relative parity.
 * NA2D_F16 = fp16 in/out (mixed-precision training I/O): the bf16 tensor-core kernels with fp16
 * MMA operands (P and dS rounded to fp16) for dim = 32, kernel_size 3/5/7; the SIMT and
 * paper-decomposition kernels (fp32 arithmetic, fp16 loads/stores) otherwise.
 */
#ifndef NA2D_H_
#define NA2D_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NA2D_VERSION 100 /* 1.0.0 */

typedef enum {
  NA2D_OK = 0,
  NA2D_ERR_NULL_POINTER = 1,  /* a required pointer is NULL */
  NA2D_ERR_KERNEL_SIZE = 2,   /* kernel_size even or < 3 ("odd number greater than 1") */
  NA2D_ERR_SHAPE = 3,         /* a dimension <= 0, overflow, or a band that misses needed rows */
  NA2D_ERR_DTYPE = 4,         /* dtype not an na2d_dtype */
  NA2D_ERR_UNSUPPORTED = 5,   /* valid but not implemented (dim > 128 or dim odd) */
  NA2D_ERR_ALIGNMENT = 6,     /* a tensor base pointer not 16-byte aligned */
  NA2D_ERR_WORKSPACE = 7,     /* workspace_bytes < na2d_backward_workspace_bytes() */
  NA2D_ERR_INVALID_ARG = 8,   /* scale not finite/positive; rpb/drpb NULL mismatch */
  NA2D_ERR_CUDA = 9           /* a CUDA runtime call or kernel launch failed */
} na2d_status;

typedef enum { NA2D_BF16 = 0, NA2D_F32 = 1, NA2D_F16 = 2 } na2d_dtype;

typedef struct {
  int32_t batch;        /* B */
  int32_t heads;        /* attention heads (independent instances) */
  int32_t height;       /* query rows held (= H for a whole map) */
  int32_t width;        /* W */
  int32_t dim;          /* per-head channels d (even, <= 128) */
  int32_t kernel_size;  /* L: odd, >= 3 */
  int32_t dtype;        /* na2d_dtype */
  float scale;          /* multiplier on (q.k + B); 1/sqrt(dim) reproduces Eq. 1's scaling */
  int32_t map_height;   /* global map rows; 0 => height */
  int32_t q_row0;       /* global row of the first held query row */
  int32_t kv_row0;      /* global row of the first held key/value row */
  int32_t kv_rows;      /* key/value rows held; 0 => height */
} na2d_problem;

/* Human-readable status text (static storage). */
const char *na2d_status_string(na2d_status s);

/* NA2D_VERSION of the loaded library. */
int na2d_version(void);

/* Forward pass, steps a1-a5 (geometry, RPB gather, QK^T + RPB, softmax, AV).
 * out: required.  lse: may be NULL (inference); it is a precondition of na2d_backward. */
na2d_status na2d_forward(const na2d_problem *p, const void *q, const void *k, const void *v,
                         const float *rpb, void *out, float *lse, void *stream);

/* Device workspace (bytes) na2d_backward needs for this problem: D (fp32 per query) plus the
 * tensor-core path's per-CTA dRPB partial tables, or the SIMT path's per-query window-slot dS
 * (B*heads*H*W*L*L fp32).  Both paths sum dRPB in a fixed order: drpb is bitwise reproducible for a
 * given problem and device. */
size_t na2d_backward_workspace_bytes(const na2d_problem *p);

/* Backward pass, steps a6-a10.  out and lse must be the na2d_forward results for the same
 * inputs.  dq, dk, dv are overwritten; drpb (NULL iff rpb is NULL) is overwritten with the
 * sum over the batch.  workspace: device memory of at least
 * na2d_backward_workspace_bytes(p) bytes, 16-byte aligned, not shared with a concurrent call. */
na2d_status na2d_backward(const na2d_problem *p, const void *q, const void *k, const void *v,
                          const float *rpb, const void *out, const float *lse, const void *dout,
                          void *dq, void *dk, void *dv, float *drpb, void *workspace,
                          size_t workspace_bytes, void *stream);

/* End-to-end step through HOST buffers: copies q,k,v,dout,rpb host->device, runs forward and
 * backward, copies out,lse,dq,dk,dv,drpb device->host.  The work is pipelined over up to 16 batch
 * chunks on three non-blocking streams owned by the library (created once per host thread and
 * device): chunk c+1's host->device copies and chunk c-1's device->host copies overlap chunk c's
 * kernels.  It starts after the work already enqueued on `stream`, and `stream` waits for its
 * completion, so callers synchronise on `stream` as before.  The host buffers (pinned memory
 * required for overlap) must stay valid until the stream is synchronised.
 * device_workspace: >= na2d_step_host_workspace_bytes(p) bytes of device memory.  Whole
 * maps only (no band fields). */
size_t na2d_step_host_workspace_bytes(const na2d_problem *p);
na2d_status na2d_step_host(const na2d_problem *p, const void *q, const void *k, const void *v,
                           const float *rpb, const void *dout, void *out, float *lse, void *dq,
                           void *dk, void *dv, float *drpb, void *device_workspace,
                           size_t workspace_bytes, void *stream);

/* The paper's own NA decomposition (App. A), kept as a
 * comparison path: a QK kernel that adds the RPB while writing the attention weights
 * [B][heads][rows][W][Lh*Lw] (fp32, Lh = min(L, height), Lw = min(L, width), window positions in
 * row-major order), a softmax kernel (in place; writes lse) and an AV kernel; the backward runs
 * the three kernels' gradients from the stored weights (dB by fp32 atomics, so its rounding order
 * is not fixed).  Same semantics as na2d_forward / na2d_backward (Eq. 2).
 * attn: device memory of na2d_paper_attn_bytes(p) bytes written by na2d_paper_forward and read by
 * na2d_paper_backward; dS: another buffer of the same size (backward scratch).  All pointers
 * 16-byte aligned device memory; lse required (it is written).  Errors as na2d_forward. */
size_t na2d_paper_attn_bytes(const na2d_problem *p);
na2d_status na2d_paper_forward(const na2d_problem *p, const void *q, const void *k, const void *v,
                               const float *rpb, void *out, float *lse, float *attn, void *stream);
na2d_status na2d_paper_backward(const na2d_problem *p, const void *q, const void *k, const void *v,
                                const void *dout, const float *attn, float *dS, void *dq, void *dk,
                                void *dv, float *drpb, void *stream);

/* Number of kernel launches na2d_forward (which = 0) or na2d_backward (which = 1) issues
 * for this problem, or -1 if the problem is invalid.  For launch accounting in benchmarks. */
int na2d_launch_count(const na2d_problem *p, int which);

/* Name of the kernel family the dispatcher selects for this problem/pass ("tcgen05" or
 * "simt"); NULL if the problem is invalid. */
const char *na2d_kernel_family(const na2d_problem *p, int which);

/* Text of the CUDA error behind the most recent NA2D_ERR_CUDA returned on this host thread
 * ("no error" if none).  Static/thread-local storage; valid until the next call. */
const char *na2d_last_cuda_error(void);

/* Per-kernel timing for benchmarks.  na2d_profile_enable(1) clears the record and makes every
 * subsequent launch bracket itself with CUDA events recorded on its own stream (the stream the
 * kernel is launched on); na2d_profile_enable(0) stops recording.  na2d_profile_read
 * synchronises the recorded events and writes up to max_entries aggregates: names (each
 * NUL-terminated, packed into names_out of name_cap bytes), total milliseconds and launch
 * counts per kernel name.  Returns the number of distinct kernel names, or -1 on error.
 * Not thread-safe with concurrent launches from other host threads. */
na2d_status na2d_profile_enable(int on);
int na2d_profile_read(char *names_out, size_t name_cap, float *total_ms, int *counts, int max_entries);

/* Development aid, effective only in builds with -DNA2D_TRACE: device buffer of >= 24000 int64
 * that the tensor-core kernels fill with clock64() timestamps of their pipeline events (first 32
 * tiles / chunks of CTAs 0-3: forward and B2 in slots [0, 4096), B1 in [4096, 8192)) and
 * %globaltimer wall-clock points (per-CTA spans from 16384, forward / B2 prologue and epilogue
 * points from 18000 / 19200; scripts/trace_balance.py, scripts/trace_fixed.py); NULL disables. */
na2d_status na2d_debug_set_trace(void *device_buffer);

#ifdef __cplusplus
}
#endif

#endif /* NA2D_H_ */
