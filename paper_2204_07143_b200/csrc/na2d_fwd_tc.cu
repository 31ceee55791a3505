// na2d_fwd_tc.cu -- NA2D forward on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Eq. 2 for bf16 Q/K/V, head dim 32, L in {3,5,7}.
//
// Tiling.  A CTA tile is 8 x 16 queries, split into two sub-tiles of 4 x 16 (rows 0-3, 4-7),
// each a tcgen05 M=64 MMA whose accumulator rows land in TMEM lanes 0-15 (sub-tile 0) or 16-31
// (sub-tile 1) of every 32-lane quarter.  All neighbourhoods rho of the tile
// lie in the halo rows [wstart(i0), +8+L-1) x cols [wstart(j0), +24) (global clamped
// coordinates, row pitch padded to 24), which TMA stages in shared memory (zero fill outside the
// tensor).  Sub-tile s only needs the 4+L-1 halo rows starting at rb_s = wstart(i0+4s) -
// wstart(i0), i.e. a contiguous, 512-byte aligned run of NSUB = (4+L-1)*24 keys:
//     S_s = Q_s K[rb_s..]^T   (M=64, N=NSUB, K=32)   tcgen05.mma SS -> TMEM [0, NSUB)
//     O_s = P_s V[rb_s..]     (M=64, N=32, K=NSUB)   tcgen05.mma TS (P from TMEM)
// Softmax.  TMEM lane quarter q holds the 4 x 4 query block at tile columns [4q, 4q+4) of both
// sub-tiles; the union of its windows is (4+L-1) rows x (4+L-1) columns of S (loaded as L+5
// even-aligned columns; the exponentials skip the two outside the union).  Per element pair, in
// packed fp32x2 arithmetic: x = s*scale*log2e + T[cell], T a shared-memory table of the head's
// relative positional bias B[h][p-i+L-1][q-j+L-1] pre-multiplied by scale*log2e, with
// -inf outside the query's own window (one table per column-clamp class, plus an all -inf row for
// rows outside the window; two copies shifted by one column so every lane reads 8-byte aligned
// pairs).  Exact two-pass softmax (the whole window sits in one tile): pass 1 computes x and the
// row max (FMNMX3) and stores x compacted to 12 columns per union row over consumed S columns;
// pass 2 writes P = exp2(x - max) as bf16 pairs in place, one union row pair at a time, each pair
// released at once to the PV MMAs (which accumulate O in the columns the compaction freed), so
// PV overlaps pass 2.
// Pipeline.  Persistent CTAs (one per SM), contiguous head-major tile ranges.  Warp 8: tile
// descriptions + TMA (3-stage ring); warp 9: MMA issue (QK of tile t, then PV of tile t-1 pair by
// pair); warps 0-3 and 4-7: two softmax + epilogue groups that ping-pong between two TMEM slots
// of 256 columns.
#include <math.h>

#include <mutex>

#include "na2d_internal.cuh"
#include "na2d_profile.cuh"
#include "na2d_sm100.cuh"
#include "na2d_tc.cuh"
#include "na2d_tc_common.cuh"
#include "na2d_tmap.cuh"


namespace na2d {
namespace {

using namespace sm100;
using namespace tc;

constexpr int kStagesQK = 3;      // Q + K halo ring (released when the QK MMAs complete)
constexpr int kStagesV = 3;       // V halo ring (released when the PV MMAs complete)
constexpr int kTInfo = 8;         // tile-description ring (>= 5: see the producer)
constexpr int kThreads = 640;     // 20 warps
// The SM sub-partition scheduler favours the highest warp id among eligible warps: the producer and
// MMA-issue warps take the two highest ids so the busy elementwise warps sharing their
// sub-partitions (warp % 4) never delay a TMA or MMA issue.
constexpr int kProducerWarp = 16, kMmaWarp = 17, kProducerVWarp = 18, kPvWarp = 19;
// O accumulators outside both S slots, shared by the two slots' tiles: the next QK of a slot waits
// only for that slot's PV MMAs (not for its epilogue), and PV of tile t waits for the epilogue
// of tile t - 1 (which precedes it by half a slot cycle)
#ifndef NA2D_FWD_SHARED_O
#define NA2D_FWD_SHARED_O 1
#endif

template <int L>
struct Cfg {
  static constexpr int HR = kTQH + L - 1;      // halo rows
  static constexpr int UR = 4 + L - 1;         // union rows per sub-tile
  static constexpr int PAIRS = UR / 2;         // union row pairs (3 PV K-steps each)
  static constexpr int NSUB = UR * kHCP;       // S columns per sub-tile (keys)
  static constexpr int P_COL = 0;              // P (bf16 pairs) aliased over consumed S
#if NA2D_FWD_SHARED_O
  static constexpr int SLOT = NSUB;            // TMEM columns per slot: S (then x / P)
  static constexpr int O_COL = 2 * NSUB;       // O partial accumulators (absolute column)
  static constexpr int OACC = (512 - O_COL) / kD < 3 ? (512 - O_COL) / kD : 3;  // independent PV chains
  static_assert(OACC >= 1, "TMEM budget");
#else
  static constexpr int SLOT = 256;
  static constexpr int O_COL = NSUB / 2;       // O partial accumulators past the compacted x / P (in the slot)
  static constexpr int OACC = 3;
  static_assert(O_COL + OACC * kD <= 256, "slot budget");
#endif
  static_assert(2 * kHCP == 3 * 16, "a union row pair is 3 PV K-steps");
  static constexpr int KV_ROWS = HR * kHCP;
  static constexpr int Q_BYTES = 128 * kRowBytes;
  static constexpr int KV_BYTES = KV_ROWS * kRowBytes;
  static constexpr int QK_BYTES = Q_BYTES + KV_BYTES;
  static_assert(QK_BYTES % 1024 == 0 && KV_BYTES % 1024 == 0, "stages must stay 1 KB aligned (swizzled TMA / UMMA)");
  static constexpr int V_OFF = kStagesQK * QK_BYTES;
  static constexpr int TT = 2 * L - 1;
  static constexpr int TROWS = TT + 1;                             // + all -inf row
  static constexpr int TBL_FLOATS = L * TROWS * kTblStride;        // one table copy
  static constexpr int TBL_OFF = V_OFF + kStagesV * KV_BYTES;      // 2 groups x 2 parity copies
  static constexpr int TI_OFF = TBL_OFF + 4 * TBL_FLOATS * 4;
  static constexpr int VI_OFF = TI_OFF + kTInfo * 64;                // V ring: halo row offsets
  static constexpr int BAR_OFF = VI_OFF + kStagesV * 16;
  static constexpr int SMEM = BAR_OFF + 320 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

struct FwdParams {
  int B, heads, H, W, q_rows, q_row0, kv_row0;
  int tiles_h, tiles_w, num_tiles;
  float scale_log2;  // scale * log2(e)
  const float *rpb;  // [heads][TT][TT] or null
  __nv_bfloat16 *out;
  float *lse;
  long long *trace;  // debug timeline (na2d_debug_set_trace, builds with -DNA2D_TRACE) or null
};

// Tile description (ring of kTInfo), written by the Q/K producer before it arms full_qk.
struct FTile {
  int bh, head, i0, j0, hr0, hc0;
  int rb[2];  // first halo row of sub-tile s (relative to hr0)
  int uc[4];  // union origin of lane quarter q: bit 0 = first needed column odd, rest = even column
};
static_assert(sizeof(FTile) <= 64, "FTile");

#ifdef NA2D_TRACE
// Debug timeline: trace[(cta * kTraceTiles + it) * kTraceEv + ev] = clock64() for CTAs < 4.
constexpr int kTraceTiles = 32, kTraceEv = 32;
__device__ __forceinline__ void trace_ev(const FwdParams &p, int it, int ev) {
  if (p.trace && blockIdx.x < 4 && it < kTraceTiles)
    p.trace[((size_t)blockIdx.x * kTraceTiles + it) * kTraceEv + ev] = clock64();
}
#else
__device__ __forceinline__ void trace_ev(const FwdParams &, int, int) {}
#endif

template <int L, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
  using C = Cfg<L>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float *tables = (float *)(smem + C::TBL_OFF);
  FTile *tinfo = (FTile *)(smem + C::TI_OFF);
  int *vinfo = (int *)(smem + C::VI_OFF);  // [V slot][2]: rb of the two sub-tiles
  uint64_t *bars = (uint64_t *)(smem + C::BAR_OFF);
  uint64_t *full = bars, *empty = bars + kStagesQK;                     // Q/K ring
  uint64_t *full_v = bars + 2 * kStagesQK, *empty_v = full_v + kStagesV;  // V ring
  uint64_t *s_full = full_v + 2 * kStagesV, *o_full = s_full + 2, *tmem_free = s_full + 4;
  uint64_t *p_pair = s_full + 6;  // [slot][pair]: union row pair of P written by the 4 warps
  // tile description it % kTInfo written (the elementwise warps must not wait on full[]: by the time
  // a slow group gets there, full[] may already have completed the next phase of its stage)
  uint64_t *ti_full = p_pair + 2 * C::PAIRS;
  uint64_t *o_free = ti_full + kTInfo;  // shared O read out by the epilogue of the previous tile
  uint32_t *tmem_slot = (uint32_t *)(o_free + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t_begin = (int)((long)p.num_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long)p.num_tiles * (blockIdx.x + 1) / gridDim.x);
  const int q_end = p.q_row0 + p.q_rows;

  if (warp == kProducerWarp && lane == 0) {
    for (int s = 0; s < kStagesQK; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kTInfo; ++s) mbar_init(&ti_full[s], 1);
    for (int s = 0; s < kStagesV; ++s) {
      mbar_init(&full_v[s], 1);
      mbar_init(&empty_v[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&o_full[s], 1);
      mbar_init(&tmem_free[s], NA2D_FWD_SHARED_O ? 1 : 8);  // PV commit / both lane-half groups' epilogue
      for (int k = 0; k < C::PAIRS; ++k) mbar_init(&p_pair[s * C::PAIRS + k], 8);
    }
    mbar_init(o_free, 8);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == kProducerWarp) tmem_alloc<512>(tmem_slot);
#ifdef NA2D_TRACE
  if (threadIdx.x == 0 && p.trace) {  // per-CTA wall-clock span (load balance)
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[16384 + 2 * blockIdx.x] = (long long)gt;
  }
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // the previous kernel on the stream is complete: global memory from here on

  if (warp == kProducerWarp) {
    // ================= producer (whole warp converged; one elected thread writes the tile
    // description and issues the TMA loads: Q 4x4 blocks, K / V halo).  Head-major tile order
    // (consecutive tiles share the head: bias table rebuilds are rare), stepped incrementally.
    const int per = p.tiles_h * p.tiles_w;
    const int u0 = t_begin / per, rem0 = t_begin - u0 * per;
    int h = u0 / p.B, b = u0 - h * p.B, tr = rem0 / p.tiles_w, tcol = rem0 - tr * p.tiles_w;
    for (int it = 0; it < t_end - t_begin; ++it) {
      const int s = it % kStagesQK;
      // full[s] re-arms once QK(it - 3) has completed; the description slot it % kTInfo was last read
      // (tile it - kTInfo) before that tile's epilogue, which precedes QK(it - kTInfo + 2) <= QK(it - 3)
      mbar_wait_sleep(&empty[s], ((it / kStagesQK) & 1) ^ 1, 1024);
      if (lane == 0) trace_ev(p, it, 0);
      const int bh = b * p.heads + h;
      const int i0 = p.q_row0 + tr * kTQH, j0 = tcol * kTQW;
      const int hr0 = wstart(i0, p.H, L), hc0 = wstart(j0, p.W, L);
      if (elect_one()) {
        FTile *ti = tinfo + it % kTInfo;
        ti->bh = bh;
        ti->head = h;
        ti->i0 = i0;
        ti->j0 = j0;
        ti->hr0 = hr0;
        ti->hc0 = hc0;
        ti->rb[0] = wstart(min(i0, q_end - 1), p.H, L) - hr0;
        ti->rb[1] = wstart(min(i0 + 4, q_end - 1), p.H, L) - hr0;
#pragma unroll
        for (int q = 0; q < 4; ++q) ti->uc[q] = wstart(min(j0 + 4 * q, p.W - 1), p.W, L) - hc0;
        mbar_arrive(&ti_full[it % kTInfo]);  // release: the description above is visible to its waiters
        uint8_t *st = smem + s * C::QK_BYTES;
        mbar_expect_tx(&full[s], C::QK_BYTES);
        // Q: sub-tile sb, quarter qb -> 16 rows = 4x4 block (rows i0+4sb.., cols j0+4qb..)
#pragma unroll
        for (int sb = 0; sb < 2; ++sb)
#pragma unroll
          for (int qb = 0; qb < 4; ++qb)
            tma_load_4d(st + (64 * sb + 16 * qb) * kRowBytes, &tm_q, &full[s], 0, j0 + 4 * qb, i0 - p.q_row0 + 4 * sb, bh);
        tma_load_4d(st + C::Q_BYTES, &tm_k, &full[s], 0, hc0, hr0 - p.kv_row0, bh);
      }
      __syncwarp();
      if (++tcol == p.tiles_w) {
        tcol = 0;
        if (++tr == p.tiles_h) {
          tr = 0;
          if (++b == p.B) {
            b = 0;
            ++h;
          }
        }
      }
    }
  } else if (warp == kProducerVWarp) {
    // ================= V producer: the V halo of tile it into ring slot it % kStagesV once PV of
    // tile it - kStagesV has completed (same head-major incremental tile walk as the Q/K producer)
    const int per = p.tiles_h * p.tiles_w;
    const int u0 = t_begin / per, rem0 = t_begin - u0 * per;
    int h = u0 / p.B, b = u0 - h * p.B, tr = rem0 / p.tiles_w, tcol = rem0 - tr * p.tiles_w;
    for (int it = 0; it < t_end - t_begin; ++it) {
      const int s = it % kStagesV;
      mbar_wait_sleep(&empty_v[s], ((it / kStagesV) & 1) ^ 1, 1024);
      const int bh = b * p.heads + h;
      const int i0 = p.q_row0 + tr * kTQH, j0 = tcol * kTQW;
      if (elect_one()) {
        const int hr0 = wstart(i0, p.H, L);
        vinfo[2 * s] = wstart(min(i0, q_end - 1), p.H, L) - hr0;
        vinfo[2 * s + 1] = wstart(min(i0 + 4, q_end - 1), p.H, L) - hr0;
        mbar_expect_tx(&full_v[s], C::KV_BYTES);
        tma_load_4d(smem + C::V_OFF + s * C::KV_BYTES, &tm_v, &full_v[s], 0, wstart(j0, p.W, L),
                    wstart(i0, p.H, L) - p.kv_row0, bh);
      }
      __syncwarp();
      if (++tcol == p.tiles_w) {
        tcol = 0;
        if (++tr == p.tiles_h) {
          tr = 0;
          if (++b == p.B) {
            b = 0;
            ++h;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ================= QK issuer (whole warp converged, one elected thread issues): S of tile it
    // into TMEM slot it & 1 once its Q / K have landed and the slot's previous epilogue has read O.
    // The PV MMAs have their own issuing warp, so neither stream waits behind the other's
    // dependencies.  Shared-memory descriptors are built once per stage and advanced by
    // (byte offset >> 4).
    constexpr uint32_t idesc_qk = idesc_el<F16>(64, C::NSUB, false);
    for (int it = 0; it < t_end - t_begin; ++it) {
      const int s = it % kStagesQK, slot = it & 1;
      mbar_wait(&full[s], (it / kStagesQK) & 1);
      const int rb0 = tinfo[it % kTInfo].rb[0], rb1 = tinfo[it % kTInfo].rb[1];
      if (lane == 0) trace_ev(p, it, 1);
      mbar_wait(&tmem_free[slot], ((it >> 1) & 1) ^ 1);
      if (lane == 0) trace_ev(p, it, 2);
      tc_fence_after();
      const uint64_t dq = sdesc_sw64(smem_u32(smem + s * C::QK_BYTES));
      const uint64_t dk = dq + (C::Q_BYTES >> 4);
      const uint64_t dk0 = dk + ((rb0 * kHCP * kRowBytes) >> 4), dk1 = dk + ((rb1 * kHCP * kRowBytes) >> 4);
      const uint32_t d0 = tmem + slot * C::SLOT, d1 = d0 + ((uint32_t)16 << 16);
      if (elect_one()) {  // two independent accumulation chains (sub-tiles) interleaved
        mma_ss(d0, dq, dk0, idesc_qk, 0);
        mma_ss(d1, dq + (4096 >> 4), dk1, idesc_qk, 0);
        mma_ss(d0, dq + (32 >> 4), dk0 + (32 >> 4), idesc_qk, 1);
        mma_ss(d1, dq + ((4096 + 32) >> 4), dk1 + (32 >> 4), idesc_qk, 1);
        mma_commit(&s_full[slot]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else if (warp == kPvWarp) {
    // ================= PV issuer: O of tile it (slot it & 1) one union row pair at a time as the
    // elementwise warps release it (the PV overlaps pass 2)
    constexpr uint32_t idesc_pv = idesc_el<F16>(64, kD, true);
    for (int it = 0; it < t_end - t_begin; ++it) {
      const int s = it % kStagesV, slot = it & 1;
      mbar_wait(&full_v[s], (it / kStagesV) & 1);
      const int rb0 = vinfo[2 * s], rb1 = vinfo[2 * s + 1];
      const uint64_t dv = sdesc_sw64(smem_u32(smem + C::V_OFF + s * C::KV_BYTES));
      const uint64_t dv0 = dv + ((rb0 * kHCP * kRowBytes) >> 4), dv1 = dv + ((rb1 * kHCP * kRowBytes) >> 4);
      const uint32_t b0 = tmem + slot * C::SLOT, b1 = b0 + ((uint32_t)16 << 16);
#if NA2D_FWD_SHARED_O
      const uint32_t o0 = tmem + C::O_COL, o1 = o0 + ((uint32_t)16 << 16);
#else
      const uint32_t o0 = b0 + C::O_COL, o1 = b1 + C::O_COL;
#endif
      // fully unrolled: every descriptor / TMEM address below is the tile's base + an immediate, so
      // each pair's issue is a short independent burst (no dependent address chain per pair)
#pragma unroll
      for (int k = 0; k < C::PAIRS; ++k) {
#if NA2D_FWD_SHARED_O
        if (k == 0 && it > 0) mbar_wait(o_free, (it - 1) & 1);  // epilogue of tile it - 1 read O
#endif
        mbar_wait(&p_pair[slot * C::PAIRS + k], (it >> 1) & 1);
        if (lane == 0) trace_ev(p, it, 19 + k);
        tc_fence_after();
        // 2 sub-tiles x kOAcc partial accumulators = independent MMA chains, interleaved
        constexpr uint32_t acc = 1;
        if (elect_one()) {
#pragma unroll
          for (int k3 = 0; k3 < 3; ++k3) {
            const int ks = 3 * k + k3;
            const uint32_t voff = (ks * 16 * kRowBytes) >> 4, oc = (ks % C::OACC) * kD;
            const uint32_t a = ks >= C::OACC ? acc : 0u;
            mma_ts(o0 + oc, b0 + C::P_COL + ks * 8, dv0 + voff, idesc_pv, a);
            mma_ts(o1 + oc, b1 + C::P_COL + ks * 8, dv1 + voff, idesc_pv, a);
          }
          if (k == C::PAIRS - 1) {
            mma_commit(&o_full[slot]);
            mma_commit(&empty_v[s]);
#if NA2D_FWD_SHARED_O
            mma_commit(&tmem_free[slot]);  // P read: the slot may take the next QK
#endif
          }
        }
        __syncwarp();
      }
      if (lane == 0) trace_ev(p, it, 3);
    }
  } else {
    // ================= softmax + epilogue: 4 groups of 4 warps.  Group g works on TMEM slot g >> 1
    // (tiles it with it & 1 == slot) and on sub-tile / TMEM lane half h = g & 1 of those tiles; its
    // warp of lane quarter q reads the 16 lanes [32q + 16h, +16) with the .16x32bx2 shapes, so two
    // threads share a query: thread t handles query (t & 15) and union columns [6 (t >> 4), +6).
    const int grp = warp >> 2, slot = grp >> 1, hh = grp & 1;
    const int quarter = warp & 3;
    const int hf = lane >> 4, ql = lane & 15, r = ql >> 2, c = ql & 3;
    float *tbl = tables + slot * 2 * C::TBL_FLOATS;  // the slot's two parity copies (both halves share)
    const int stid = threadIdx.x - slot * 256;       // 0..255 within the slot's two groups
    const int Lh = wlen(p.H, L), Lw = wlen(p.W, L);
    const float2 sl2x2 = make_float2(p.scale_log2, p.scale_log2);
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32 + 16 * hh) << 16) + slot * C::SLOT;
#if NA2D_FWD_SHARED_O
    const uint32_t o_addr = tmem + ((uint32_t)(quarter * 32 + 16 * hh) << 16) + C::O_COL;
#else
    const uint32_t o_addr = lane_addr + C::O_COL;
#endif
    int cur_head = -1;
    for (int it = slot; it < t_end - t_begin; it += 2) {
      const uint32_t ph = (it >> 1) & 1;
      // tile description of tile it: its ring slot is rewritten (tile it + 8) only after QK(it + 5),
      // which needs the epilogue of tile it + 3, whose PV is issued after PV(it + 2), i.e. after this
      // group has read the description of tile it (and processed tile it + 2)
      mbar_wait(&ti_full[it % kTInfo], (it / kTInfo) & 1);
      const FTile &ti = tinfo[it % kTInfo];
      const int bh = ti.bh, h = ti.head, i0 = ti.i0, j0 = ti.j0, hr0 = ti.hr0, hc0 = ti.hc0;
      const int rb = ti.rb[hh], ucr = ti.uc[quarter];
      if (h != cur_head) {  // (re)build the slot's masked, pre-scaled bias tables (two parity copies:
        // copy x holds column b at kTblOff + x + b, so every thread's row start is 8-byte aligned)
        named_bar_sync(1 + slot, 256);
        for (int e = stid; e < 2 * C::TBL_FLOATS; e += 256) {
          const int x = e >= C::TBL_FLOATS, e2 = e - x * C::TBL_FLOATS;
          const int dc = e2 / (C::TROWS * kTblStride);
          const int rr = (e2 / kTblStride) % C::TROWS;
          const int cb = e2 % kTblStride - kTblOff - x;
          float v = -INFINITY;
          if (rr < C::TT && cb >= dc && cb < dc + Lw) v = p.rpb ? __ldg(&p.rpb[(h * C::TT + rr) * C::TT + cb]) * p.scale_log2 : 0.f;
          tbl[e] = v;
        }
        named_bar_sync(1 + slot, 256);
        cur_head = h;
      }
      // this thread's query and window geometry
      const int i = i0 + 4 * hh + r, j = j0 + 4 * quarter + c;
      const int ic = min(i, q_end - 1), jc = min(j, p.W - 1);
      const int si = wstart(ic, p.H, L), sj = wstart(jc, p.W, L);
      const int uc = ucr & ~1;                                       // even union origin (warp-uniform)
      const int dc = sj - jc + L - 1;                                // column-clamp class
      const int bcol0 = hc0 + uc - jc + L - 1;                       // bias column of union col 0
      const int cp = bcol0 & 1;                                      // parity copy: aligned row start
      const float *tcls = tbl + cp * C::TBL_FLOATS + dc * C::TROWS * kTblStride + kTblOff + cp + bcol0 + 6 * hf;

      const bool tr = grp == 0 && quarter == 2 && lane == 0;
      if (tr) trace_ev(p, it, 4);
      mbar_wait(&s_full[slot], ph);
      if (tr) trace_ev(p, it, 5);
      tc_fence_after();
      // ---- pass 1 (union row pair k per step, software-pipelined): x = s*scale*log2e + T in packed
      // fp32x2 over this thread's 6 columns; row max (FMNMX3); x stored compacted: union row u at
      // columns [12u, 12u+12) over consumed S columns, freeing [NSUB/2, 256) for O during pass 2
      float mx = -INFINITY;
      {
        uint32_t S[2][16];  // [buffer][row a: 0-7 | row b: 8-15] (columns 6, 7 of each row unused)
        float2 T[2][6];     // bias pairs: row a 0-2, row b 3-5
        auto load_tbl = [&](int u, float2(&t)[6]) {
          const int pr = hr0 + rb + u;  // key row of union row u
          const bool rva = (unsigned)(pr - si) < (unsigned)Lh, rvb = (unsigned)(pr + 1 - si) < (unsigned)Lh;
          const float2 *ta = (const float2 *)(tcls + (rva ? pr - ic + L - 1 : C::TT) * kTblStride);
          const float2 *tb = (const float2 *)(tcls + (rvb ? pr + 1 - ic + L - 1 : C::TT) * kTblStride);
#pragma unroll
          for (int z = 0; z < 3; ++z) {
            t[z] = ta[z];
            t[3 + z] = tb[z];
          }
        };
        auto load_s = [&](int u, uint32_t(&d)[16]) {
          tmem_ld_h8<6>(lane_addr + u * kHCP + uc, *reinterpret_cast<uint32_t(*)[8]>(&d[0]));
          tmem_ld_h8<6>(lane_addr + (u + 1) * kHCP + uc, *reinterpret_cast<uint32_t(*)[8]>(&d[8]));
        };
        load_s(0, S[0]);
        load_tbl(0, T[0]);
#pragma unroll
        for (int k = 0; k < C::PAIRS; ++k) {
          const int u = 2 * k;
          uint32_t(&cur)[16] = S[k & 1];
          const float2(&tc)[6] = T[k & 1];
          tc_wait_ld();
          if (k + 1 < C::PAIRS) {
            load_s(u + 2, S[(k + 1) & 1]);
            load_tbl(u + 2, T[(k + 1) & 1]);
          }
          float2 x[6];
#pragma unroll
          for (int z = 0; z < 3; ++z) {
            x[z] = __ffma2_rn(make_float2(__uint_as_float(cur[2 * z]), __uint_as_float(cur[2 * z + 1])), sl2x2, tc[z]);
            x[3 + z] = __ffma2_rn(make_float2(__uint_as_float(cur[8 + 2 * z]), __uint_as_float(cur[9 + 2 * z])), sl2x2,
                                  tc[3 + z]);
          }
          mx = fmax3(mx, fmax3(fmax3(x[0].x, x[0].y, x[1].x), fmax3(x[1].y, x[2].x, x[2].y),
                               fmax3(x[3].x, x[3].y, x[4].x)),
                     fmax3(x[4].y, x[5].x, x[5].y));
          const uint32_t xa4[4] = {__float_as_uint(x[0].x), __float_as_uint(x[0].y), __float_as_uint(x[1].x),
                                   __float_as_uint(x[1].y)};
          const uint32_t xa2[2] = {__float_as_uint(x[2].x), __float_as_uint(x[2].y)};
          const uint32_t xb4[4] = {__float_as_uint(x[3].x), __float_as_uint(x[3].y), __float_as_uint(x[4].x),
                                   __float_as_uint(x[4].y)};
          const uint32_t xb2[2] = {__float_as_uint(x[5].x), __float_as_uint(x[5].y)};
          tmem_st_h4<6>(lane_addr + u * 12, xa4);
          tmem_st_h2<6>(lane_addr + u * 12 + 4, xa2);
          tmem_st_h4<6>(lane_addr + u * 12 + 12, xb4);
          tmem_st_h2<6>(lane_addr + u * 12 + 16, xb2);
        }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));  // the query's other 6 columns
      tc_wait_st();
      if (tr) trace_ev(p, it, 6);
      // ---- pass 2 (row pair k per step, pipelined): P = exp2(x - max) -> bf16 pairs in place (each
      // halo row of P zeroed, then the union span written); pair k-1 is released to the PV MMAs once
      // pair k is computed (its stores have drained by then)
      float2 sum2 = make_float2(0.f, 0.f);
      const int zb = uc >> 1;  // packed column where the union span starts (warp-uniform)
      {
        uint32_t X[2][12];  // [buffer][row a: 0-5 | row b: 6-11]
        auto load_x = [&](int u, uint32_t(&d)[12]) {
          tmem_ld_h4<6>(lane_addr + u * 12, *reinterpret_cast<uint32_t(*)[4]>(&d[0]));
          tmem_ld_h2<6>(lane_addr + u * 12 + 4, *reinterpret_cast<uint32_t(*)[2]>(&d[4]));
          tmem_ld_h4<6>(lane_addr + u * 12 + 12, *reinterpret_cast<uint32_t(*)[4]>(&d[6]));
          tmem_ld_h2<6>(lane_addr + u * 12 + 16, *reinterpret_cast<uint32_t(*)[2]>(&d[10]));
        };
        load_x(0, X[0]);
        const float2 nm = make_float2(-mx, -mx);
        const uint32_t z4[4] = {0u, 0u, 0u, 0u}, z2[2] = {0u, 0u};
#pragma unroll
        for (int k = 0; k < C::PAIRS; ++k) {
          const int u = 2 * k;
          uint32_t(&cur)[12] = X[k & 1];
          tc_wait_ld();
          if (k + 1 < C::PAIRS) load_x(u + 2, X[(k + 1) & 1]);
          uint32_t pk[6];
#pragma unroll
          for (int z = 0; z < 6; ++z) {
            const float2 a = __fadd2_rn(make_float2(__uint_as_float(cur[2 * z]), __uint_as_float(cur[2 * z + 1])), nm);
            const float2 e = make_float2(ex2(a.x), ex2(a.y));
            sum2 = __fadd2_rn(sum2, e);
            pk[z] = pack_el<F16>(e.x, e.y);
          }
          if (k > 0) {
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_pair[slot * C::PAIRS + k - 1]);
          }
          // P row u: 12 packed columns at [12u, 12u+12) -- each half zeroes its 6, then the union span
          // (6 packed columns from zb; this thread's 3 at zb + 3 hf)
          const uint32_t prow = lane_addr + C::P_COL + u * (kHCP / 2);
          tmem_st_h4<6>(prow, z4);
          tmem_st_h2<6>(prow + 4, z2);
          tmem_st_h4<6>(prow + 12, z4);
          tmem_st_h2<6>(prow + 16, z2);
          const uint32_t pa2[2] = {pk[0], pk[1]}, pb2[2] = {pk[3], pk[4]};
          tmem_st_h2<3>(prow + zb, pa2);
          tmem_st_h1<3>(prow + zb + 2, pk[2]);
          tmem_st_h2<3>(prow + 12 + zb, pb2);
          tmem_st_h1<3>(prow + 12 + zb + 2, pk[5]);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_pair[slot * C::PAIRS + C::PAIRS - 1]);
      }
      float sum = sum2.x + sum2.y;
      sum += __shfl_xor_sync(0xffffffffu, sum, 16);
      if (tr) trace_ev(p, it, 7);
      // ---- epilogue: O / sum -> bf16 (this thread: head dims [16 hf, 16 hf + 16)), LSE
      mbar_wait(&o_full[slot], ph);
      if (tr) trace_ev(p, it, 8);
      tc_fence_after();
      float o[16];
      {
        uint32_t oa[C::OACC][16];
#pragma unroll
        for (int a = 0; a < C::OACC; ++a) tmem_ld_h16<16>(o_addr + a * kD, oa[a]);
        tc_wait_ld();
#pragma unroll
        for (int z = 0; z < 16; ++z) {
          float acc = __uint_as_float(oa[0][z]);
#pragma unroll
          for (int a = 1; a < C::OACC; ++a) acc += __uint_as_float(oa[a][z]);
          o[z] = acc;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(NA2D_FWD_SHARED_O ? o_free : &tmem_free[slot]);
      if (i < q_end && j < p.W) {
        const float inv = 1.f / sum;
        const size_t qi = ((size_t)bh * p.q_rows + (i - p.q_row0)) * p.W + j;
        uint4 *dst = (uint4 *)(p.out + qi * kD + 16 * hf);
#pragma unroll
        for (int z = 0; z < 16; z += 8)
          dst[z / 8] = make_uint4(pack_el<F16>(o[z] * inv, o[z + 1] * inv), pack_el<F16>(o[z + 2] * inv, o[z + 3] * inv),
                                  pack_el<F16>(o[z + 4] * inv, o[z + 5] * inv), pack_el<F16>(o[z + 6] * inv, o[z + 7] * inv));
        if (p.lse && hf == 0) p.lse[qi] = (mx + __log2f(sum)) * 0.69314718055994531f;
      }
      if (tr) trace_ev(p, it, 9);
    }
  }
  __syncthreads();
  if (warp == kProducerWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
#ifdef NA2D_TRACE
    if (lane == 0 && p.trace) {
      uint64_t gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.trace[16384 + 2 * blockIdx.x + 1] = (long long)gt;
    }
#endif
  }
}

template <int L, bool F16>
cudaError_t launch_fwd(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  using C = Cfg<L>;
  const cudaError_t attr_err = tc::ensure_smem_attr((const void *)na2d_fwd_tc_kernel<L, F16>, C::SMEM);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tk, tv;
  const int BH = g.B * g.heads;
  if (!make_tmap_e16_4d(F16, &tq, q, kD, g.W, g.q_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tk, k, kD, g.W, g.kv_rows, BH, kHCP, C::HR) ||
      !make_tmap_e16_4d(F16, &tv, v, kD, g.W, g.kv_rows, BH, kHCP, C::HR))
    return cudaErrorInvalidValue;
  FwdParams p;
  p.B = g.B;
  p.heads = g.heads;
  p.H = g.H;
  p.W = g.W;
  p.q_rows = g.q_rows;
  p.q_row0 = g.q_row0;
  p.kv_row0 = g.kv_row0;
  p.tiles_h = (g.q_rows + kTQH - 1) / kTQH;
  p.tiles_w = (g.W + kTQW - 1) / kTQW;
  p.num_tiles = BH * p.tiles_h * p.tiles_w;
  p.scale_log2 = g.scale * 1.4426950408889634f;
  p.rpb = rpb;
  p.out = (__nv_bfloat16 *)out;
  p.lse = lse;
  p.trace = (long long *)debug_trace_buffer();
  const int grid = p.num_tiles < num_sms() ? p.num_tiles : num_sms();
  ProfScope ps("na2d_fwd_tc", st);
  const cudaError_t e = launch_pdl(na2d_fwd_tc_kernel<L, F16>, grid, kThreads, C::SMEM, st, tq, tk, tv, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

bool tc_forward_supported(const Geo &g) {
  return (g.dtype == NA2D_BF16 || g.dtype == NA2D_F16) && g.d == kD && (g.L == 3 || g.L == 5 || g.L == 7) && tmap_available();
}

cudaError_t tc_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  const bool f16 = g.dtype == NA2D_F16;
  switch (g.L) {
    case 3: return f16 ? launch_fwd<3, true>(g, q, k, v, rpb, out, lse, st)
                 : launch_fwd<3, false>(g, q, k, v, rpb, out, lse, st);
    case 5: return f16 ? launch_fwd<5, true>(g, q, k, v, rpb, out, lse, st)
                 : launch_fwd<5, false>(g, q, k, v, rpb, out, lse, st);
    case 7: return f16 ? launch_fwd<7, true>(g, q, k, v, rpb, out, lse, st)
                 : launch_fwd<7, false>(g, q, k, v, rpb, out, lse, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace na2d
