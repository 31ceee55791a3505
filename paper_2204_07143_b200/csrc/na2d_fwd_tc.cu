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
// sub-tiles (lanes 0-15: sub-tile 0, lanes 16-31: sub-tile 1); relative to each sub-tile's own halo
// base the union of the block's windows is the same (4+L-1) x (4+L-1) keys, so one warp serves
// both lane halves with the plain 32x32b TMEM shapes, one thread per query.  The union rows are
// split between two warps per quarter; each thread loads its rows' S (L+5 even-aligned columns,
// one wait), keeps x = s*scale*log2e + T in registers (packed fp32x2 FFMA2), T a shared-memory
// table of the head's relative positional bias B[h][p-i+L-1][q-j+L-1] pre-multiplied by
// scale*log2e, with -inf outside the query's own window (one table per column-clamp class, an
// all -inf row, two copies shifted by one column so every row read is 8-byte aligned).  Exact
// softmax (the whole window is in one tile): row max and sum are combined across the two warps
// through shared memory; P = exp2(x - max) goes to TMEM as bf16 pairs over consumed S columns
// (each P row zeroed, then its union span written), and the PV MMAs accumulate O.
// Pipeline.  Persistent CTAs (one per SM), contiguous head-major tile ranges.  Warp 16: tile
// descriptions + Q/K TMA (3-stage ring); warp 18: V TMA (3-stage ring); warp 17: QK issue;
// warp 19: PV issue; warps 0-7 and 8-15: softmax + epilogue of the two TMEM slots (alternating
// tiles).  Waits use mbarrier try_wait with a suspend-time hint (no spin loops).
#include <math.h>

#include <mutex>
#include <type_traits>

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

// waits of the issuing and elementwise warps (NA2D_FWD_WAIT=2: try_wait with a suspend-time hint)
#if defined(NA2D_FWD_WAIT) && NA2D_FWD_WAIT == 2
__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t parity) { mbar_wait_hint(bar, parity); }
#else
__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }
#endif

constexpr int kTInfo = 8;         // tile-description ring (>= 5: see the producer)
constexpr int kThreads = 640;     // 20 warps: 16 elementwise (two groups of 8), 4 producer / MMA-issue
// The SM sub-partition scheduler favours the highest warp id among eligible warps: the producer and
// MMA-issue warps take the highest ids so the busy elementwise warps sharing their sub-partitions
// (warp % 4) never delay a TMA or MMA issue.
constexpr int kProducerWarp = 16, kMmaWarp = 17, kProducerVWarp = 18, kPvWarp = 19;

template <int L, int D>
struct Cfg {
  static_assert(D == 16 || D == 32 || D == 64, "head dim");
  static constexpr int ROWB = 2 * D;            // bytes per 16-bit row: one swizzle atom (32 / 64 / 128 B)
  // Q + K halo ring (released when the QK MMAs complete), V halo ring (released when PV completes);
  // single-stage at D = 64 (shared memory)
  static constexpr int SQK = D <= 32 ? 2 : 1, SV = D <= 32 ? 2 : 1;
  static constexpr int HP = kTQW + L - 1;       // halo width = row pitch of the K / V sub-tile buffers
  static constexpr int PW = HP / 2;             // pair mode: key columns of member m start at m * PW
  static constexpr int UR = 4 + L - 1;          // halo rows of a sub-tile (4 query rows)
  static constexpr int UH = UR / 2;             // union rows per elementwise warp (two warps per lane quarter)
  static_assert(UR % 2 == 0, "union rows split evenly between the two warps of a quarter");
  static constexpr int UW = L + 3;              // union width (keys) of a lane quarter's 4 x 4 query block
  static constexpr int PROW = HP / 2;           // packed P columns per halo row
  // keys per sub-tile: UR x HP halo keys (+2: an odd union origin loads one column past the union),
  // padded to whole PV K-steps of 16 keys; the tail keys are zero rows of K / V
  static constexpr int NSUB = (UR * HP + 2 + 15) / 16 * 16;
  static constexpr int KSTEPS = NSUB / 16;
  static constexpr int BOX_BYTES = UR * HP * ROWB;       // one sub-tile's TMA box
  static constexpr int SUB_BYTES = (NSUB * ROWB + 1023) / 1024 * 1024;  // one sub-tile's K or V buffer
  static_assert(SUB_BYTES % 1024 == 0, "sub-tile buffers stay 1 KB aligned (swizzled TMA / UMMA)");
  // TMEM: two slots (one per elementwise group) of NSUB columns: S, then P (NSUB/2 packed columns)
  // over the consumed S; O accumulators past both, shared by the groups' alternating tiles
  static constexpr int O_COL = 2 * NSUB;
  static constexpr int OACC = (512 - O_COL) / D < 4 ? (512 - O_COL) / D : 4;  // PV chains per sub-tile
  static_assert(OACC >= 1, "TMEM budget");
  static constexpr int Q_BYTES = 128 * ROWB;
  static constexpr int QK_BYTES = Q_BYTES + 2 * SUB_BYTES;
  static constexpr int V_BYTES = 2 * SUB_BYTES;
  static constexpr int V_OFF = SQK * QK_BYTES;
  static constexpr int TT = 2 * L - 1;
  static constexpr int TROWS = TT + 1;                             // + all -inf row
  static constexpr int TBL_FLOATS = L * TROWS * kTblStride;        // one table copy
  static constexpr int TBL_OFF = V_OFF + SV * V_BYTES;             // 2 groups x 2 parity copies
  static constexpr int EX_OFF = TBL_OFF + 4 * TBL_FLOATS * 4;      // row max / sum exchange [2][2][4][2][32]
  static constexpr int RB_OFF = EX_OFF + 2 * 2 * 4 * 2 * 32 * 4;   // per group: scaled RPB + window max
  static constexpr int RB_FLOATS = 320;  // scaled RPB, window maxima, row-wise sliding maxima
  static_assert(TT * TT + L * L + TT * L <= RB_FLOATS, "RPB staging");
  static constexpr int TI_OFF = RB_OFF + 2 * RB_FLOATS * 4;
  static constexpr int BAR_OFF = TI_OFF + kTInfo * 64;
  static constexpr int SMEM = BAR_OFF + 320 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

struct FwdParams {
  int B, heads, H, W, q_rows, q_row0, kv_row0;
  int pair;          // small-map pair mode (tc::pair_mode): B counts map pairs, K / V maps are pair views
  int tiles_h, tiles_w, num_tiles;
  float scale_log2;  // scale * log2(e)
  const float *rpb;  // [heads][TT][TT] or null
  __nv_bfloat16 *out;
  float *lse;
  long long *trace;  // debug timeline (na2d_debug_set_trace, builds with -DNA2D_TRACE) or null
};

#ifdef NA2D_TRACE
// Debug timeline: trace[(cta * kTraceTiles + it) * kTraceEv + ev] = clock64() for CTAs < 4.
constexpr int kTraceTiles = 32, kTraceEv = 32;
__device__ __forceinline__ void trace_ev(const FwdParams &p, int it, int ev) {
  if (p.trace && blockIdx.x < 4 && it < kTraceTiles)
    p.trace[((size_t)blockIdx.x * kTraceTiles + it) * kTraceEv + ev] = clock64();
}
// wall clock of prologue / epilogue points: trace[18000 + 8 * cta + k] (scripts/trace_fixed.py)
__device__ __forceinline__ void trace_gt(const FwdParams &p, int k) {
  if (p.trace) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[18000 + 8 * blockIdx.x + k] = (long long)gt;
  }
}
#else
__device__ __forceinline__ void trace_ev(const FwdParams &, int, int) {}
__device__ __forceinline__ void trace_gt(const FwdParams &, int) {}
#endif

// Tile description (ring of kTInfo), written by the Q/K producer before it arms full_qk.
struct FTile {
  int bh, head, i0, j0, hr0, hc0;
  int rb[2];  // first halo row of sub-tile s (relative to hr0)
  int uc[4];  // union origin (first needed halo column) of lane quarter q
};
static_assert(sizeof(FTile) <= 64, "FTile");

template <int L, int D, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
  using C = Cfg<L, D>;
  constexpr int kStagesQK = C::SQK, kStagesV = C::SV, kRB = C::ROWB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  FTile *tinfo = (FTile *)(smem + C::TI_OFF);
  uint64_t *bars = (uint64_t *)(smem + C::BAR_OFF);
  uint64_t *full = bars, *empty = bars + kStagesQK;                     // Q/K ring
  uint64_t *full_v = bars + 2 * kStagesQK, *empty_v = full_v + kStagesV;  // V ring
  uint64_t *s_full = full_v + 2 * kStagesV;  // [group]: S of the group's tile in its slot
  uint64_t *slot_free = s_full + 2;          // [group]: PV of the slot's tile complete (P read)
  uint64_t *p_ready = s_full + 4;            // [group]: P written by the group's 8 warps
  uint64_t *o_full = s_full + 6;             // [group]: PV of the group's tile complete
  uint64_t *o_free = s_full + 8;             // shared O read out by the epilogue of the previous tile
  // tile description it % kTInfo written (the elementwise warps must not wait on full[]: by the time
  // a slow group gets there, full[] may already have completed the next phase of its stage)
  uint64_t *ti_full = s_full + 9;
  uint32_t *tmem_slot = (uint32_t *)(ti_full + kTInfo);

  // broadcast from lane 0 so the compiler treats the warp index (and the TMEM addresses
  // derived from it) as warp-uniform: they stay in uniform registers, no R2UR per tcgen05.ld
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int t_begin = (int)((long)p.num_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long)p.num_tiles * (blockIdx.x + 1) / gridDim.x);
  const int ntile = t_end - t_begin;
  const int q_end = p.q_row0 + p.q_rows;
  if (threadIdx.x == 0) trace_gt(p, 0);

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
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&slot_free[g], 1);
      mbar_init(&p_ready[g], 8);
      mbar_init(&o_full[g], 1);
    }
    mbar_init(o_free, 8);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == kProducerWarp) tmem_alloc<512>(tmem_slot);
  // the K / V sub-tile buffer rows past the TMA box (keys [UR*HP, NSUB)) are read by the MMAs but
  // never loaded: zero them once (S / O stay finite there; P is zero for those keys)
  for (int e = threadIdx.x; e < (kStagesQK + kStagesV) * 2 * (C::SUB_BYTES - C::BOX_BYTES) / 16; e += kThreads) {
    constexpr int per = (C::SUB_BYTES - C::BOX_BYTES) / 16;
    const int buf = e / per, o = e % per;
    uint8_t *base = buf < 2 * kStagesQK ? smem + (buf >> 1) * C::QK_BYTES + C::Q_BYTES + (buf & 1) * C::SUB_BYTES
                                        : smem + C::V_OFF + (buf - 2 * kStagesQK) * C::SUB_BYTES;
    *(uint4 *)(base + C::BOX_BYTES + o * 16) = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // the previous kernel on the stream is complete: global memory from here on
  if (threadIdx.x == 0) trace_gt(p, 1);
#ifdef NA2D_TRACE
  if (threadIdx.x == 0 && p.trace) {  // per-CTA wall-clock span (load balance, scripts/trace_balance.py)
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[16384 + 2 * blockIdx.x] = (long long)gt;
  }
#endif

  if (warp == kProducerWarp) {
    // ================= producer (whole warp converged; one elected thread writes the tile
    // description and issues the TMA loads: Q 4x4 blocks, the K halo rows of each sub-tile).
    // Head-major tile order (consecutive tiles share the head: bias table rebuilds are rare).
    const int per = p.tiles_h * p.tiles_w;
    const int u0 = t_begin / per, rem0 = t_begin - u0 * per;
    int h = u0 / p.B, b = u0 - h * p.B, tr = rem0 / p.tiles_w, tcol = rem0 - tr * p.tiles_w;
    for (int it = 0; it < ntile; ++it) {
      const int s = it % kStagesQK;
      // full[s] re-arms once QK(it - kStagesQK) has completed; the description slot it % kTInfo was
      // last read (tile it - kTInfo) before that tile's S was loaded, long before
      mbar_wait_producer(&empty[s], ((it / kStagesQK) & 1) ^ 1);
      if (lane == 0) trace_ev(p, it, 0);
      const int bh = p.pair ? 2 * b * p.heads + h : b * p.heads + h;  // (pair: member 0)
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
        for (int q = 0; q < 4; ++q)
          ti->uc[q] = p.pair ? (q >> 1) * C::PW + wstart(min(4 * (q & 1), p.W - 1), p.W, L)
                             : wstart(min(j0 + 4 * q, p.W - 1), p.W, L) - hc0;
        mbar_arrive(&ti_full[it % kTInfo]);  // release: the description above is visible to its waiters
        uint8_t *st = smem + s * C::QK_BYTES;
        mbar_expect_tx(&full[s], C::Q_BYTES + 2 * C::BOX_BYTES);
        // Q: sub-tile sb, quarter qb -> 16 rows = 4x4 block (rows i0+4sb.., cols j0+4qb..)
#pragma unroll
        for (int sb = 0; sb < 2; ++sb)
#pragma unroll
          for (int qb = 0; qb < 4; ++qb)
            tma_load_4d(st + (64 * sb + 16 * qb) * kRB, &tm_q, &full[s], 0, p.pair ? 4 * (qb & 1) : j0 + 4 * qb,
                        i0 - p.q_row0 + 4 * sb, p.pair ? bh + (qb >> 1) * p.heads : bh);
#pragma unroll
        for (int sb = 0; sb < 2; ++sb) {
          if (p.pair)  // both members' halo rows side by side: row pitch 2 * PW = HP
            tma_load_5d(st + C::Q_BYTES + sb * C::SUB_BYTES, &tm_k, &full[s], 0, 0, 0, hr0 + ti->rb[sb] - p.kv_row0, bh);
          else
            tma_load_4d(st + C::Q_BYTES + sb * C::SUB_BYTES, &tm_k, &full[s], 0, hc0, hr0 + ti->rb[sb] - p.kv_row0, bh);
        }
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
    // ================= V producer: the V halo rows of each sub-tile of tile it into ring slot
    // it % kStagesV once PV of tile it - kStagesV has completed
    const int per = p.tiles_h * p.tiles_w;
    const int u0 = t_begin / per, rem0 = t_begin - u0 * per;
    int h = u0 / p.B, b = u0 - h * p.B, tr = rem0 / p.tiles_w, tcol = rem0 - tr * p.tiles_w;
    for (int it = 0; it < ntile; ++it) {
      const int s = it % kStagesV;
      mbar_wait_producer(&empty_v[s], ((it / kStagesV) & 1) ^ 1);
      const int bh = p.pair ? 2 * b * p.heads + h : b * p.heads + h;
      const int i0 = p.q_row0 + tr * kTQH, j0 = tcol * kTQW;
      if (elect_one()) {
        mbar_expect_tx(&full_v[s], 2 * C::BOX_BYTES);
#pragma unroll
        for (int sb = 0; sb < 2; ++sb) {
          uint8_t *dst = smem + C::V_OFF + s * C::V_BYTES + sb * C::SUB_BYTES;
          const int row = wstart(min(i0 + 4 * sb, q_end - 1), p.H, L) - p.kv_row0;
          if (p.pair) tma_load_5d(dst, &tm_v, &full_v[s], 0, 0, 0, row, bh);
          else tma_load_4d(dst, &tm_v, &full_v[s], 0, wstart(j0, p.W, L), row, bh);
        }
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
    // into slot it & 1 once its Q / K have landed and the slot's previous PV has read its P
    constexpr uint32_t idesc_qk = idesc_el<F16>(64, C::NSUB, false);
    for (int it = 0; it < ntile; ++it) {
      const int s = it % kStagesQK, g = it & 1;
      wait_bar(&full[s], (it / kStagesQK) & 1);
      if (lane == 0) trace_ev(p, it, 1);
      wait_bar(&slot_free[g], ((it >> 1) & 1) ^ 1);
      if (lane == 0) trace_ev(p, it, 2);
      tc_fence_after();
      const uint64_t dq = sdesc_sw<kRB>(smem_u32(smem + s * C::QK_BYTES));
      const uint64_t dk0 = dq + (C::Q_BYTES >> 4), dk1 = dk0 + (C::SUB_BYTES >> 4);
      const uint32_t d0 = tmem + g * C::NSUB, d1 = d0 + ((uint32_t)16 << 16);
      if (elect_one()) {  // two independent accumulation chains (sub-tiles) interleaved; K-steps of 16
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ko = (k * 32) >> 4;
          mma_ss(d0, dq + ko, dk0 + ko, idesc_qk, k);
          mma_ss(d1, dq + ((64 * kRB) >> 4) + ko, dk1 + ko, idesc_qk, k);
        }
        mma_commit(&s_full[g]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else if (warp == kPvWarp) {
    // ================= PV issuer: O of tile it from P in slot it & 1 once its group wrote it and the
    // epilogue of tile it - 1 (the other group) has read the shared O accumulators
    constexpr uint32_t idesc_pv = idesc_el<F16>(64, D, true);
    for (int it = 0; it < ntile; ++it) {
      const int s = it % kStagesV, g = it & 1;
      wait_bar(&full_v[s], (it / kStagesV) & 1);
      const uint64_t dv0 = sdesc_sw<kRB>(smem_u32(smem + C::V_OFF + s * C::V_BYTES)), dv1 = dv0 + (C::SUB_BYTES >> 4);
      const uint32_t b0 = tmem + g * C::NSUB, b1 = b0 + ((uint32_t)16 << 16);
      const uint32_t o0 = tmem + C::O_COL, o1 = o0 + ((uint32_t)16 << 16);
      wait_bar(&p_ready[g], (it >> 1) & 1);
      if (lane == 0) trace_ev(p, it, 3);
      if (it > 0) wait_bar(o_free, (it - 1) & 1);
      if (lane == 0) trace_ev(p, it, 4);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < C::KSTEPS; ++ks) {
          const uint32_t voff = (ks * 16 * kRB) >> 4, oc = (ks % C::OACC) * D;
          const uint32_t a = ks >= C::OACC ? 1u : 0u;
          mma_ts(o0 + oc, b0 + ks * 8, dv0 + voff, idesc_pv, a);
          mma_ts(o1 + oc, b1 + ks * 8, dv1 + voff, idesc_pv, a);
        }
        mma_commit(&o_full[g]);
        mma_commit(&empty_v[s]);
        mma_commit(&slot_free[g]);
      }
      __syncwarp();
    }
  } else {
    // ================= softmax + epilogue: two groups of 8 warps alternate tiles (group g = tiles
    // with it & 1 == g, TMEM slot g).  In a group, warp w: lane quarter q = w & 3, union-row half
    // hf = (w >> 2) & 1.  One thread per query: lane l < 16 is query l of the quarter's 4x4 block of
    // sub-tile 0, lane l >= 16 of sub-tile 1 (their S rows are relative to their own halo base rb_s,
    // so both halves share the union columns).  S of the warp's UH union rows goes to registers (one
    // wait), the two warps of a quarter combine row max and sum through shared memory, and P is
    // written row by row over the consumed S.
    // Softmax with an upper-bound shift: m = max(raw s over the union) * scale*log2e + the bias max
    // over the query's window (per window class, from a small table); m >= the true row max, so every
    // exp2(x - m) <= 1, and P = exp2(x - m) / sum is exact up to fp32 rounding unless m overshoots by
    // > 60 (log2) -- detected by sum < 2^-60, then the rows are redone with the exact max.
    const int g = warp >> 3, hf = (warp >> 2) & 1, quarter = warp & 3;
    const int sub = lane >> 4, r = (lane >> 2) & 3, c = lane & 3;
    const int u0 = hf * C::UH;  // first union row of this warp
    float *tbl = (float *)(smem + C::TBL_OFF) + g * 2 * C::TBL_FLOATS;  // the group's two parity copies
    float *ex_max = (float *)(smem + C::EX_OFF) + g * 512;             // [quarter][half][lane]
    float *ex_sum = ex_max + 256;
    float *rbs = (float *)(smem + C::RB_OFF) + g * C::RB_FLOATS;       // scaled RPB, then window maxima
    float *tmx = rbs + C::TT * C::TT;
    const int stid = threadIdx.x - g * 256;
    const int Lh = wlen(p.H, L), Lw = wlen(p.W, L);
    const float2 sl2x2 = make_float2(p.scale_log2, p.scale_log2);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t slot_base = lane_base + g * C::NSUB;
    const int ex_me = (quarter * 2 + hf) * 32 + lane, ex_other = ex_me + (hf ? -32 : 32);
    const uint32_t bar_q = 3 + g * 4 + quarter;  // named barrier of the quarter's two warps
    int cur_head = -1;
    for (int it = g; it < ntile; it += 2) {
      const uint32_t ph = (it >> 1) & 1;
      wait_bar(&ti_full[it % kTInfo], (it / kTInfo) & 1);
      const FTile &ti = tinfo[it % kTInfo];
      const int bh = ti.bh, h = ti.head, i0 = ti.i0, j0 = ti.j0, hr0 = ti.hr0, hc0 = ti.hc0;
      const int ucr = __shfl_sync(0xffffffffu, ti.uc[quarter], 0);
      const int rb = ti.rb[sub];
      if (h != cur_head) {  // (re)build the group's masked, pre-scaled bias tables (two parity copies:
        // copy x holds column b at kTblOff + x + b, so every thread's row start is 8-byte aligned) and
        // the bias maximum over each window class (dr, dc)
        named_bar_sync(1 + g, 256);
        for (int e = stid; e < C::TT * C::TT; e += 256) rbs[e] = p.rpb ? __ldg(&p.rpb[h * C::TT * C::TT + e]) * p.scale_log2 : 0.f;
        named_bar_sync(1 + g, 256);
        for (int row = stid; row < 2 * L * C::TROWS; row += 256) {  // one table row per thread
          const int x = row / (L * C::TROWS), dc = row / C::TROWS % L, rr = row % C::TROWS;
          float *dst = tbl + row * kTblStride;
          const float *src = rbs + rr * C::TT;
          const bool rv = rr < C::TT;
#pragma unroll 4
          for (int e = 0; e < kTblStride; ++e) {
            const int cb = e - kTblOff - x;
            dst[e] = (rv && cb >= dc && cb < dc + Lw) ? src[cb] : -INFINITY;
          }
        }
        // window maxima, separably: row-wise sliding maxima m1[a][dc] over [dc, dc + Lw), then
        // tmx[dr][dc] = max over rows [dr, dr + Lh) of m1 (7 + 7 dependent loads instead of 49)
        float *m1 = tmx + L * L;
        for (int e = stid; e < C::TT * L; e += 256) {
          const int a = e / L, dc = e - a * L;
          float m = -INFINITY;
          for (int b2 = dc; b2 < dc + Lw; ++b2) m = fmaxf(m, rbs[a * C::TT + b2]);
          m1[e] = m;
        }
        named_bar_sync(1 + g, 256);
        for (int e = stid; e < L * L; e += 256) {
          const int dr = e / L, dc = e - dr * L;
          float m = -INFINITY;
          for (int a = dr; a < dr + Lh; ++a) m = fmaxf(m, m1[a * L + dc]);
          tmx[e] = m;
        }
        named_bar_sync(1 + g, 256);
        cur_head = h;
        if (stid == 0 && it < 2) trace_gt(p, 2);
      }
      // this thread's query and window geometry (pair mode: j is the column inside member
      // quarter >> 1, whose keys start at halo column (quarter >> 1) * PW)
      const int i = i0 + 4 * sub + r, j = p.pair ? 4 * (quarter & 1) + c : j0 + 4 * quarter + c;
      const int jv = p.pair ? (quarter >> 1) * C::PW : 0;  // halo column offset of the member
      const int ic = min(i, q_end - 1), jc = min(j, p.W - 1);
      const int si = wstart(ic, p.H, L), sj = wstart(jc, p.W, L);
      const int dc = sj - jc + L - 1;                                // column-clamp class
      const float tmax = tmx[(si - ic + L - 1) * L + dc];            // bias max over the window
      const bool trc = g == 0 && hf == 0 && quarter == 0 && lane == 0;
      float sum, mq;
      // the tile's softmax for an even (ODD = 0: UW loaded columns, all in the union) or odd union
      // origin (ODD = 1: UW + 2 columns from the even column before it; the first and last are
      // outside the union).  The origin is per quarter (warp-uniform), and even except at borders.
      auto softmax = [&](auto odd_tag) {
        constexpr int ODD = decltype(odd_tag)::value;
        constexpr int NC = C::UW + 2 * ODD, NPK = NC / 2;
        const int uc = ucr - ODD;                                    // first loaded (even) column
        const int bcol0 = hc0 + uc - jc - jv + L - 1;                // bias column of loaded col 0
        const int cp = bcol0 & 1;                                    // parity copy: aligned row start
        const float *tcls = tbl + cp * C::TBL_FLOATS + dc * C::TROWS * kTblStride + kTblOff + cp + bcol0;
        auto trow = [&](int u) {  // bias row of union row u0 + u (the -inf row outside the window)
          const int pr = hr0 + rb + u0 + u;
          return (const float2 *)(tcls + ((unsigned)(pr - si) < (unsigned)Lh ? pr - ic + L - 1 : C::TT) * kTblStride);
        };
        if (trc) trace_ev(p, it, 5);
        wait_bar(&s_full[g], ph);
        if (trc) trace_ev(p, it, 6);
        if (trc && it == 0) trace_gt(p, 3);
        tc_fence_after();
        uint32_t sv[C::UH][NC];
#pragma unroll
        for (int u = 0; u < C::UH; ++u) ld_row<NC>(slot_base + (u0 + u) * C::HP + uc, sv[u]);
        tc_wait_ld();
        float ms = -INFINITY;
#pragma unroll
        for (int u = 0; u < C::UH; ++u)
#pragma unroll
          for (int k = ODD; k < NC - ODD; k += 2)
            ms = ODD ? fmax3(ms, __uint_as_float(sv[u][k]), k + 1 < NC - ODD ? __uint_as_float(sv[u][k + 1]) : -INFINITY)
                     : fmax3(ms, __uint_as_float(sv[u][k]), __uint_as_float(sv[u][k + 1]));
        ex_max[ex_me] = ms;
        named_bar_sync(bar_q, 64);  // also: both warps' S is in registers, P may overwrite S
        ms = fmaxf(ms, ex_max[ex_other]);
        if (trc) trace_ev(p, it, 7);
        // P rows: the warp's packed rows zeroed (the second warp also the K-step padding), then each
        // row's NPK packed union columns written at the quarter's (even) union origin
        const uint32_t p_addr = slot_base + u0 * C::PROW;
        if (hf == 0) st_zero<C::UH * C::PROW>(p_addr);
        else st_zero<C::NSUB / 2 - C::UH * C::PROW>(p_addr);
        tc_wait_st();
        auto exp_rows = [&](float m) {
          const float2 nm = make_float2(-m, -m);
          float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int u = 0; u < C::UH; ++u) {
            const float2 *t = trow(u);
            float2 tv[NPK];
#pragma unroll
            for (int k = 0; k < NPK; ++k) tv[k] = t[k];
            uint32_t pk[NPK];
#pragma unroll
            for (int k = 0; k < NPK; ++k) {
              const float2 xx = __ffma2_rn(make_float2(__uint_as_float(sv[u][2 * k]), __uint_as_float(sv[u][2 * k + 1])),
                                           sl2x2, tv[k]);
              const float2 a = __fadd2_rn(xx, nm);
              const float2 e = make_float2(ODD && k == 0 ? 0.f : ex2(a.x), ODD && k == NPK - 1 ? 0.f : ex2(a.y));
              sum2 = __fadd2_rn(sum2, e);
              pk[k] = pack_el<F16>(e.x, e.y);
            }
            st_row<NPK>(p_addr + u * C::PROW + (uc >> 1), pk);
          }
          const float sm = sum2.x + sum2.y;
          ex_sum[ex_me] = sm;
          named_bar_sync(bar_q, 64);
          return sm + ex_sum[ex_other];
        };
        mq = fmaf(ms, p.scale_log2, tmax);
        while (true) {
          sum = exp_rows(mq);
          if (!__any_sync(0xffffffffu, !(sum >= 0x1p-60f))) break;
          // rare (bias range > ~60 in log2 units inside one window): redo with the exact row max of x.
          // Both warps of the quarter take this branch together (same queries, same sums); after it
          // the row maximum contributes exp2(0) = 1 to the sum, so the loop ends.
          float mx = -INFINITY;
#pragma unroll
          for (int u = 0; u < C::UH; ++u) {
            const float2 *t = trow(u);
#pragma unroll
            for (int k = 0; k < NPK; ++k) {
              const float2 xx = __ffma2_rn(make_float2(__uint_as_float(sv[u][2 * k]), __uint_as_float(sv[u][2 * k + 1])),
                                           sl2x2, t[k]);
              mx = fmax3(mx, ODD && k == 0 ? -INFINITY : xx.x, ODD && k == NPK - 1 ? -INFINITY : xx.y);
            }
          }
          ex_max[ex_me] = mx;
          named_bar_sync(bar_q, 64);  // (the other warp read ex_sum before arriving here)
          mx = fmaxf(mx, ex_max[ex_other]);
          if (!(sum >= 0x1p-60f)) mq = mx;
        }
      };
      if (ucr & 1) softmax(std::integral_constant<int, 1>());
      else softmax(std::integral_constant<int, 0>());
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_ready[g]);
      if (trc) trace_ev(p, it, 9);
      // ---- epilogue: O / sum -> 16-bit (this warp: head dims [16 hf, 16 hf + 16)), LSE
      wait_bar(&o_full[g], ph);
      if (trc) trace_ev(p, it, 10);
      tc_fence_after();
      constexpr int DH = D / 2;  // head dims of this thread (two warps per lane quarter)
      float o[DH];
      {
        uint32_t oa[C::OACC][DH];
#pragma unroll
        for (int a = 0; a < C::OACC; ++a) ld_row<DH>(lane_base + C::O_COL + a * D + DH * hf, oa[a]);
        tc_wait_ld();
#pragma unroll
        for (int z = 0; z < DH; ++z) {
          float acc = __uint_as_float(oa[0][z]);
#pragma unroll
          for (int a = 1; a < C::OACC; ++a) acc += __uint_as_float(oa[a][z]);
          o[z] = acc;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
      if (trc) trace_ev(p, it, 12);
      if (i < q_end && j < p.W) {
        const float inv = 1.f / sum;
        const int bhq = p.pair ? bh + (quarter >> 1) * p.heads : bh;
        const size_t qi = ((size_t)bhq * p.q_rows + (i - p.q_row0)) * p.W + j;
        uint4 *dst = (uint4 *)(p.out + qi * D + DH * hf);
#pragma unroll
        for (int z = 0; z < DH; z += 8)
          dst[z / 8] = make_uint4(pack_el<F16>(o[z] * inv, o[z + 1] * inv), pack_el<F16>(o[z + 2] * inv, o[z + 3] * inv),
                                  pack_el<F16>(o[z + 4] * inv, o[z + 5] * inv), pack_el<F16>(o[z + 6] * inv, o[z + 7] * inv));
        if (p.lse && hf == 0) p.lse[qi] = (mq + __log2f(sum)) * 0.69314718055994531f;
      }
      if (trc) trace_ev(p, it, 13);
    }
    if (threadIdx.x == 0) trace_gt(p, 4);
  }
  __syncthreads();
  if (warp == kProducerWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) trace_gt(p, 5);
#ifdef NA2D_TRACE
  if (threadIdx.x == 0 && p.trace) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[16384 + 2 * blockIdx.x + 1] = (long long)gt;
  }
#endif
}

template <int L, int D, bool F16>
cudaError_t launch_fwd(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  using C = Cfg<L, D>;
  const cudaError_t attr_err = tc::ensure_smem_attr((const void *)na2d_fwd_tc_kernel<L, D, F16>, C::SMEM);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tk, tv;
  const int BH = g.B * g.heads;
  const bool pair = pair_mode(g.B, g.H, g.W, g.q_row0, g.q_rows, g.kv_row0, g.kv_rows);
  if (!make_tmap_e16_4d(F16, &tq, q, D, g.W, g.q_rows, BH, 4, 4) ||
      !(pair ? make_tmap_e16_pair(F16, &tk, k, D, g.W, g.kv_rows, g.heads, BH, C::PW, C::UR)
             : make_tmap_e16_4d(F16, &tk, k, D, g.W, g.kv_rows, BH, C::HP, C::UR)) ||
      !(pair ? make_tmap_e16_pair(F16, &tv, v, D, g.W, g.kv_rows, g.heads, BH, C::PW, C::UR)
             : make_tmap_e16_4d(F16, &tv, v, D, g.W, g.kv_rows, BH, C::HP, C::UR)))
    return cudaErrorInvalidValue;
  FwdParams p;
  p.pair = pair;
  p.B = pair ? g.B / 2 : g.B;
  p.heads = g.heads;
  p.H = g.H;
  p.W = g.W;
  p.q_rows = g.q_rows;
  p.q_row0 = g.q_row0;
  p.kv_row0 = g.kv_row0;
  p.tiles_h = (g.q_rows + kTQH - 1) / kTQH;
  p.tiles_w = (g.W + kTQW - 1) / kTQW;
  p.num_tiles = p.B * g.heads * p.tiles_h * p.tiles_w;
  p.scale_log2 = g.scale * 1.4426950408889634f;
  p.rpb = rpb;
  p.out = (__nv_bfloat16 *)out;
  p.lse = lse;
  p.trace = (long long *)debug_trace_buffer();
  const int grid = p.num_tiles < num_sms() ? p.num_tiles : num_sms();
  ProfScope ps("na2d_fwd_tc", st);
  const cudaError_t e = launch_pdl(na2d_fwd_tc_kernel<L, D, F16>, grid, kThreads, C::SMEM, st, tq, tk, tv, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

bool tc_forward_supported(const Geo &g) {
  return (g.dtype == NA2D_BF16 || g.dtype == NA2D_F16) && (g.d == 16 || g.d == 32 || g.d == 64) &&
         (g.L == 3 || g.L == 5 || g.L == 7) && tmap_available();
}

namespace {
template <int D, bool F16>
cudaError_t fwd_for_d(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                      float *lse, cudaStream_t st) {
  switch (g.L) {
    case 3: return launch_fwd<3, D, F16>(g, q, k, v, rpb, out, lse, st);
    case 5: return launch_fwd<5, D, F16>(g, q, k, v, rpb, out, lse, st);
    case 7: return launch_fwd<7, D, F16>(g, q, k, v, rpb, out, lse, st);
  }
  return cudaErrorInvalidValue;
}
template <bool F16>
cudaError_t fwd_for_el(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  switch (g.d) {
    case 16: return fwd_for_d<16, F16>(g, q, k, v, rpb, out, lse, st);
    case 32: return fwd_for_d<32, F16>(g, q, k, v, rpb, out, lse, st);
    case 64: return fwd_for_d<64, F16>(g, q, k, v, rpb, out, lse, st);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t tc_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  return g.dtype == NA2D_F16 ? fwd_for_el<true>(g, q, k, v, rpb, out, lse, st)
                             : fwd_for_el<false>(g, q, k, v, rpb, out, lse, st);
}

}  // namespace na2d
