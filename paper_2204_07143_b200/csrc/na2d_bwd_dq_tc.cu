// na2d_bwd_dq_tc.cu -- backward kernel B1 (query-centric) on tcgen05/TMEM/TMA, sm_100a:
// steps a6, a7, a9, a10 of the analytic gradient of Eq. 2 (R5):
//   D_q   = dO_q . O_q = sum_k P dP  (exact fp32 from the recomputed P, dP; written for B2)
//   P     = exp2(s*scale*log2e + B' - LSE_q*log2e)      (recomputed; B' masked pre-scaled bias)
//   dP    = dO_q . v_k                                  (tcgen05, TMEM)
//   dS    = P (dP - D_q)
//   dQ_q  = scale * sum_k dS k_k                        (tcgen05 TS MMA, dS bf16 from TMEM)
//   dB    = scale * sum dS over (b, q, k) per relative-position cell
// Geometry is the forward's: 8 x 16 query tiles = two M=64 sub-tiles, halo 14(+) x 24 keys, TMEM
// lane quarter q owns the 4 x 4 query blocks at columns [4q, 4q+4) of both sub-tiles and
// processes the (4+L-1) x (L+5) union of their windows.
// dRPB without per-element atomics: tiles are visited in an order grouped by geometry class
// (interior tile rows/columns form one class, each border tile row/column its own) and head;
// within a class each lane's union element -> bias cell map is fixed, so each lane accumulates
// dS in union coordinates in registers and flushes (masked to its window) into a per-CTA
// shared table only when the class or head changes.  Per-CTA partial tables are reduced in
// fixed CTA order by a separate small kernel.
#include <math.h>

#include <mutex>

#include "na2d_internal.cuh"
#include "na2d_profile.cuh"
#include "na2d_sm100.cuh"
#include "na2d_tc.cuh"
#include "na2d_tc_bwd.cuh"
#include "na2d_tc_common.cuh"
#include "na2d_tmap.cuh"

namespace na2d {
namespace {

using namespace sm100;
using namespace tc;

#ifndef NA2D_B1_GROUPS
#define NA2D_B1_GROUPS 3
#endif
constexpr int kGroups = NA2D_B1_GROUPS;  // elementwise warp groups (each covers the 4 TMEM lane quarters)
// S / dP issued per elementwise group's union row pairs, last group first, each part with its own
// commit: a group starts pass 1 as soon as its own columns have landed
#ifndef NA2D_B1_SPLIT
#define NA2D_B1_SPLIT 1
#endif
static_assert(!NA2D_B1_SPLIT || kGroups == 3, "S / dP parts of 1 or 2 row pairs (N = 48 / 96) assume 3 groups");
constexpr int kThreads = 64 + kGroups * 128;  // warps 0.. elementwise, then the TMA and MMA warps
// (the sub-partition scheduler favours the highest warp id: the producer / MMA warps never wait for
// the elementwise warps sharing their sub-partitions)
constexpr int kProducerWarp = 4 * kGroups, kMmaWarp = 4 * kGroups + 1;

// Per-stage tile description, written by the producer before it arms full[stage] (the class-grouped
// order's decode and the window origins, computed once instead of in every warp).
struct TileInfoQ {
  int bh, i0, j0, cls, hr0, hc0;
  int rb[2];  // first union row of sub-tile / half h (relative to hr0)
  int uc[4];  // even first union column of lane quarter q (relative to hc0)
};

template <int L, int D>
struct CfgQ {
  static constexpr int ROWB = 2 * D;  // bytes per 16-bit row: one swizzle atom (32 / 64 / 128 B)
  static constexpr int HR = kTQH + L - 1;
  static constexpr int UR = 4 + L - 1;
  static constexpr int NSUB = UR * kHCP;
  static constexpr int UCW = L + 5;
  // union row pairs split between the kGroups elementwise warps of a TMEM lane quarter: group g
  // takes pairs [pr0(g), pr0(g+1)).  Each group writes its dS rows over its own consumed S rows
  // (row u at DS_COL + u*12 + shift(g), shift(g) = pr0(g)*24), so dQ MMA K-step ks (16 keys; a
  // row pair is 3 K-steps) reads from column ks*8 + shift(group of pair ks/3)
  static constexpr int PAIRS = UR / 2;
  static constexpr int PA = (PAIRS + kGroups - 1) / kGroups;  // max pairs of a group
  __host__ __device__ static constexpr int pr0(int g) { return g * PAIRS / kGroups; }
  __host__ __device__ static constexpr int ds_shift_of_ks(int ks) {
    int g = 0;
    while (g + 1 < kGroups && pr0(g + 1) <= ks / 3) ++g;
    return pr0(g) * kHCP;
  }
  static_assert(2 * kHCP == 3 * 16, "a row pair is 3 K-steps");
  static constexpr int DS_COL = 0;         // dS (bf16 pairs) over consumed S columns
  // TMEM: S [0, NSUB), dP [NSUB, 2 NSUB), dQ partial accumulators [2 NSUB, +QACC*32).  dQ lives
  // outside S / dP, so S / dP of the next tile are issued right behind this tile's dQ MMAs and the
  // dQ read-out (epilogue) leaves the critical path.
  static constexpr int DP_COL = NSUB;
  static constexpr int Q_COL = 2 * NSUB;
  // dQ MMAs of N = QN head dims per pass (NQP passes: at d = 64 the 32 free TMEM columns hold one
  // 32-dim half at a time, read out by the epilogue before the next half), QACC independent chains
  static constexpr int QN = D < 32 ? D : 32, NQP = D / QN;
  static constexpr int QACC = (512 - Q_COL) / QN < 3 ? (512 - Q_COL) / QN : 3;
  static_assert(QACC >= 1, "TMEM budget");
  static constexpr int NST = D <= 32 ? 2 : 1;  // Q / dO / K / V stages (one at d = 64: shared memory)
  static constexpr int KV_ROWS = HR * kHCP;
  static constexpr int Q_BYTES = 128 * ROWB;
  static constexpr int KV_BYTES = (KV_ROWS * ROWB + 1023) / 1024 * 1024;
  static constexpr int TX_BYTES = 2 * Q_BYTES + 2 * KV_ROWS * ROWB;  // Q, dO, K, V by TMA
  static constexpr int LD_BYTES = 2 * Q_BYTES + 2 * KV_BYTES;          // their (padded) buffers
  static constexpr int LSE_OFF = LD_BYTES;                          // + the tile's 128 LSE (log2)
  static constexpr int STAGE_BYTES = LD_BYTES + 1024;
  static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1 KB aligned (swizzled TMA / UMMA)");
  static constexpr int TT = 2 * L - 1;
  static constexpr int TBL_OFF = NST * STAGE_BYTES;
  // two parity copies of the masked bias table (8-byte aligned element pairs: LDS.64)
  static constexpr int OUT_OFF = (TBL_OFF + 2 * BiasTable<L>::FLOATS * 4 + 1023) / 1024 * 1024;  // dQ staging
  static constexpr int HALF_B = 16 * ROWB;                 // one 4 x 4 block of dQ rows (TMA store box)
  static constexpr int DB_OFF = OUT_OFF + 4 * 2 * HALF_B;
  static constexpr int DP_OFF = DB_OFF + ((8 * kGroups * TT * TT * 4 + 255) / 256) * 256;  // partial D
  static constexpr int RS_OFF = DP_OFF + kGroups * 128 * 4;  // the head's bias values (table build)
  static constexpr int TI_OFF = RS_OFF + (TT * TT * 4 + 15) / 16 * 16;
  static constexpr int BAR_OFF = TI_OFF + NST * 64;
  static_assert(sizeof(TileInfoQ) <= 64, "TileInfoQ");
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

__device__ __forceinline__ TileOrder::Tile decode(const BwdQParams &p, int t) { return p.order.decode(t); }
// debug timeline: trace[4096 + (cta / 37 * 32 + tile) * 32 + ev] for CTAs 0, 37, 74, 111 (tile = CTA-local tile index;
// the first 4096 slots belong to B2)
__device__ __forceinline__ void qtrace_gt(const BwdQParams &p, int slot) {  // wall clock into tile row 0
#ifndef NA2D_TRACE
  return;
#endif
  if (p.trace && blockIdx.x % 37 == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[4096 + ((size_t)(blockIdx.x / 37) * 32) * 32 + slot] = (long long)gt;
  }
}
__device__ __forceinline__ void qtrace(const BwdQParams &p, int it, int ev) {
#ifndef NA2D_TRACE
  return;
#endif
  if (p.trace && blockIdx.x % 37 == 0 && it < 32) p.trace[4096 + ((size_t)(blockIdx.x / 37) * 32 + it) * 32 + ev] = clock64();
}

template <int L, int D, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const __grid_constant__ CUtensorMap tm_dq, const BwdQParams p) {
  using C = CfgQ<L, D>;
  constexpr int kRB = C::ROWB, kStages = C::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float *tbl = (float *)(smem + C::TBL_OFF);
  float *s_db = (float *)(smem + C::DB_OFF);  // 16 private dRPB tables: (elementwise warp, half)
  TileInfoQ *tinfo = (TileInfoQ *)(smem + C::TI_OFF);
  uint64_t *bars = (uint64_t *)(smem + C::BAR_OFF);
  uint64_t *full = bars, *empty = bars + kStages;
  uint64_t *sp_full = bars + 2 * kStages, *ds_full = sp_full + 1, *dq_full = sp_full + 2, *dq_free = sp_full + 3;
  uint64_t *sp_part = sp_full + 4;  // [kGroups]: S / dP columns of group g's row pairs (NA2D_B1_SPLIT)
  uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages + 4 + kGroups);

  // broadcast from lane 0 so the compiler treats the warp index (and the TMEM addresses
  // derived from it) as warp-uniform: they stay in uniform registers, no R2UR per tcgen05.ld
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int t_begin = p.ranges.start[blockIdx.x], t_end = p.ranges.start[blockIdx.x + 1];
  const int q_end = p.q_row0 + p.q_rows;
  if (threadIdx.x == 0) qtrace_gt(p, 16);

  if (warp == kProducerWarp && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1 + 32);  // expect_tx arrive + 32 lanes staging the tile's LSE
      mbar_init(&empty[s], 1);
    }
    mbar_init(sp_full, 1);
    for (int g = 0; g < kGroups; ++g) mbar_init(&sp_part[g], 1);
    mbar_init(ds_full, 4 * kGroups);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_dq);
  }
  for (int c = threadIdx.x; c < 8 * kGroups * C::TT * C::TT; c += kThreads) s_db[c] = 0.f;
  if (warp == kProducerWarp) tmem_alloc<512>(tmem_slot);
#ifdef NA2D_TRACE
  if (threadIdx.x == 0 && p.trace) {  // per-CTA wall-clock span (load balance)
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[16896 + 2 * blockIdx.x] = (long long)gt;
  }
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // the masked bias table of head h (elementwise warps, named barrier 1): the head's bias values
  // staged in shared memory (one global load per thread), then the two parity copies built from there
  constexpr int kEw = kGroups * 128;  // elementwise threads
  const int Lw = wlen(p.W, L);
  const float sl2 = p.scale * 1.4426950408889634f;
  auto build_table = [&](int h) {
    named_bar_sync(1, kEw);
    float *rs = (float *)(smem + C::RS_OFF);
    for (int e = threadIdx.x; e < C::TT * C::TT; e += kEw) rs[e] = p.rpb ? __ldg(&p.rpb[h * C::TT * C::TT + e]) * sl2 : 0.f;
    named_bar_sync(1, kEw);
    BiasTable<L>::build_rows_smem(tbl, p.rpb ? rs : nullptr, Lw, 2, 0, threadIdx.x, kEw);
    named_bar_sync(1, kEw);
  };
  // the first tile's table is built before griddepcontrol.wait: the RPB is an input, not an output of
  // the previous kernel, so this overlaps that kernel's tail
  const int first_head = t_begin < t_end ? decode(p, t_begin).bh % p.heads : -1;
  if (warp < 4 * kGroups && first_head >= 0) build_table(first_head);
  pdl_wait();  // the previous kernel (forward / last step's B2) is complete: global memory from here on
  if (threadIdx.x == 0) qtrace_gt(p, 19);
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.b2_tile_counter) *p.b2_tile_counter = 0;  // for B2 (next)
  if (p.drpb_part) {  // this CTA's partial tables (only this CTA writes them; B2 reads them after B1)
    for (int c = threadIdx.x; c < p.heads * C::TT * C::TT; c += kThreads)
      p.drpb_part[(size_t)blockIdx.x * p.heads * C::TT * C::TT + c] = 0.f;
    __syncthreads();
  }

  if (warp == kProducerWarp) {
    // ================= producer: TMA (Q, dO 4x4 blocks; K, V halo) + the tile's LSE (log2 units)
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      const int s = it % kStages;
      mbar_wait_producer(&empty[s], ((it / kStages) & 1) ^ 1);
      const TileOrder::Tile g = decode(p, t);
      const int hr0 = wstart(g.i0, p.H, L), hc0 = wstart(g.j0, p.W, L);
      uint8_t *st = smem + s * C::STAGE_BYTES;
      TileInfoQ *ti = tinfo + s;
      const bool pair = p.order.pair;  // members at halo columns 0 / kHCP / 2 (tc::pair_mode)
      if (lane < 2) ti->rb[lane] = wstart(min(g.i0 + 4 * lane, q_end - 1), p.H, L) - hr0;
      if (lane < 4)
        ti->uc[lane] = (pair ? (lane >> 1) * (kHCP / 2) + wstart(min(4 * (lane & 1), p.W - 1), p.W, L)
                             : wstart(min(g.j0 + 4 * lane, p.W - 1), p.W, L) - hc0) & ~1;
      if (lane == 0) {
        ti->bh = g.bh;
        ti->i0 = g.i0;
        ti->j0 = g.j0;
        ti->cls = g.cls;
        ti->hr0 = hr0;
        ti->hc0 = hc0;
      }
      __syncwarp();
      if (elect_one()) {
        mbar_expect_tx(&full[s], C::TX_BYTES);
#pragma unroll
        for (int sb = 0; sb < 2; ++sb)
#pragma unroll
          for (int qb = 0; qb < 4; ++qb) {
            const int r0 = (64 * sb + 16 * qb) * kRB;
            const int qc = pair ? 4 * (qb & 1) : g.j0 + 4 * qb, qbh = pair ? g.bh + (qb >> 1) * p.heads : g.bh;
            tma_load_4d(st + r0, &tm_q, &full[s], 0, qc, g.i0 - p.q_row0 + 4 * sb, qbh);
            tma_load_4d(st + C::Q_BYTES + r0, &tm_do, &full[s], 0, qc, g.i0 - p.q_row0 + 4 * sb, qbh);
          }
        if (pair) {  // both members' halo rows side by side (pair tensor maps, row pitch kHCP)
          tma_load_5d(st + 2 * C::Q_BYTES, &tm_k, &full[s], 0, 0, 0, hr0 - p.kv_row0, g.bh);
          tma_load_5d(st + 2 * C::Q_BYTES + C::KV_BYTES, &tm_v, &full[s], 0, 0, 0, hr0 - p.kv_row0, g.bh);
        } else {
          tma_load_4d(st + 2 * C::Q_BYTES, &tm_k, &full[s], 0, hc0, hr0 - p.kv_row0, g.bh);
          tma_load_4d(st + 2 * C::Q_BYTES + C::KV_BYTES, &tm_v, &full[s], 0, hc0, hr0 - p.kv_row0, g.bh);
        }
      }
      __syncwarp();
      // LSE of query (half, quarter, r, c) at e = half*64 + quarter*16 + r*4 + c; 0 if outside
      float *lse_s = (float *)(st + C::LSE_OFF);
      float lv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = lane + 32 * u, qq = (e >> 4) & 3;
        const int i = g.i0 + 4 * (e >> 6) + ((e >> 2) & 3), j = (pair ? 4 * (qq & 1) : g.j0 + 4 * qq) + (e & 3);
        const int qbh = pair ? g.bh + (qq >> 1) * p.heads : g.bh;
        lv[u] = (i < q_end && j < p.W)
                    ? __ldg(&p.lse[((size_t)qbh * p.q_rows + (i - p.q_row0)) * p.W + j]) * 1.4426950408889634f
                    : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) lse_s[lane + 32 * u] = lv[u];
      mbar_arrive(&full[s]);
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer: S / dP of tile 0; then per tile: (wait dS) dQ of tile it, then
    // S / dP of tile it + 1 straight behind it (the in-order tensor pipe finishes reading dS and the
    // K tile before S / dP overwrite their columns), so the elementwise warps start the next tile
    // while the epilogue reads dQ.
    constexpr uint32_t idesc_s = idesc_el<F16>(64, C::NSUB, false);
    constexpr uint32_t idesc_p1 = idesc_el<F16>(64, 2 * kHCP, false), idesc_p2 = idesc_el<F16>(64, 4 * kHCP, false);
    constexpr uint32_t idesc_q = idesc_el<F16>(64, C::QN, true);
    const int n = t_end - t_begin;
    const uint32_t t0 = tmem, t1 = tmem + ((uint32_t)16 << 16);
    auto issue_sdp = [&](int it) {
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      if (lane == 0) qtrace(p, it, 0);
      const int rb0 = tinfo[s].rb[0], rb1 = tinfo[s].rb[1];
      tc_fence_after();
      // descriptors: per-stage bases + immediate offsets (short issue bursts, no per-MMA chains)
      const uint64_t dqs = sdesc_sw<kRB>(smem_u32(smem + s * C::STAGE_BYTES));
      const uint64_t dk0 = dqs + ((2 * C::Q_BYTES + rb0 * kHCP * kRB) >> 4);
      const uint64_t dk1 = dqs + ((2 * C::Q_BYTES + rb1 * kHCP * kRB) >> 4);
      if (elect_one()) {
#if NA2D_B1_SPLIT
        // group g's row pairs = S / dP columns [48 pr0(g), 48 pr0(g+1)) = keys of the same range
#pragma unroll
        for (int g = kGroups - 1; g >= 0; --g) {
          const int c0 = 2 * kHCP * C::pr0(g), nc = 2 * kHCP * (C::pr0(g + 1) - C::pr0(g));
          const uint32_t id = nc == 2 * kHCP ? idesc_p1 : idesc_p2;
          const uint32_t bo = (c0 * kRB) >> 4;  // key offset of the part in the K / V halos
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t ko = (k * 32) >> 4;
            mma_ss(t0 + c0, dqs + ko, dk0 + bo + ko, id, k);
            mma_ss(t0 + C::DP_COL + c0, dqs + (C::Q_BYTES >> 4) + ko, dk0 + (C::KV_BYTES >> 4) + bo + ko, id, k);
            mma_ss(t1 + c0, dqs + ((64 * kRB) >> 4) + ko, dk1 + bo + ko, id, k);
            mma_ss(t1 + C::DP_COL + c0, dqs + ((C::Q_BYTES + 64 * kRB) >> 4) + ko, dk1 + (C::KV_BYTES >> 4) + bo + ko, id, k);
          }
          mma_commit(&sp_part[g]);
        }
#else
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ko = (k * 32) >> 4;
          mma_ss(t0, dqs + ko, dk0 + ko, idesc_s, k);
          mma_ss(t0 + C::DP_COL, dqs + (C::Q_BYTES >> 4) + ko, dk0 + (C::KV_BYTES >> 4) + ko, idesc_s, k);
          mma_ss(t1, dqs + ((64 * kRB) >> 4) + ko, dk1 + ko, idesc_s, k);
          mma_ss(t1 + C::DP_COL, dqs + ((C::Q_BYTES + 64 * kRB) >> 4) + ko, dk1 + (C::KV_BYTES >> 4) + ko, idesc_s, k);
        }
        mma_commit(sp_full);
#endif
      }
      __syncwarp();
      if (lane == 0) qtrace(p, it, 2);
    };
    if (n > 0) issue_sdp(0);
    for (int it = 0; it < n; ++it) {
      const int s = it % kStages;
      const uint32_t ph = it & 1;
      mbar_wait(ds_full, ph);
      if (lane == 0) qtrace(p, it, 3);
      const int rb0 = tinfo[s].rb[0], rb1 = tinfo[s].rb[1];
      const uint64_t dk0 = sdesc_sw<kRB>(smem_u32(smem + s * C::STAGE_BYTES) + 2 * C::Q_BYTES + rb0 * kHCP * kRB);
      const uint64_t dk1 = dk0 + (((rb1 - rb0) * kHCP * kRB) >> 4);
#pragma unroll 1
      for (int hq = 0; hq < C::NQP; ++hq) {
        const int np = it * C::NQP + hq;  // dQ pass index (one dq_full / dq_free phase each)
        mbar_wait(dq_free, (np & 1) ^ 1);  // the epilogue has read the previous pass
        if (lane == 0) qtrace(p, it, 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ho = (hq * C::QN * 2) >> 4;  // head-dim offset of the pass in K's rows
#pragma unroll
          for (int ks = 0; ks < C::NSUB / 16; ++ks) {
            const uint32_t ko = (ks * 16 * kRB) >> 4;
            const uint32_t ao = C::DS_COL + ks * 8 + C::ds_shift_of_ks(ks), qo = C::Q_COL + (ks % C::QACC) * C::QN;
            mma_ts(t0 + qo, t0 + ao, dk0 + ko + ho, idesc_q, ks >= C::QACC);
            mma_ts(t1 + qo, t1 + ao, dk1 + ko + ho, idesc_q, ks >= C::QACC);
          }
          mma_commit(dq_full);
          if (hq == C::NQP - 1) mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) qtrace(p, it, 4);
      if (it + 1 < n) issue_sdp(it + 1);
    }
  } else {
    // ================= elementwise (warps 2.. -> TMEM lane quarter warp % 4): group grp takes union
    // row pairs [pr0, pr1) of every tile; group 0 also runs the epilogue
    const int quarter = warp & 3, grp = warp >> 2;
    const int pr0 = C::pr0(grp), pr1 = C::pr0(grp + 1);
    const int half = lane >> 4, r = (lane >> 2) & 3, c = lane & 3;
    const int gtid = threadIdx.x;
    float *s_dpart = (float *)(smem + C::DP_OFF);
    const int Lh = wlen(p.H, L);
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const float2 sl2x2 = make_float2(sl2, sl2);
    // this (warp, half)'s private dRPB table: within one instruction the 16 lanes of a half touch
    // distinct cells (no intra-instruction address conflicts, no other warp contending), but
    // different (u, z) of different lanes do meet, so the adds stay atomic (RED to shared)
    float *my_db = s_db + ((grp * 4 + quarter) * 2 + half) * C::TT * C::TT;
    uint8_t *ostage = smem + C::OUT_OFF + quarter * 2 * C::HALF_B;
    // dRPB accumulator in union coordinates for the current (class, head) and its geometry
    float2 acc[2 * C::PA][C::UCW / 2];  // local rows: union row 2 * pr0 + u
#pragma unroll
    for (int u = 0; u < 2 * C::PA; ++u)
#pragma unroll
      for (int z = 0; z < C::UCW / 2; ++z) acc[u][z] = make_float2(0.f, 0.f);
    int cur_key = -1, cur_head = -1;
    int f_wr = 0, f_wc = 0, f_brow = 0, f_bcol = 0;  // geometry of the accumulated class
    bool f_valid = false;  // own query inside the map / band (constant within a class)
    auto flush = [&]() {
      // masked to this lane's window; cells (f_brow + ug, f_bcol + z) for union row ug.  Lanes of
      // queries past the edge (clamped onto an edge query's cells, dS = 0) skip the adds.
#pragma unroll
      for (int u = 0; u < 2 * C::PA; ++u) {
        const int ug = 2 * pr0 + u;
        if (ug >= 2 * pr1) break;
#pragma unroll
        for (int z = 0; z < C::UCW; ++z) {
          const float v = (z & 1) ? acc[u][z / 2].y : acc[u][z / 2].x;
          if (f_valid && (unsigned)(ug - f_wr) < (unsigned)Lh && (unsigned)(z - f_wc) < (unsigned)Lw)
            atomicAdd(&my_db[(f_brow + ug) * C::TT + f_bcol + z], v);
        }
      }
#pragma unroll
      for (int u = 0; u < 2 * C::PA; ++u)
#pragma unroll
        for (int z = 0; z < C::UCW / 2; ++z) acc[u][z] = make_float2(0.f, 0.f);
    };
    uint64_t committed = 0;  // heads (< 64) whose partial table this CTA has written already
    auto commit_head = [&](int head) {  // sum of the private tables -> partials[cta][head]; clear
      named_bar_sync(1, kEw);
      if (head >= 0 && p.drpb_part) {
        // first commit of a head: plain store (no dependent global load); the table was zeroed at entry
        const bool again = head >= 64 || ((committed >> head) & 1);
        for (int e = gtid; e < C::TT * C::TT; e += kEw) {
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < 8 * kGroups; ++w) {
            v += s_db[w * C::TT * C::TT + e];
            s_db[w * C::TT * C::TT + e] = 0.f;
          }
          float *dst = &p.drpb_part[((size_t)blockIdx.x * p.heads + head) * C::TT * C::TT + e];
          *dst = again ? *dst + p.scale * v : p.scale * v;
        }
        if (head < 64) committed |= 1ull << head;
      }
      named_bar_sync(1, kEw);
    };
    cur_head = first_head;  // its table was built before griddepcontrol.wait
    if (gtid == 0) qtrace_gt(p, 20);
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      const uint32_t ph = it & 1;
      const int stage = it % kStages;
      mbar_wait(&full[stage], (it / kStages) & 1);  // tile description and LSE staged
      // copied to registers: the producer refills this stage once the tile's dQ MMAs complete,
      // before the epilogue ends
      const TileInfoQ &ti = tinfo[stage];
      const int bh = ti.bh, i0 = ti.i0, j0 = ti.j0, hr0 = ti.hr0, hc0 = ti.hc0;
      const int rb = ti.rb[half], uc = ti.uc[quarter];
      const int h = bh % p.heads;
      const int key = ti.cls * p.heads + h;
      // pair mode: j is the column inside member quarter >> 1, whose keys start at halo column jv
      const bool pair = p.order.pair;
      const int i = i0 + 4 * half + r, j = pair ? 4 * (quarter & 1) + c : j0 + 4 * quarter + c;
      const int jv = pair ? (quarter >> 1) * (kHCP / 2) : 0, bhq = pair ? bh + (quarter >> 1) * p.heads : bh;
      const int ic = min(i, q_end - 1), jc = min(j, p.W - 1);
      const int si = wstart(ic, p.H, L), sj = wstart(jc, p.W, L);
      const int dc = sj - jc + L - 1;
      const int brow0 = hr0 + rb - ic + L - 1, bcol0 = hc0 + uc - jc - jv + L - 1;
      if (key != cur_key) {
        if (p.rpb && cur_key >= 0) flush();
        if (h != cur_head) {
          if (p.rpb) commit_head(cur_head);
          build_table(h);
          cur_head = h;
        }
        cur_key = key;
        f_valid = i < q_end && j < p.W;
        f_wr = si - hr0 - rb;
        f_wc = sj + jv - hc0 - uc;
        f_brow = brow0;
        f_bcol = bcol0;
      }
      const bool qvalid = i < q_end && j < p.W;
      const size_t qi = ((size_t)bhq * p.q_rows + (ic - p.q_row0)) * p.W + jc;
      // parity copy: row starts (and so every element pair z, z + 1 with z even) 8-byte aligned
      const int cpar = bcol0 & 1;
      const float *tcls = tbl + cpar * BiasTable<L>::FLOATS + dc * BiasTable<L>::TROWS * kTblStride + kTblOff + cpar + bcol0;
      const bool tq = grp == 0 && quarter == 2 && lane == 0;
      if (tq) qtrace(p, it, 8);
      const float nlse2 = -((const float *)(smem + stage * C::STAGE_BYTES + C::LSE_OFF))[half * 64 + quarter * 16 + r * 4 + c];
      const float2 nlse2x2 = make_float2(nlse2, nlse2);
      mbar_wait(NA2D_B1_SPLIT ? &sp_part[grp] : sp_full, ph);
      if (tq) qtrace(p, it, 9);
      if (gtid == 0 && it == 0) qtrace_gt(p, 21);
      tc_fence_after();
      // ---- pass 1: P = exp2(s*scale*log2e + B' - LSE*log2e) (fp32, written over S in place) and
      // D = dO.O = sum_window P dP (exact in fp32: O = sum P V, so dO.O = sum P (dO.v)); element
      // pairs in packed fp32x2 arithmetic
      float Dq = 0.f;
#pragma unroll 1
      for (int u = 2 * pr0; u < 2 * pr1; u += 2) {
        uint32_t sa[C::UCW], sb_[C::UCW], pa_[C::UCW], pb_[C::UCW];
        const uint32_t ca = lane_addr + u * kHCP + uc;
        ld_row<C::UCW>(ca, sa);
        ld_row<C::UCW>(ca + kHCP, sb_);
        ld_row<C::UCW>(ca + C::DP_COL, pa_);
        ld_row<C::UCW>(ca + C::DP_COL + kHCP, pb_);
        const int pr = hr0 + rb + u;
        const bool rva = (unsigned)(pr - si) < (unsigned)Lh, rvb = (unsigned)(pr + 1 - si) < (unsigned)Lh;
        const float *ta = tcls + (rva ? pr - ic + L - 1 : C::TT) * kTblStride;
        const float *tb = tcls + (rvb ? pr + 1 - ic + L - 1 : C::TT) * kTblStride;
        tc_wait_ld();
        // two accumulators per row (shorter dependent FFMA2 chains behind the exp2 results)
        float2 da[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, db[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int z = 0; z < C::UCW; z += 2) {
          const float2 tta = *reinterpret_cast<const float2 *>(ta + z), ttb = *reinterpret_cast<const float2 *>(tb + z);
          const float2 xa = __fadd2_rn(__ffma2_rn(make_float2(__uint_as_float(sa[z]), __uint_as_float(sa[z + 1])),
                                                  sl2x2, tta), nlse2x2);
          const float2 xb = __fadd2_rn(__ffma2_rn(make_float2(__uint_as_float(sb_[z]), __uint_as_float(sb_[z + 1])),
                                                  sl2x2, ttb), nlse2x2);
          const float2 Pa = make_float2(ex2(xa.x), ex2(xa.y)), Pb = make_float2(ex2(xb.x), ex2(xb.y));
          const int w = (z >> 1) & 1;
          da[w] = __ffma2_rn(Pa, make_float2(__uint_as_float(pa_[z]), __uint_as_float(pa_[z + 1])), da[w]);
          db[w] = __ffma2_rn(Pb, make_float2(__uint_as_float(pb_[z]), __uint_as_float(pb_[z + 1])), db[w]);
          sa[z] = __float_as_uint(Pa.x);
          sa[z + 1] = __float_as_uint(Pa.y);
          sb_[z] = __float_as_uint(Pb.x);
          sb_[z + 1] = __float_as_uint(Pb.y);
        }
        Dq += ((da[0].x + da[1].x) + (da[0].y + da[1].y)) + ((db[0].x + db[1].x) + (db[0].y + db[1].y));
        st_row<C::UCW>(ca, sa);
        st_row<C::UCW>(ca + kHCP, sb_);
      }
      // D over the whole window: the two groups' partial sums, added in a fixed order
      s_dpart[grp * 128 + quarter * 32 + lane] = Dq;
      named_bar_sync(2 + quarter, 32 * kGroups);
      Dq = 0.f;
#pragma unroll
      for (int g2 = 0; g2 < kGroups; ++g2) Dq += s_dpart[g2 * 128 + quarter * 32 + lane];
      if (qvalid && grp == 0) p.D[qi] = Dq;
      if (tq) qtrace(p, it, 10);
      tc_wait_st();
      // ---- pass 2: dS = P (dP - D) -> dRPB accumulators (union coordinates) and bf16 pairs over
      // the consumed S/P columns (the dQ MMA's A operand)
      const int zb = uc >> 1;
      const float2 nD = make_float2(-Dq, -Dq);
      const uint32_t ds_base = lane_addr + C::DS_COL + pr0 * kHCP;
#pragma unroll
      for (int lp = 0; lp < C::PA; ++lp) {
        if (pr0 + lp >= pr1) break;
        const int u = 2 * (pr0 + lp), ul = 2 * lp;  // union row, local accumulator row
        uint32_t sa[C::UCW], sb_[C::UCW], pa_[C::UCW], pb_[C::UCW];
        const uint32_t ca = lane_addr + u * kHCP + uc;
        ld_row<C::UCW>(ca, sa);
        ld_row<C::UCW>(ca + kHCP, sb_);
        ld_row<C::UCW>(ca + C::DP_COL, pa_);
        ld_row<C::UCW>(ca + C::DP_COL + kHCP, pb_);
        tc_wait_ld();
        uint32_t da[C::UCW / 2], db[C::UCW / 2];
#pragma unroll
        for (int z = 0; z < C::UCW; z += 2) {
          const float2 dsa = __fmul2_rn(make_float2(__uint_as_float(sa[z]), __uint_as_float(sa[z + 1])),
                                        __fadd2_rn(make_float2(__uint_as_float(pa_[z]), __uint_as_float(pa_[z + 1])), nD));
          const float2 dsb = __fmul2_rn(make_float2(__uint_as_float(sb_[z]), __uint_as_float(sb_[z + 1])),
                                        __fadd2_rn(make_float2(__uint_as_float(pb_[z]), __uint_as_float(pb_[z + 1])), nD));
          acc[ul][z / 2] = __fadd2_rn(acc[ul][z / 2], dsa);
          acc[ul + 1][z / 2] = __fadd2_rn(acc[ul + 1][z / 2], dsb);
          da[z / 2] = pack_el<F16>(dsa.x, dsa.y);
          db[z / 2] = pack_el<F16>(dsb.x, dsb.y);
        }
        const uint32_t prow = ds_base + u * (kHCP / 2);
        st_zero12(prow);
        st_zero12(prow + kHCP / 2);
        st_row<C::UCW / 2>(prow + zb, da);
        st_row<C::UCW / 2>(prow + kHCP / 2 + zb, db);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (tq) qtrace(p, it, 11);
      if (grp) continue;
      // ---- epilogue (group 0): dQ = scale * sum of partial accumulators -> bf16, TMA stores
      // dQ per pass of QN head dims (16-column parts: register pressure): partial accumulators summed,
      // scaled, packed into the swizzled staging row of query (r, c) of block `half` (row R of the box;
      // 16-byte chunk z at the TMA swizzle position of rows of kRB bytes)
      const int R = r * 4 + c;
      uint8_t *orow = ostage + half * C::HALF_B + R * kRB;
      if (lane == 0) bulk_wait_read0();  // this warp's previous store has left the staging
      __syncwarp();
#pragma unroll 1
      for (int hq = 0; hq < C::NQP; ++hq) {
        mbar_wait(dq_full, (it * C::NQP + hq) & 1);
        if (tq) qtrace(p, it, 12);
        tc_fence_after();
        uint32_t o[C::QN / 16][16];
#pragma unroll
        for (int hh = 0; hh < C::QN / 16; ++hh) {
          tmem_ld16(lane_addr + C::Q_COL + 16 * hh, o[hh]);
#pragma unroll
          for (int a = 1; a < C::QACC; ++a) {
            uint32_t oa[16];
            tmem_ld16(lane_addr + C::Q_COL + a * C::QN + 16 * hh, oa);
            tc_wait_ld();
#pragma unroll
            for (int z = 0; z < 16; ++z) o[hh][z] = __float_as_uint(__uint_as_float(o[hh][z]) + __uint_as_float(oa[z]));
          }
        }
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dq_free);
        if (tq) qtrace(p, it, 13);
#pragma unroll
        for (int hh = 0; hh < C::QN / 16; ++hh)
#pragma unroll
          for (int z2 = 0; z2 < 2; ++z2) {
            const int z = (hq * C::QN) / 8 + 2 * hh + z2;
            const int zs = kRB == 32 ? (z ^ ((R >> 2) & 1)) : kRB == 64 ? (z ^ ((R >> 1) & 3)) : (z ^ (R & 7));
            const uint32_t *v = o[hh] + 8 * z2;
            *(uint4 *)(orow + 16 * zs) = make_uint4(
                pack_el<F16>(__uint_as_float(v[0]) * p.scale, __uint_as_float(v[1]) * p.scale),
                pack_el<F16>(__uint_as_float(v[2]) * p.scale, __uint_as_float(v[3]) * p.scale),
                pack_el<F16>(__uint_as_float(v[4]) * p.scale, __uint_as_float(v[5]) * p.scale),
                pack_el<F16>(__uint_as_float(v[6]) * p.scale, __uint_as_float(v[7]) * p.scale));
          }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {  // queries past the map / band edge are clipped by the TMA unit
        const int oc = pair ? 4 * (quarter & 1) : j0 + 4 * quarter;
        tma_store_4d(&tm_dq, ostage, 0, oc, i0 - p.q_row0, bhq);
        tma_store_4d(&tm_dq, ostage + C::HALF_B, 0, oc, i0 - p.q_row0 + 4, bhq);
        bulk_commit();
      }
      if (tq) qtrace(p, it, 14);
    }
    if (threadIdx.x == 64 + 64) qtrace_gt(p, 17);
    if (gtid == 0) qtrace_gt(p, 22);
    if (p.rpb) {
      if (cur_key >= 0) flush();
      commit_head(cur_head);
    }
    if (gtid == 0) qtrace_gt(p, 23);
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (threadIdx.x == 0) qtrace_gt(p, 18);
  if (warp == kProducerWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
#ifdef NA2D_TRACE
    if (lane == 0 && p.trace) {
      uint64_t gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.trace[16896 + 2 * blockIdx.x + 1] = (long long)gt;
    }
#endif
  }
}

template <int L, int HD, bool F16>
cudaError_t launch_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const void *out,
                      const float *lse, const void *dout, void *dq, float *drpb, float *D, float *part,
                      int *b2_tile_counter, cudaStream_t st) {
  using C = CfgQ<L, HD>;
  const cudaError_t attr_err = tc::ensure_smem_attr((const void *)na2d_bwd_dq_kernel<L, HD, F16>, C::SMEM);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tdo, tk, tv, tdq;
  const int BH = g.B * g.heads;
  const bool pair = pair_mode(g.B, g.H, g.W, g.q_row0, g.q_rows, g.kv_row0, g.kv_rows);
  if (!make_tmap_e16_4d(F16, &tq, q, HD, g.W, g.q_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tdo, dout, HD, g.W, g.q_rows, BH, 4, 4) ||
      !(pair ? make_tmap_e16_pair(F16, &tk, k, HD, g.W, g.kv_rows, g.heads, BH, kHCP / 2, C::HR)
             : make_tmap_e16_4d(F16, &tk, k, HD, g.W, g.kv_rows, BH, kHCP, C::HR)) ||
      !(pair ? make_tmap_e16_pair(F16, &tv, v, HD, g.W, g.kv_rows, g.heads, BH, kHCP / 2, C::HR)
             : make_tmap_e16_4d(F16, &tv, v, HD, g.W, g.kv_rows, BH, kHCP, C::HR)) ||
      !make_tmap_e16_4d(F16, &tdq, dq, HD, g.W, g.q_rows, BH, 4, 4))
    return cudaErrorInvalidValue;
  BwdQParams p;
  p.heads = g.heads;
  p.H = g.H;
  p.W = g.W;
  p.q_rows = g.q_rows;
  p.q_row0 = g.q_row0;
  p.kv_row0 = g.kv_row0;
  p.order = make_tile_order(g, L);
  p.num_tiles = p.order.num_tiles;
  p.scale = g.scale;
  p.rpb = rpb;
  p.lse = lse;
  p.out = (const __nv_bfloat16 *)out;
  p.dout = (const __nv_bfloat16 *)dout;
  p.dq = (__nv_bfloat16 *)dq;
  p.D = D;
  p.drpb_part = rpb ? part : nullptr;
  p.b2_tile_counter = b2_tile_counter;
  p.trace = (long long *)debug_trace_buffer();
  const int grid = dq_grid(g);
  make_b1_ranges(p.order, g, grid, &p.ranges);
  (void)drpb;  // summed from the partial tables by B2
  {
    ProfScope ps("na2d_bwd_dq_tc", st);
    const cudaError_t e = launch_pdl(na2d_bwd_dq_kernel<L, HD, F16>, grid, kThreads, C::SMEM, st, tq, tdo, tk, tv, tdq, p);
    if (e != cudaSuccess) return e;
  }
  // the per-CTA dRPB partial tables are summed by the dK/dV kernel (B2), which runs next
  return cudaGetLastError();
}

}  // namespace

int dq_grid(const Geo &g) {
  const TileOrder o = make_tile_order(g, g.L);
  const int grid = o.num_tiles < tc::num_sms() ? o.num_tiles : tc::num_sms();
  return grid < kMaxB1Ctas ? grid : kMaxB1Ctas;
}

namespace {
template <int D, bool F16>
cudaError_t dq_for_d(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const void *out,
                     const float *lse, const void *dout, void *dq, float *drpb, float *D_, float *part,
                     int *b2_tile_counter, cudaStream_t st) {
  switch (g.L) {
    case 3: return launch_dq<3, D, F16>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D_, part, b2_tile_counter, st);
    case 5: return launch_dq<5, D, F16>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D_, part, b2_tile_counter, st);
    case 7: return launch_dq<7, D, F16>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D_, part, b2_tile_counter, st);
  }
  return cudaErrorInvalidValue;
}
template <bool F16>
cudaError_t dq_for_el(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const void *out,
                      const float *lse, const void *dout, void *dq, float *drpb, float *D_, float *part,
                      int *b2_tile_counter, cudaStream_t st) {
  switch (g.d) {
    case 16: return dq_for_d<16, F16>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D_, part, b2_tile_counter, st);
    case 32: return dq_for_d<32, F16>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D_, part, b2_tile_counter, st);
    case 64: return dq_for_d<64, F16>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D_, part, b2_tile_counter, st);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t tc_backward_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                           const void *out, const float *lse, const void *dout, void *dq, float *drpb, float *D,
                           float *part, int *b2_tile_counter, cudaStream_t st) {
  return g.dtype == NA2D_F16 ? dq_for_el<true>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st)
                             : dq_for_el<false>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st);
}

}  // namespace na2d
