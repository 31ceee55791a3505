// na2d_bwd_dq_tc.cu -- backward kernel B1 (query-centric) on tcgen05/TMEM/TMA, sm_100a:
// steps a6, a7, a9, a10 of the analytic gradient of Eq. 2 (R5):
//   P     = exp2(s*scale*log2e + B' - LSE_q*log2e)      (recomputed; B' masked pre-scaled bias)
//   dP    = dO_q . v_k                                  (tcgen05, TMEM)
//   D_q   = dO_q . O_q = sum_k P dP  (exact fp32 from the recomputed P, dP; written for B2)
//   dS    = P (dP - D_q)
//   dQ_q  = scale * sum_k dS k_k                        (tcgen05 TS MMA, dS 16-bit from TMEM)
//   dB    = scale * sum dS over (b, q, k) per relative-position cell
// Geometry is the forward's: 8 x 16 query tiles = two M=64 sub-tiles (rows 0-3 / 4-7, TMEM lanes
// 0-15 / 16-31 of every lane quarter), halo of 8+L-1 rows x 24 keys; TMEM lane quarter q owns the
// 4 x 4 query blocks at columns [4q, 4q+4) of both sub-tiles, whose windows lie in a union of
// (4+L-1) rows x (L+5) even-aligned columns relative to each sub-tile's own halo base rb_s.
//
// Chunk pipeline.  D needs the whole window before any dS, so the elementwise work is two passes.
// The union rows are split into PAIRS = (L+3)/2 chunks of two halo rows (N = 48 keys per sub-tile).
// Per chunk c the tensor core computes
//   S_c, dP_c   (SS, into one of two rotating 96-column slots)   -> pass 1: P (fp16, kept in a
//               TMEM "P region", PAIRS x 24 columns) and the partial D;
//   dP_c again  (SS, into one of two rotating 48-column slots)   -> pass 2 (after D): dS = P (dP - D)
//               written over P, dRPB accumulated;
//   dQ += dS_c K_c (TS, three accumulation chains, one per K-step of the chunk).
// Recomputing dP instead of keeping the fp32 dP of the whole tile (or S and dP as fp32, 2 x 224
// columns) keeps the tile's TMEM footprint at P region + slots + dQ (504 of 512 columns at L = 7),
// so S / dP of the next chunks stream while the elementwise warps work and the dQ MMAs of a chunk
// follow as soon as its dS lands; no stage waits for a whole tile.  P is kept for pass 2 as fp16
// (P in [0, 1]; relative rounding <= 2^-12, a quarter of dS's own bf16 rounding for the dQ MMA).
// Union row pairs are bound to elementwise groups (group g owns chunks [pr0(g), pr0(g+1))), so each
// lane's dRPB accumulator covers fixed union rows: tiles are visited grouped by geometry class
// (interior tile rows/columns form one class, each border tile row/column its own) and head; within
// a class each lane's union element -> bias cell map is fixed, so dS is accumulated in union
// coordinates in registers and flushed (masked to the lane's window) into per-(warp, half)
// shared tables only when the class or head changes; per-CTA tables are summed in fixed CTA order
// by B2's prologue.
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

constexpr int kStages = 2;
constexpr int kGroups = 3;                    // elementwise warp groups (each covers the 4 TMEM lane quarters)
constexpr int kThreads = (4 * kGroups + 4) * 32;  // elementwise warps, then TMA, S/dP, dP (pass 2), dQ issuers
// (the sub-partition scheduler favours the highest warp id: the producer / MMA warps never wait for
// the elementwise warps sharing their sub-partitions)
constexpr int kProducerWarp = 4 * kGroups, kMmaWarpA = 4 * kGroups + 1, kMmaWarpB = 4 * kGroups + 2,
              kMmaWarpC = 4 * kGroups + 3;
constexpr int kChunkN = 2 * kHCP;             // keys per chunk and sub-tile (two halo rows)

// Per-stage tile description, written by the producer before it arms full[stage] (the class-grouped
// order's decode and the window origins, computed once instead of in every warp).
struct TileInfoQ {
  int bh, i0, j0, cls, hr0, hc0;
  int rb[2];  // first union row of sub-tile / half h (relative to hr0)
  int uc[4];  // even first union column of lane quarter q (relative to hc0)
};

template <int L>
struct CfgQ {
  static constexpr int HR = kTQH + L - 1;
  static constexpr int UR = 4 + L - 1;
  static constexpr int UCW = L + 5;
  static constexpr int PAIRS = UR / 2;                         // chunks per tile
  static constexpr int PA = (PAIRS + kGroups - 1) / kGroups;   // max chunks of a group
  __host__ __device__ static constexpr int pr0(int g) { return g * PAIRS / kGroups; }
  static_assert(UR % 2 == 0 && PAIRS >= kGroups, "every group owns at least one chunk");
  // TMEM columns
  static constexpr int S1_COL = 0;                   // two pass-1 slots: S [x*96, +48), dP [x*96+48, +48)
  static constexpr int S2_COL = 4 * kChunkN;         // two pass-2 slots: dP [S2_COL + x*48, +48)
  static constexpr int P_COL = S2_COL + 2 * kChunkN; // P / dS (16-bit pairs): chunk c at P_COL + 24c
  static constexpr int QACC = 3;                     // dQ chains (one per K-step of a chunk)
  static constexpr int Q_COL = 512 - QACC * kD;
  static_assert(P_COL + PAIRS * (kChunkN / 2) <= Q_COL, "TMEM budget");
  static constexpr int KV_ROWS = HR * kHCP;
  static constexpr int Q_BYTES = 128 * kRowBytes;
  static constexpr int KV_BYTES = KV_ROWS * kRowBytes;
  static constexpr int TX_BYTES = 2 * Q_BYTES + 2 * KV_BYTES;     // Q, dO, K, V by TMA
  static constexpr int LSE_OFF = TX_BYTES;                          // + the tile's 128 LSE (log2)
  static constexpr int STAGE_BYTES = TX_BYTES + 1024;
  static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1 KB aligned (swizzled TMA / UMMA)");
  static constexpr int TT = 2 * L - 1;
  static constexpr int TBL_OFF = kStages * STAGE_BYTES;
  static constexpr int OUT_OFF = (TBL_OFF + BiasTable<L>::FLOATS * 4 + 1023) / 1024 * 1024;  // dQ staging
  static constexpr int DB_OFF = OUT_OFF + 4 * 2048;
  static constexpr int DP_OFF = DB_OFF + ((8 * kGroups * TT * TT * 4 + 255) / 256) * 256;  // partial D [2][groups][128]
  static constexpr int TI_OFF = DP_OFF + 2 * kGroups * 128 * 4;
  static constexpr int BAR_OFF = TI_OFF + kStages * 64;
  static_assert(sizeof(TileInfoQ) <= 64, "TileInfoQ");
  static constexpr int NBARS = 2 * kStages + 4 + 4 * PAIRS + 2;
  static constexpr int SMEM = BAR_OFF + NBARS * 8 + 16 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

__device__ __forceinline__ TileOrder::Tile decode(const BwdQParams &p, int t) { return p.order.decode(t); }

#ifdef NA2D_TRACE
// debug timeline (CTA 0): trace[(warp * 64 + tile) * 16 + ev] = clock64()
#define TR(tile, ev)                                                                                \
  do {                                                                                              \
    if (p.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (tile) < 64)                       \
      p.trace[32768 + ((threadIdx.x / 32) * 64 + (tile)) * 16 + (ev)] = clock64();                        \
  } while (0)
#else
#define TR(tile, ev)
#endif
#ifdef NA2D_DEBUG_HANG
// development aid: every wait publishes (tag, parity) of the calling warp to the trace buffer (host
// memory mapped into the device) before spinning, so a host watchdog can see where a hang sits
#define DBG_MARK(tag, ph)                                                                           \
  do {                                                                                               \
    if (p.trace && (threadIdx.x & 31) == 0)                                                          \
      *(volatile long long *)&p.trace[blockIdx.x * 16 + threadIdx.x / 32] =                          \
          ((long long)(tag) << 40) | ((long long)(ph) << 32) | (unsigned)dbg_it;                      \
  } while (0)
#define MBAR_WAIT(b, ph, tag)                                                                       \
  do {                                                                                               \
    DBG_MARK(tag, ph);                                                                               \
    mbar_wait(b, ph);                                                                                \
    DBG_MARK((tag) + 100, ph);                                                                       \
  } while (0)
#else
#define MBAR_WAIT(b, ph, tag) mbar_wait(b, ph)
#define DBG_MARK(tag, ph)
#endif

template <int L, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const __grid_constant__ CUtensorMap tm_dq, const BwdQParams p) {
  using C = CfgQ<L>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float *tbl = (float *)(smem + C::TBL_OFF);
  float *s_db = (float *)(smem + C::DB_OFF);  // private dRPB tables: (elementwise warp, half)
  TileInfoQ *tinfo = (TileInfoQ *)(smem + C::TI_OFF);
  uint64_t *bars = (uint64_t *)(smem + C::BAR_OFF);
  uint64_t *full = bars, *empty = bars + kStages;          // TMA stages
  // Slot barriers: *_free per rotating TMEM slot (the issuer waits for the slot's previous chunk), *_full
  // per chunk index (one completion per tile).  A group consumes only its own chunks, so it may reach
  // its next chunk two slot uses ahead of a lagging issuer: a per-slot full barrier would then be two
  // phases behind and its parity test would pass on the stale phase.
  uint64_t *p1_free = bars + 2 * kStages, *p2_free = p1_free + 2;  // pass-1 slots (S, dP), pass-2 slots (dP)
  uint64_t *p1_full = p1_free + 4;                         // [PAIRS] S / dP of chunk c in its slot
  uint64_t *p2_full = p1_full + C::PAIRS;                  // [PAIRS] dP (pass 2) of chunk c in its slot
  uint64_t *pfree = p2_full + C::PAIRS;                    // [PAIRS] P region chunk c read by dQ(c)
  uint64_t *ds_full = pfree + C::PAIRS;                    // [PAIRS] dS of chunk c written
  uint64_t *dq_full = ds_full + C::PAIRS, *dq_free = dq_full + 1;
  uint32_t *tmem_slot = (uint32_t *)(bars + C::NBARS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int dbg_it = 0;  // (NA2D_DEBUG_HANG) progress counter published with each wait
  (void)dbg_it;
  const int t_begin = (int)((long)p.num_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long)p.num_tiles * (blockIdx.x + 1) / gridDim.x);
  const int n_tiles = t_end - t_begin;
  const int q_end = p.q_row0 + p.q_rows;

  if (warp == kProducerWarp && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1 + 32);  // expect_tx arrive + 32 lanes staging the tile's LSE
      mbar_init(&empty[s], 3);      // the three issuers' last MMAs reading the stage
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&p1_free[x], 4);  // the owning group's four quarter warps have loaded the slot
      mbar_init(&p2_free[x], 4);
    }
    for (int c = 0; c < C::PAIRS; ++c) {
      mbar_init(&p1_full[c], 1);
      mbar_init(&p2_full[c], 1);
      mbar_init(&pfree[c], 1);
      mbar_init(&ds_full[c], 4);
    }
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // the previous kernel (forward / last step's B2) is complete: global memory from here on
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
      mbar_wait_sleep(&empty[s], ((it / kStages) & 1) ^ 1, 1024);
      TR(it, 0);
      const TileOrder::Tile g = decode(p, t);
      const int hr0 = wstart(g.i0, p.H, L), hc0 = wstart(g.j0, p.W, L);
      uint8_t *st = smem + s * C::STAGE_BYTES;
      TileInfoQ *ti = tinfo + s;
      if (lane < 2) ti->rb[lane] = wstart(min(g.i0 + 4 * lane, q_end - 1), p.H, L) - hr0;
      if (lane < 4) ti->uc[lane] = (wstart(min(g.j0 + 4 * lane, p.W - 1), p.W, L) - hc0) & ~1;
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
            const int r0 = (64 * sb + 16 * qb) * kRowBytes;
            tma_load_4d(st + r0, &tm_q, &full[s], 0, g.j0 + 4 * qb, g.i0 - p.q_row0 + 4 * sb, g.bh);
            tma_load_4d(st + C::Q_BYTES + r0, &tm_do, &full[s], 0, g.j0 + 4 * qb, g.i0 - p.q_row0 + 4 * sb, g.bh);
          }
        tma_load_4d(st + 2 * C::Q_BYTES, &tm_k, &full[s], 0, hc0, hr0 - p.kv_row0, g.bh);
        tma_load_4d(st + 2 * C::Q_BYTES + C::KV_BYTES, &tm_v, &full[s], 0, hc0, hr0 - p.kv_row0, g.bh);
      }
      __syncwarp();
      // LSE of query (half, quarter, r, c) at e = half*64 + quarter*16 + r*4 + c; 0 if outside
      float *lse_s = (float *)(st + C::LSE_OFF);
      float lv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = lane + 32 * u;
        const int i = g.i0 + 4 * (e >> 6) + ((e >> 2) & 3), j = g.j0 + 4 * ((e >> 4) & 3) + (e & 3);
        lv[u] = (i < q_end && j < p.W)
                    ? __ldg(&p.lse[((size_t)g.bh * p.q_rows + (i - p.q_row0)) * p.W + j]) * 1.4426950408889634f
                    : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) lse_s[lane + 32 * u] = lv[u];
      mbar_arrive(&full[s]);
    }
  } else if (warp == kMmaWarpA) {
    // ================= S / dP issuer (pass 1): chunk n = it*PAIRS + c into pass-1 slot n & 1 once the
    // group that loaded that slot's previous chunk (n - 2) has released it
    constexpr uint32_t idesc_s = idesc_el<F16>(64, kChunkN, false);
    for (int it = 0; it < n_tiles; ++it) {
      const int s = it % kStages;
      dbg_it = it;
      MBAR_WAIT(&full[s], (it / kStages) & 1, 1);
      const int rb0 = tinfo[s].rb[0], rb1 = tinfo[s].rb[1];
      const uint64_t dqs = sdesc_sw64(smem_u32(smem + s * C::STAGE_BYTES));
      const uint64_t dk0 = dqs + ((2 * C::Q_BYTES + rb0 * kHCP * kRowBytes) >> 4);
      const uint64_t dk1 = dqs + ((2 * C::Q_BYTES + rb1 * kHCP * kRowBytes) >> 4);
      constexpr uint32_t vo = C::KV_BYTES >> 4, doo = C::Q_BYTES >> 4;
#pragma unroll 1
      for (int c = 0; c < C::PAIRS; ++c) {
        const int n = it * C::PAIRS + c, x = n & 1;
        MBAR_WAIT(&p1_free[x], ((n >> 1) & 1) ^ 1, 2);
        TR(it, c);
        tc_fence_after();
        const uint32_t co = (c * kChunkN * kRowBytes) >> 4;  // the chunk's first key in the halos
        const uint32_t d0 = tmem + C::S1_COL + x * 2 * kChunkN, d1 = d0 + ((uint32_t)16 << 16);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t ko = (k * 32) >> 4;
            mma_ss(d0, dqs + ko, dk0 + co + ko, idesc_s, k);
            mma_ss(d1, dqs + (4096 >> 4) + ko, dk1 + co + ko, idesc_s, k);
            mma_ss(d0 + kChunkN, dqs + doo + ko, dk0 + vo + co + ko, idesc_s, k);
            mma_ss(d1 + kChunkN, dqs + doo + (4096 >> 4) + ko, dk1 + vo + co + ko, idesc_s, k);
          }
          mma_commit(&p1_full[c]);
          if (c == C::PAIRS - 1) mma_commit(&empty[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarpB) {
    // ================= dP issuer (pass 2): chunk n into pass-2 slot n & 1 as soon as pass 2 of chunk n - 2
    // has loaded that slot (dP does not depend on D: it runs ahead of the elementwise passes)
    constexpr uint32_t idesc_s = idesc_el<F16>(64, kChunkN, false);
    const int total = n_tiles * C::PAIRS;
#pragma unroll 1
    for (int n = 0; n < total; ++n) {
      const int it = n / C::PAIRS, c = n - it * C::PAIRS, s = it % kStages, x = n & 1;
      dbg_it = n;
      if (c == 0) MBAR_WAIT(&full[s], (it / kStages) & 1, 3);
      MBAR_WAIT(&p2_free[x], ((n >> 1) & 1) ^ 1, 4);
      TR(it, c);
      tc_fence_after();
      const int rb0 = tinfo[s].rb[0], rb1 = tinfo[s].rb[1];
      const uint64_t dqs = sdesc_sw64(smem_u32(smem + s * C::STAGE_BYTES));
      const uint64_t dv0 = dqs + ((2 * C::Q_BYTES + C::KV_BYTES + (rb0 * kHCP + c * kChunkN) * kRowBytes) >> 4);
      const uint64_t dv1 = dqs + ((2 * C::Q_BYTES + C::KV_BYTES + (rb1 * kHCP + c * kChunkN) * kRowBytes) >> 4);
      constexpr uint32_t doo = C::Q_BYTES >> 4;
      const uint32_t d0 = tmem + C::S2_COL + x * kChunkN, d1 = d0 + ((uint32_t)16 << 16);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t ko = (k * 32) >> 4;
          mma_ss(d0, dqs + doo + ko, dv0 + ko, idesc_s, k);
          mma_ss(d1, dqs + doo + (4096 >> 4) + ko, dv1 + ko, idesc_s, k);
        }
        mma_commit(&p2_full[c]);
        if (c == C::PAIRS - 1) mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarpC) {
    // ================= dQ issuer: dQ += dS_c K_c once chunk c's dS is in TMEM (three chains: K-step ks of
    // every chunk accumulates into chain ks)
    constexpr uint32_t idesc_q = idesc_el<F16>(64, kD, true);
    const int total = n_tiles * C::PAIRS;
#pragma unroll 1
    for (int n = 0; n < total; ++n) {
      const int it = n / C::PAIRS, c = n - it * C::PAIRS, s = it % kStages;
      dbg_it = n;
      MBAR_WAIT(&ds_full[c], it & 1, 5);
      if (c == 0) MBAR_WAIT(dq_free, (it & 1) ^ 1, 6);  // the epilogue of tile it - 1 has read dQ
      TR(it, c);
      tc_fence_after();
      const int rb0 = tinfo[s].rb[0], rb1 = tinfo[s].rb[1];
      const uint64_t dk0 = sdesc_sw64(smem_u32(smem + s * C::STAGE_BYTES) + 2 * C::Q_BYTES +
                                      (rb0 * kHCP + c * kChunkN) * kRowBytes);
      const uint64_t dk1 = dk0 + (((rb1 - rb0) * kHCP * kRowBytes) >> 4);
      const uint32_t t0 = tmem, t1 = tmem + ((uint32_t)16 << 16);
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < kChunkN / 16; ++ks) {
          const uint32_t ko = (ks * 16 * kRowBytes) >> 4;
          const uint32_t ao = C::P_COL + c * (kChunkN / 2) + ks * 8, qo = C::Q_COL + ks * kD;
          mma_ts(t0 + qo, t0 + ao, dk0 + ko, idesc_q, c > 0 ? 1u : 0u);
          mma_ts(t1 + qo, t1 + ao, dk1 + ko, idesc_q, c > 0 ? 1u : 0u);
        }
        mma_commit(&pfree[c]);
        if (c == C::PAIRS - 1) {
          mma_commit(dq_full);
          mma_commit(&empty[s]);
        }
      }
      __syncwarp();
    }
  } else {
    // ================= elementwise (warps 0.. -> TMEM lane quarter warp % 4): group grp owns chunks
    // [pr0, pr1) of every tile; group 0 also runs the dQ epilogue (deferred by one tile)
    const int quarter = warp & 3, grp = warp >> 2;
    const int pr0 = C::pr0(grp), pr1 = C::pr0(grp + 1);
    const int half = lane >> 4, r = (lane >> 2) & 3, c = lane & 3;
    const int gtid = threadIdx.x;
    float *s_dpart = (float *)(smem + C::DP_OFF);
    const int Lh = wlen(p.H, L), Lw = wlen(p.W, L);
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = p.scale * 1.4426950408889634f;
    const float2 sl2x2 = make_float2(sl2, sl2);
    // this (warp, half)'s private dRPB table: within one instruction the 16 lanes of a half touch
    // distinct cells (no intra-instruction address conflicts, no other warp contending), but
    // different (u, z) of different lanes do meet, so the adds stay atomic (RED to shared)
    float *my_db = s_db + ((grp * 4 + quarter) * 2 + half) * C::TT * C::TT;
    constexpr int kEw = kGroups * 128;  // elementwise threads
    uint8_t *ostage = smem + C::OUT_OFF + quarter * 2048;
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
    auto commit_head = [&](int head) {  // sum of the private tables -> partials[cta][head]; clear
      named_bar_sync(1, kEw);
      if (head >= 0 && p.drpb_part)
        for (int e = gtid; e < C::TT * C::TT; e += kEw) {
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < 8 * kGroups; ++w) {
            v += s_db[w * C::TT * C::TT + e];
            s_db[w * C::TT * C::TT + e] = 0.f;
          }
          float *dst = &p.drpb_part[((size_t)blockIdx.x * p.heads + head) * C::TT * C::TT + e];
          *dst += p.scale * v;
        }
      named_bar_sync(1, kEw);
    };
    // ---- dQ epilogue of tile eit (group 0): dQ = scale * sum of the chains -> 16-bit, TMA stores
    auto epilogue = [&](int eit, int bh, int i0, int j0) {
      MBAR_WAIT(dq_full, eit & 1, 7);
      tc_fence_after();
      // chains summed, scaled, packed into the SW64 staging row of query (r, c) of block `half`
      // (row R of the 1 KB box; 16-byte chunk z at z ^ (R/2 % 4)), 8 columns at a time
      const int R = r * 4 + c;
      uint8_t *orow = ostage + half * 1024 + R * 64;
      if (lane == 0) bulk_wait_read0();  // this warp's previous store has left the staging
      __syncwarp();
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        uint32_t o[C::QACC][8];
#pragma unroll
        for (int a = 0; a < C::QACC; ++a) tmem_ld8(lane_addr + C::Q_COL + a * kD + 8 * z, o[a]);
        tc_wait_ld();
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float acc_ = __uint_as_float(o[0][e]);
#pragma unroll
          for (int a = 1; a < C::QACC; ++a) acc_ += __uint_as_float(o[a][e]);
          v[e] = acc_ * p.scale;
        }
        *(uint4 *)(orow + 16 * ((z ^ (R >> 1)) & 3)) =
            make_uint4(pack_el<F16>(v[0], v[1]), pack_el<F16>(v[2], v[3]), pack_el<F16>(v[4], v[5]), pack_el<F16>(v[6], v[7]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {  // queries past the map / band edge are clipped by the TMA unit
        tma_store_4d(&tm_dq, ostage, 0, j0 + 4 * quarter, i0 - p.q_row0, bh);
        tma_store_4d(&tm_dq, ostage + 1024, 0, j0 + 4 * quarter, i0 - p.q_row0 + 4, bh);
        bulk_commit();
      }
    };
    int pend_it = -1, pend_bh = 0, pend_i0 = 0, pend_j0 = 0;  // deferred epilogue (group 0)
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      const int stage = it % kStages;
      dbg_it = it;
      MBAR_WAIT(&full[stage], (it / kStages) & 1, 8);  // tile description and LSE staged
      TR(it, 0);
      // copied to registers: the producer refills this stage once the tile's MMAs complete
      const TileInfoQ &ti = tinfo[stage];
      const int bh = ti.bh, i0 = ti.i0, j0 = ti.j0, hr0 = ti.hr0, hc0 = ti.hc0;
      const int rb = ti.rb[half], uc = ti.uc[quarter];
      const int h = bh % p.heads;
      const int key = ti.cls * p.heads + h;
      const int i = i0 + 4 * half + r, j = j0 + 4 * quarter + c;
      const int ic = min(i, q_end - 1), jc = min(j, p.W - 1);
      const int si = wstart(ic, p.H, L), sj = wstart(jc, p.W, L);
      const int dc = sj - jc + L - 1;
      const int brow0 = hr0 + rb - ic + L - 1, bcol0 = hc0 + uc - jc + L - 1;
      const float nlse2 = -((const float *)(smem + stage * C::STAGE_BYTES + C::LSE_OFF))[half * 64 + quarter * 16 + r * 4 + c];
      if (key != cur_key) {
        if (p.rpb && cur_key >= 0) flush();
        if (h != cur_head) {
          if (p.rpb) commit_head(cur_head);
          named_bar_sync(1, kEw);
          BiasTable<L>::build_elems(tbl, p.rpb, h, Lw, sl2, gtid, kEw);  // (measured fastest here)
          named_bar_sync(1, kEw);
          cur_head = h;
        }
        cur_key = key;
        f_valid = i < q_end && j < p.W;
        f_wr = si - hr0 - rb;
        f_wc = sj - hc0 - uc;
        f_brow = brow0;
        f_bcol = bcol0;
      }
      const bool qvalid = i < q_end && j < p.W;
      const size_t qi = ((size_t)bh * p.q_rows + (ic - p.q_row0)) * p.W + jc;
      const float *tcls = tbl + dc * BiasTable<L>::TROWS * kTblStride + kTblOff + bcol0;
      const float2 nlse2x2 = make_float2(nlse2, nlse2);
      const int zb = uc >> 1;
      // ---- pass 1 over the group's chunks: P = exp2(s*scale*log2e + B' - LSE*log2e) -> 16-bit pairs in
      // the P region, D = dO.O = sum_window P dP (exact in fp32: O = sum P V, so dO.O = sum P (dO.v))
      float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int lc = 0; lc < C::PA; ++lc) {
        const int ch = pr0 + lc;
        if (ch >= pr1) break;
        const int n = it * C::PAIRS + ch, x = n & 1;
        const int u = 2 * ch;  // union row of the chunk's first row
        MBAR_WAIT(&p1_full[ch], it & 1, 9);
        TR(it, 1 + lc);
        tc_fence_after();
        const uint32_t ca = lane_addr + C::S1_COL + x * 2 * kChunkN + uc;
        const int pr = hr0 + rb + u;
        // the chunk's two rows one at a time (register budget: 128 per thread at 15 warps)
        uint32_t pk[2][C::UCW / 2];
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          uint32_t sv[C::UCW], dv[C::UCW];
          ld_row<C::UCW>(ca + y * kHCP, sv);
          ld_row<C::UCW>(ca + kChunkN + y * kHCP, dv);
          const bool rv = (unsigned)(pr + y - si) < (unsigned)Lh;
          const float *tr = tcls + (rv ? pr + y - ic + L - 1 : C::TT) * kTblStride;
          tc_wait_ld();
          if (y == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p1_free[x]);  // slot loaded: the next S / dP may overwrite it
          }
#pragma unroll
          for (int z = 0; z < C::UCW; z += 2) {
            const float2 tt = make_float2(tr[z], tr[z + 1]);
            const float2 xa = __fadd2_rn(__ffma2_rn(make_float2(__uint_as_float(sv[z]), __uint_as_float(sv[z + 1])),
                                                    sl2x2, tt), nlse2x2);
            const float2 Pa = make_float2(ex2(xa.x), ex2(xa.y));
            d2 = __ffma2_rn(Pa, make_float2(__uint_as_float(dv[z]), __uint_as_float(dv[z + 1])), d2);
            pk[y][z / 2] = pack_f16(Pa.x, Pa.y);  // P kept as fp16 (2^-11) for pass 2
          }
        }
        // the P region chunk is free once dQ of the previous tile's chunk has read its dS
        MBAR_WAIT(&pfree[ch], (it & 1) ^ 1, 10);
        TR(it, 3 + lc);
        tc_fence_after();
        const uint32_t prow = lane_addr + C::P_COL + ch * (kChunkN / 2);
        st_zero12(prow);
        st_zero12(prow + kHCP / 2);
        st_row<C::UCW / 2>(prow + zb, pk[0]);
        st_row<C::UCW / 2>(prow + kHCP / 2 + zb, pk[1]);
      }
      // D over the whole window: the groups' partial sums, added in a fixed order
      float *dpb = s_dpart + (it & 1) * kGroups * 128;
      dpb[grp * 128 + quarter * 32 + lane] = d2.x + d2.y;
      named_bar_sync(2 + quarter, 32 * kGroups);
      float Dq = 0.f;
#pragma unroll
      for (int g2 = 0; g2 < kGroups; ++g2) Dq += dpb[g2 * 128 + quarter * 32 + lane];
      TR(it, 5);
      if (qvalid && grp == 0) p.D[qi] = Dq;
      tc_wait_st();
      // deferred dQ epilogue of the previous tile (group 0): its dQ MMAs have had this tile's pass 1
      // to complete, and this tile's dQ MMAs wait for it (dq_free)
      if (grp == 0 && pend_it >= 0) {
        epilogue(pend_it, pend_bh, pend_i0, pend_j0);
        pend_it = -1;
      }
      TR(it, 6);
      // ---- pass 2: dS = P (dP - D) -> dRPB accumulators (union coordinates) and 16-bit pairs over P
      // (the dQ MMA's A operand)
      const float2 nD = make_float2(-Dq, -Dq);
#pragma unroll
      for (int lc = 0; lc < C::PA; ++lc) {
        const int ch = pr0 + lc;
        if (ch >= pr1) break;
        const int n = it * C::PAIRS + ch, x = n & 1;
        const int ul = 2 * lc;  // local accumulator row
        MBAR_WAIT(&p2_full[ch], it & 1, 11);
        TR(it, 7 + lc);
        tc_fence_after();
        uint32_t qa[C::UCW / 2], qb[C::UCW / 2], pa_[C::UCW], pb_[C::UCW];
        const uint32_t prow = lane_addr + C::P_COL + ch * (kChunkN / 2) + zb;
        const uint32_t da_ = lane_addr + C::S2_COL + x * kChunkN + uc;
        ld_row<C::UCW / 2>(prow, qa);
        ld_row<C::UCW / 2>(prow + kHCP / 2, qb);
        ld_row<C::UCW>(da_, pa_);
        ld_row<C::UCW>(da_ + kHCP, pb_);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p2_free[x]);
        uint32_t da[C::UCW / 2], db[C::UCW / 2];
#pragma unroll
        for (int z = 0; z < C::UCW; z += 2) {
          // fp16 P pairs -> fp32 (exact)
          const float2 Pa = __half22float2(*reinterpret_cast<const __half2 *>(&qa[z / 2]));
          const float2 Pb = __half22float2(*reinterpret_cast<const __half2 *>(&qb[z / 2]));
          const float2 dsa = __fmul2_rn(Pa, __fadd2_rn(make_float2(__uint_as_float(pa_[z]), __uint_as_float(pa_[z + 1])), nD));
          const float2 dsb = __fmul2_rn(Pb, __fadd2_rn(make_float2(__uint_as_float(pb_[z]), __uint_as_float(pb_[z + 1])), nD));
          acc[ul][z / 2] = __fadd2_rn(acc[ul][z / 2], dsa);
          acc[ul + 1][z / 2] = __fadd2_rn(acc[ul + 1][z / 2], dsb);
          da[z / 2] = pack_el<F16>(dsa.x, dsa.y);
          db[z / 2] = pack_el<F16>(dsb.x, dsb.y);
        }
        st_row<C::UCW / 2>(prow, da);
        st_row<C::UCW / 2>(prow + kHCP / 2, db);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[ch]);
        DBG_MARK(50 + ch, n);
        TR(it, 9 + lc);
      }
      if (grp == 0) {
        pend_it = it;
        pend_bh = bh;
        pend_i0 = i0;
        pend_j0 = j0;
      }
    }
    if (grp == 0 && pend_it >= 0) epilogue(pend_it, pend_bh, pend_i0, pend_j0);
    DBG_MARK(60, 0);
    if (p.rpb) {
      if (cur_key >= 0) flush();
      commit_head(cur_head);
    }
    if (lane == 0) bulk_wait0();
    DBG_MARK(61, 0);
  }
  DBG_MARK(62, 0);
  __syncthreads();
  if (warp == kProducerWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int L, bool F16>
cudaError_t launch_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const void *out,
                      const float *lse, const void *dout, void *dq, float *drpb, float *D, float *part,
                      int *b2_tile_counter, cudaStream_t st) {
  using C = CfgQ<L>;
  const cudaError_t attr_err = tc::ensure_smem_attr((const void *)na2d_bwd_dq_kernel<L, F16>, C::SMEM);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tdo, tk, tv, tdq;
  const int BH = g.B * g.heads;
  if (!make_tmap_e16_4d(F16, &tq, q, kD, g.W, g.q_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tdo, dout, kD, g.W, g.q_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tk, k, kD, g.W, g.kv_rows, BH, kHCP, C::HR) ||
      !make_tmap_e16_4d(F16, &tv, v, kD, g.W, g.kv_rows, BH, kHCP, C::HR) ||
      !make_tmap_e16_4d(F16, &tdq, dq, kD, g.W, g.q_rows, BH, 4, 4))
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
  (void)drpb;  // summed from the partial tables by B2
  {
    ProfScope ps("na2d_bwd_dq_tc", st);
    const cudaError_t e = launch_pdl(na2d_bwd_dq_kernel<L, F16>, grid, kThreads, C::SMEM, st, tq, tdo, tk, tv, tdq, p);
    if (e != cudaSuccess) return e;
  }
  // the per-CTA dRPB partial tables are summed by the dK/dV kernel (B2), which runs next
  return cudaGetLastError();
}

}  // namespace

int dq_grid(const Geo &g) {
  const TileOrder o = make_tile_order(g, g.L);
  return o.num_tiles < tc::num_sms() ? o.num_tiles : tc::num_sms();
}

cudaError_t tc_backward_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                           const void *out, const float *lse, const void *dout, void *dq, float *drpb, float *D,
                           float *part, int *b2_tile_counter, cudaStream_t st) {
  const bool f16 = g.dtype == NA2D_F16;
  switch (g.L) {
    case 3: return f16 ? launch_dq<3, true>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st)
                 : launch_dq<3, false>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st);
    case 5: return f16 ? launch_dq<5, true>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st)
                 : launch_dq<5, false>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st);
    case 7: return f16 ? launch_dq<7, true>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st)
                 : launch_dq<7, false>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, b2_tile_counter, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace na2d
