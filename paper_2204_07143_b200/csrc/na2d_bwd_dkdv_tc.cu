// na2d_bwd_dkdv_tc.cu -- backward kernel B2 (key-centric) on tcgen05/TMEM/TMA, sm_100a:
// step a8 of the analytic gradient of Eq. 2 (R5):
//   dV_k = sum_{q : k in rho(q)} P[q,k] dO_q,     dK_k = scale sum_{q : k in rho(q)} dS[q,k] Q_q
// over the inverse neighbourhood of each key (the queries whose clamped window holds it).
//
// A CTA tile is 8 x 16 keys = two M=64 sub-tiles (key rows 0-3 / 4-7); TMEM lane quarter q owns
// the 4 x 4 key blocks at columns [4q, 4q+4) of both.  The queries that see the tile lie in a
// halo of rows [ilo(kr0), ihi(kr0+7)] x cols [jlo(kc0), jhi(kc0+15)] (<= 8+3NS rows, <= 16+3NS
// columns), staged by TMA (Q, dO; row pitch QP) together with their LSE and D values.  Each
// sub-tile's query rows are processed in chunks of CR rows (N = CR*QP = 96 queries):
//   S^T = K_s Q_c^T, dP^T = V_s dO_c^T   (tcgen05 SS, M=64, N=96)      -> TMEM chunk slot
//   elementwise: P = exp2(s*scale*log2e + B' - LSE*log2e), dS = P (dP - D), both bf16 -> TMEM
//   dV_s += P^T dO_c, dK_s += dS^T Q_c     (tcgen05 TS, A from TMEM)    -> TMEM accumulators
// Chunk slots are double-buffered; the MMA warp issues chunk k+1's S/dP before chunk k's dV/dK,
// and two elementwise groups alternate chunks.  B' is the forward's masked bias table indexed by
// the query's column-clamp class; rows outside the query's window use the all -inf row.
#include <math.h>
#include <stdlib.h>

#include <mutex>
#include <type_traits>

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

constexpr int kThreads = 352;  // warps 0-3 / 4-7 elementwise, 8 producer, 9 S^T/dP^T issuer, 10 dV/dK issuer
// (the sub-partition scheduler favours the highest warp id: the producer / MMA warps never wait for
// the elementwise warps sharing their sub-partitions)
constexpr int kProducerWarp = 8, kMmaWarp = 9, kMmaKvWarp = 10;
constexpr int kNCH = 96;       // queries per chunk (N of the S^T / dP^T MMAs)
constexpr int kSlot = 192;     // TMEM columns per chunk slot: S^T [0,96), dP^T [96,192)
constexpr int kACC_COL = 384;  // dV / dK accumulators: buffer b at 384 + 64b (dV), + 32 (dK)
constexpr int kTileInfoBytes = 512;

template <int L, int QP, int D = 32>
struct CfgK {
  static constexpr int ROWB = 2 * D;  // bytes per 16-bit row: one swizzle atom (32 / 64 / 128 B)
  // d = 64: one Q / dO / K / V stage and one dV / dK accumulator buffer (TMEM: two 192-column chunk
  // slots + dV 64 + dK 64), and the epilogue stores dV / dK rows straight to global memory (no
  // staging: the query halos take 129 KB of shared memory per stage)
  static constexpr int NST = D <= 32 ? 2 : 1, NACC = D <= 32 ? 2 : 1;
  static constexpr bool EPI_DIRECT = D > 32;
  static constexpr int NS = (L - 1) / 2;
  static constexpr int CR = kNCH / QP;             // query rows per chunk
  static constexpr int QRH = kTQH + 3 * NS;        // halo rows loaded (max needed)
  static constexpr int QRA = QRH + CR;             // halo rows allocated (tail zero)
  static constexpr int UCW = ((4 + 3 * NS + 1) + 1) / 2 * 2;  // union columns per quarter (even)
  static_assert(UCW <= 16, "union width");
  // interior quarters (every union column of clamp class NS): union of 4 keys' inverse neighbourhoods
  // is 4 + 2NS columns, + 1 for the even origin
  static constexpr int UCWF = ((4 + 2 * NS + 1) + 1) / 2 * 2;
  static constexpr int Q_BYTES = (QRA * QP * ROWB + 1023) / 1024 * 1024;  // 1 KB aligned (swizzle)
  static constexpr int KT_BYTES = 128 * ROWB;
  // LSE and D halo values: pitch LP = QP + 4 so the TMA box can start at a 16-byte aligned column
  static constexpr int LP = QP + 4;
  static constexpr int LD_FLOATS = (QRA * LP + 31) / 32 * 32;  // 128 B aligned
  static constexpr int STAGE_BYTES = (2 * Q_BYTES + 2 * KT_BYTES + 2 * LD_FLOATS * 4 + 1023) / 1024 * 1024;
  static constexpr int TX_BYTES = 2 * QRH * QP * ROWB + 2 * KT_BYTES;
  static_assert(STAGE_BYTES % 1024 == 0 && Q_BYTES % 1024 == 0, "1 KB alignment");
  static constexpr int TT = 2 * L - 1;
  static constexpr int TROWS = TT + 1;
  // the masked table's L column-clamp classes, an all -inf class (index L) and an unmasked class
  // (index L + 1: B[a][b] for every b, the border path masks per column instead)
  static constexpr int TBL_FLOATS = (L + 2) * TROWS * kTblStride;
  static constexpr int TBL_OFF = NST * STAGE_BYTES;
  // dV / dK output staging: 2 groups x 4 warps x 4 KB (SW64 boxes, 1 KB aligned)
  static constexpr int OUT_OFF = (TBL_OFF + TBL_FLOATS * 4 + 1023) / 1024 * 1024;
  static constexpr int OUT_W = EPI_DIRECT ? 0 : 4 * 16 * ROWB;  // per warp: dV, dK x two 4 x 4-key blocks
  static constexpr int TI_OFF = OUT_OFF + 8 * OUT_W;
  static constexpr int BAR_OFF = TI_OFF + NST * kTileInfoBytes;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

struct BwdKParams {
  int B, heads, H, W, q_rows, q_row0, kv_rows, kv_row0;  // B: maps per head (pair mode: map pairs)
  int pair;  // tc::pair_mode: a key tile holds maps (b, h), (b + 1, h); Q / dO halos are pair views
  int tiles_h, tiles_w, num_tiles;
  int shift_cols;  // last two key tile columns start at W-L-16 and W-16 (key_col0)
  int tma_lsd;  // LSE / D halos by TMA (W * 4 bytes 16-byte aligned) instead of lane loads
  int *tile_counter;  // dynamic tile scheduler (zero at launch): CTA b takes tile b, then gridDim + atomicAdd
  float scale;
  const float *rpb, *lse, *D;
  const float *drpb_part;  // B1's per-CTA dRPB tables (null: nothing to reduce)
  int part_ctas;
  float *drpb;
  __nv_bfloat16 *dk, *dv;
  long long *trace;
};
// debug timeline: trace[(cta * 32 + chunk) * 32 + ev] for CTAs < 4 (chunk = CTA-global chunk index)
__device__ __forceinline__ void ktrace(const BwdKParams &p, int c, int ev) {
#ifdef NA2D_TRACE
  if (p.trace && blockIdx.x < 4 && c < 32) p.trace[((size_t)blockIdx.x * 32 + c) * 32 + ev] = clock64();
#endif
}

// first / last query row (column) in [lo, hi) whose clamped window holds key row (column) p.
// Closed form of the inverse neighbourhood: for L < n, wstart(i) + L - 1 >= p  <=>  i >= p - NS
// (when p >= L) and wstart(i) <= p  <=>  i <= p + NS (when p < n - L); else unbounded.
__device__ __forceinline__ int inv_lo(int p, int n, int L, int lo, int hi) {
  const int ns = (L - 1) / 2;
  return (L >= n || p < L) ? lo : max(lo, p - ns);
}
__device__ __forceinline__ int inv_hi(int p, int n, int L, int lo, int hi) {
  const int ns = (L - 1) / 2;
  return (L >= n || p >= n - L) ? hi - 1 : min(hi - 1, p + ns);
}

// Column origin of key tile column tcol.  Normally 16 tcol; for L = 7 and W = 5, 6 mod 16 (>= 37) the
// second-to-last tile would see a 25-column query halo (its last keys reach the right clamp zone),
// so the last two tiles are moved to end at W-L-1 and W-1 (overlapping keys are computed twice,
// identically).  The host (key_tile_cols) checks every tile's halo against the pitch.
__device__ __forceinline__ int key_col0(const BwdKParams &p, int tcol, int L) {
  if (p.shift_cols && tcol >= p.tiles_w - 2) return tcol == p.tiles_w - 1 ? p.W - kTQW : p.W - L - kTQW;
  return tcol * kTQW;
}

// Query rows chunk k of a key tile actually needs, rounded up to even (a row pair is 3 MMA K-steps):
// the last chunk of an interior tile holds 2 of its 4 rows, so its MMAs use N = 48 and its
// elementwise pass stops after one row pair.
template <int CR>
__device__ __forceinline__ int chunk_rows_even(int qs_n0, int qs_n1, int k) {
  const int rows = max(qs_n0, qs_n1) - CR * k;
  return rows >= CR ? CR : max(2, (rows + 1) & ~1);
}

struct KTile {
  int bh, kr0, kc0;   // key tile origin (global row, column)
  int qr0, qc0;       // query halo origin (global)
  int qs_lo[2], qs_n[2];  // per sub-tile: first query row, number of query rows
  int nchunks;
};

template <int L, int QP>
__device__ __forceinline__ KTile ktile(const BwdKParams &p, int t) {
  using C = CfgK<L, QP>;
  KTile g;
  // head-major order: consecutive tiles share the head, so the bias table is rebuilt only when a
  // CTA's next (dynamically scheduled) tile belongs to the other head
  const int per = p.tiles_h * p.tiles_w;
  const int u = t / per, rem = t - u * per;
  const int h = u / p.B;
  g.bh = (p.pair ? 2 : 1) * (u - h * p.B) * p.heads + h;  // (pair mode: member 0)
  g.kr0 = p.kv_row0 + (rem / p.tiles_w) * kTQH;
  g.kc0 = key_col0(p, rem % p.tiles_w, L);
  const int q_end = p.q_row0 + p.q_rows, kv_end = p.kv_row0 + p.kv_rows;
  g.qr0 = inv_lo(min(g.kr0, kv_end - 1), p.H, L, p.q_row0, q_end);
  // even origin: (qc0 & 3) + uc is even, so LSE / D pairs are 8-byte aligned (LDS.64)
  g.qc0 = inv_lo(min(g.kc0, p.W - 1), p.W, L, 0, p.W) & ~1;
  int nmax = 0;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int a = min(g.kr0 + 4 * s, kv_end - 1), b = min(g.kr0 + 4 * s + 3, kv_end - 1);
    g.qs_lo[s] = inv_lo(a, p.H, L, p.q_row0, q_end);
    const int hi = inv_hi(b, p.H, L, p.q_row0, q_end);
    g.qs_n[s] = max(0, hi - g.qs_lo[s] + 1);
    nmax = max(nmax, g.qs_n[s]);
  }
  g.nchunks = max(1, (nmax + C::CR - 1) / C::CR);
  return g;
}

// Elementwise rows of one chunk for one lane (one key): for each chunk row u and union column z
//   P = exp2(s*scale*log2e + B'[row][col] - LSE*log2e),  dS = P (dP - D)  -> bf16 pairs over S / dP.
// FAST: every union column of the quarter is an interior column (column-clamp class NS): the masked
// table of class NS at trow - z (immediate offsets).  Otherwise the unmasked class at trow - z plus a
// per-column mask (0 / -inf: is this lane's key column inside the query column's window), so the
// border path also uses immediate offsets instead of per-column class offsets.
template <int L, int QP, bool FAST, bool F16>
__device__ __forceinline__ void chunk_rows(uint32_t lane_addr, int uc, const float *tbl_row0,
                                           const float2 (&mcol)[CfgK<L, QP>::UCW / 2], const float *lrow0,
                                           int pk, int i_base, int H, int rows_here, int Lh, float sl2,
                                           int rows_even) {
  using C = CfgK<L, QP>;
  constexpr int UW = FAST ? C::UCWF : C::UCW;
  constexpr float log2e = 1.4426950408889634f;
#pragma unroll
  for (int u0 = 0; u0 < C::CR; u0 += 2) {
    if (u0 >= rows_even) break;  // rows past the chunk's (even) row count are never read by the MMAs
    // two chunk rows per step: all four x16 TMEM loads in flight before the wait
    constexpr int NR = 2;
    uint32_t sv[NR][16], dpv[NR][16];
    const float *trow[NR], *lrow[NR];
#pragma unroll
    for (int y = 0; y < NR; ++y) {
      const int u = u0 + y;
      if (u >= C::CR) break;
      const uint32_t ca = lane_addr + u * QP + uc;
      tmem_ld16(ca, sv[y]);
      tmem_ld16(ca + kNCH, dpv[y]);
      // row validity: inside this half's query rows and key row pk in window(i); a = pk - i + L - 1
      const int i = i_base + u;
      const bool rv = u < rows_here && (unsigned)(pk - wstart(i, H, L)) < (unsigned)Lh;
      const int a = pk - i + L - 1;
      trow[y] = tbl_row0 + (rv ? a : C::TT) * kTblStride;
      lrow[y] = lrow0 + u * C::LP;
    }
    tc_wait_ld();
#pragma unroll
    for (int y = 0; y < NR; ++y) {
      const int u = u0 + y;
      if (u >= C::CR) break;
      uint32_t pp[UW / 2], dd[UW / 2];
#pragma unroll
      for (int z = 0; z < UW; z += 2) {
        // one element pair per step in packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2; half the
        // issue slots of scalar code), bf16x2 packs by F2FP (full rate, not on the MUFU pipe)
        const float2 lz = *reinterpret_cast<const float2 *>(lrow[y] + z);
        const float2 dz = *reinterpret_cast<const float2 *>(lrow[y] + C::LD_FLOATS + z);
        const float2 tb = FAST ? make_float2(trow[y][-z], trow[y][-(z + 1)])
                               : __fadd2_rn(make_float2(trow[y][-z], trow[y][-(z + 1)]), mcol[z / 2]);
        const float2 sz = make_float2(__uint_as_float(sv[y][z]), __uint_as_float(sv[y][z + 1]));
        const float2 xv = __ffma2_rn(sz, make_float2(sl2, sl2), tb);
        const float2 ar = __ffma2_rn(lz, make_float2(-log2e, -log2e), xv);
        const float2 P = make_float2(ex2(ar.x), ex2(ar.y));
        const float2 dp = make_float2(__uint_as_float(dpv[y][z]), __uint_as_float(dpv[y][z + 1]));
        const float2 dS = __fmul2_rn(P, __fadd2_rn(dp, make_float2(-dz.x, -dz.y)));
        pp[z / 2] = pack_el<F16>(P.x, P.y);
        dd[z / 2] = pack_el<F16>(dS.x, dS.y);
      }
      const uint32_t prow = lane_addr + u * (QP / 2);
      const uint32_t drow = prow + kNCH;
      st_zero<QP / 2>(prow);
      st_zero<QP / 2>(drow);
      st_row<UW / 2>(prow + uc / 2, pp);
      st_row<UW / 2>(drow + uc / 2, dd);
    }
  }
}

// Per-stage tile description, written by the producer warp before it arms full[stage] (so the MMA
// and elementwise warps only read it): the key tile, its query halo and per lane-quarter union.
struct TileInfo {
  int bh, kr0, kc0, qr0, qc0, nchunks, head, pad;
  int qs_lo[2], qs_n[2];
  int uc[4], fast[4];
};
static_assert(sizeof(TileInfo) <= kTileInfoBytes, "TileInfo size");

template <int L, int QP, int D, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                         const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                         const __grid_constant__ CUtensorMap tm_lse, const __grid_constant__ CUtensorMap tm_d,
                         const __grid_constant__ CUtensorMap tm_dk, const __grid_constant__ CUtensorMap tm_dv,
                         const BwdKParams p) {
  using C = CfgK<L, QP, D>;
  constexpr int kRB = C::ROWB, kStages = C::NST, kNacc = C::NACC;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float *tbl = (float *)(smem + C::TBL_OFF);
  TileInfo *tinfo = (TileInfo *)(smem + C::TI_OFF);
  uint64_t *bars = (uint64_t *)(smem + C::BAR_OFF);
  uint64_t *full = bars, *empty = bars + kStages;
  uint64_t *s_full = bars + 2 * kStages, *ds_full = s_full + 2, *acc_full = s_full + 4, *acc_free = s_full + 6;
  uint64_t *slot_free = s_full + 8;  // chunk slot x: the dV/dK MMAs reading it have completed
  // stage s's MMA operands (K / V blocks, Q / dO halos) and tile description: what the MMA warps
  // wait for; full[s] adds the LSE / D the elementwise warps need, so the MMAs never wait for those
  uint64_t *full_mma = bars + 2 * kStages + 10;
  uint32_t *tmem_slot = (uint32_t *)(full_mma + kStages);

  // broadcast from lane 0 so the compiler treats the warp index (and the TMEM addresses
  // derived from it) as warp-uniform: they stay in uniform registers, no R2UR per tcgen05.ld
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int q_end = p.q_row0 + p.q_rows;

  // zero the never-loaded tail rows of the Q / dO halos (read by partial chunks)
  for (int s = 0; s < kStages; ++s)
    for (int q2 = 0; q2 < 2; ++q2) {
      uint8_t *base = smem + s * C::STAGE_BYTES + q2 * C::Q_BYTES + C::QRH * QP * kRB;
      for (int off = threadIdx.x * 16; off < (C::QRA - C::QRH) * QP * kRB; off += kThreads * 16)
        *(uint4 *)(base + off) = make_uint4(0, 0, 0, 0);
    }
  for (int s = 0; s < kStages; ++s) {  // LSE / D halo rows the TMA box never covers
    float *lsd = (float *)(smem + s * C::STAGE_BYTES + 2 * C::Q_BYTES + 2 * C::KT_BYTES);
    for (int e = C::QRH * C::LP + threadIdx.x; e < C::LD_FLOATS; e += kThreads) {
      lsd[e] = 0.f;
      lsd[C::LD_FLOATS + e] = 0.f;
    }
  }
  fence_proxy_async_smem();
  if (warp == kProducerWarp && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], p.tma_lsd ? 1 : 1 + 32);  // expect_tx arrive (+ 32 lanes staging LSE / D)
      mbar_init(&full_mma[s], 1);
      mbar_init(&empty[s], 1 + 8);                  // MMA commit + the 8 elementwise warps
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&ds_full[s], 4);
      mbar_init(&acc_full[s], 1);  // (buffer 1 unused at d = 64)
      mbar_init(&acc_free[s], 4);
      mbar_init(&slot_free[s], 1);
    }
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    if (p.tma_lsd) {
      tma_prefetch(&tm_lse);
      tma_prefetch(&tm_d);
    }
  }
  if (warp == kProducerWarp) tmem_alloc<512>(tmem_slot);
#ifdef NA2D_TRACE
  if (threadIdx.x == 0 && p.trace) {  // per-CTA wall-clock span (load balance)
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    p.trace[17408 + 2 * blockIdx.x] = (long long)gt;
  }
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // B1 is complete (D, partial tables, zeroed tile counter): global memory from here on
  // a10 final: dRPB = sum of B1's per-CTA partial tables, one warp per cell, lane l summing CTAs
  // l, l + 32, ... in order, then a fixed butterfly (deterministic for a given B1 grid)
  if (p.drpb_part) {
    const int n = p.heads * (2 * L - 1) * (2 * L - 1);
    for (int e = blockIdx.x * (kThreads / 32) + warp; e < n; e += gridDim.x * (kThreads / 32)) {
      float acc = 0.f;
      for (int b = lane; b < p.part_ctas; b += 32) acc += __ldg(&p.drpb_part[(size_t)b * n + e]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.drpb[e] = acc;
    }
  }
  const float log2e = 1.4426950408889634f;

  if (warp == kProducerWarp) {
    // ================= producer: tile description, TMA (K, V sub-tile blocks; Q, dO halos) + LSE / D
    // Tiles are handed out dynamically (the first one per CTA statically): a CTA that runs ahead takes
    // more tiles, so the kernel does not wait for the slowest static share.  After the last tile a
    // description with bh = -1 ends every consumer's loop.
    int it = 0;
    for (int t = blockIdx.x;; ++it) {
      const int s = it % kStages;
      mbar_wait_producer(&empty[s], ((it / kStages) & 1) ^ 1);
      TileInfo *ti = tinfo + s;
      if (t >= p.num_tiles) {  // end of work: sentinel, released like a loaded stage
        if (lane == 0) {
          ti->bh = -1;
          mbar_arrive(&full_mma[s]);
          mbar_arrive(&full[s]);
        }
        if (!p.tma_lsd) {
          __syncwarp();
          mbar_arrive(&full[s]);  // the 32 lane arrivals of the LSE / D staging
        }
        break;
      }
      if (lane == 0) ktrace(p, it, 14);
      const KTile g = ktile<L, QP>(p, t);
      if (lane < 4) {  // union origin of lane quarter q = lane (warp-uniform in the consumers)
        // (pair mode: member lane >> 1's query columns start at halo column (lane >> 1) * QP / 2)
        const int ucr = p.pair ? ((lane >> 1) * (QP / 2) + inv_lo(min(4 * (lane & 1), p.W - 1), p.W, L, 0, p.W)) & ~1
                               : (inv_lo(min(g.kc0 + 4 * lane, p.W - 1), p.W, L, 0, p.W) - g.qc0) & ~1;
        // interior quarters (all union columns of class NS, UCWF wide) take the immediate-offset path
        const bool fast = !p.pair && L < p.W && g.qc0 + ucr >= C::NS && g.qc0 + ucr + C::UCWF - 1 < p.W - C::NS &&
                          ucr + C::UCWF <= QP;
        ti->uc[lane] = fast ? ucr : min(ucr, QP - C::UCW);
        ti->fast[lane] = fast;
      }
      if (lane == 0) {
        ti->bh = g.bh;
        ti->kr0 = g.kr0;
        ti->kc0 = g.kc0;
        ti->qr0 = g.qr0;
        ti->qc0 = g.qc0;
        ti->nchunks = g.nchunks;
        ti->head = g.bh % p.heads;
        ti->qs_lo[0] = g.qs_lo[0];
        ti->qs_lo[1] = g.qs_lo[1];
        ti->qs_n[0] = g.qs_n[0];
        ti->qs_n[1] = g.qs_n[1];
      }
      __syncwarp();
      uint8_t *st = smem + s * C::STAGE_BYTES;
      float *lsd = (float *)(st + 2 * C::Q_BYTES + 2 * C::KT_BYTES);
      if (elect_one()) {
        mbar_expect_tx(&full_mma[s], C::TX_BYTES);
        mbar_expect_tx(&full[s], p.tma_lsd ? 2 * C::QRH * C::LP * 4 : 0);
        uint8_t *kt = st + 2 * C::Q_BYTES;
#pragma unroll
        for (int sb = 0; sb < 2; ++sb)
#pragma unroll
          for (int qb = 0; qb < 4; ++qb) {
            const int r0 = (64 * sb + 16 * qb) * kRB;
            const int kc = p.pair ? 4 * (qb & 1) : g.kc0 + 4 * qb, kbh = p.pair ? g.bh + (qb >> 1) * p.heads : g.bh;
            tma_load_4d(kt + r0, &tm_k, &full_mma[s], 0, kc, g.kr0 - p.kv_row0 + 4 * sb, kbh);
            tma_load_4d(kt + C::KT_BYTES + r0, &tm_v, &full_mma[s], 0, kc, g.kr0 - p.kv_row0 + 4 * sb, kbh);
          }
        if (p.pair) {  // both members' query halos side by side (row pitch QP, member m at m * QP / 2)
          tma_load_5d(st, &tm_q, &full_mma[s], 0, 0, 0, g.qr0 - p.q_row0, g.bh);
          tma_load_5d(st + C::Q_BYTES, &tm_do, &full_mma[s], 0, 0, 0, g.qr0 - p.q_row0, g.bh);
        } else {
          tma_load_4d(st, &tm_q, &full_mma[s], 0, g.qc0, g.qr0 - p.q_row0, g.bh);
          tma_load_4d(st + C::Q_BYTES, &tm_do, &full_mma[s], 0, g.qc0, g.qr0 - p.q_row0, g.bh);
        }
        // LSE / D last: the MMA operands first (B2 127.3 -> 125.6 us at cfg2; the query halos before
        // the key blocks measured 132.3)
        if (p.tma_lsd) {  // box origin column rounded down to a multiple of 4 (16-byte aligned)
          tma_load_3d(lsd, &tm_lse, &full[s], g.qc0 & ~3, g.qr0 - p.q_row0, g.bh);
          tma_load_3d(lsd + C::LD_FLOATS, &tm_d, &full[s], g.qc0 & ~3, g.qr0 - p.q_row0, g.bh);
        }
      }
      __syncwarp();
      if (!p.tma_lsd) {
        // LSE and D of the halo queries by lane loads (W * 4 not 16-byte aligned); 0 outside the
        // band / map (always masked).  All of a lane's loads are issued before its stores.
        constexpr int PER_LANE = (C::QRH * C::LP + 31) / 32;
        float lv[PER_LANE], dv[PER_LANE];
#pragma unroll
        for (int u = 0; u < PER_LANE; ++u) {
          const int e = lane + 32 * u;
          const int i = g.qr0 + e / C::LP;
          int j = (g.qc0 & ~3) + e % C::LP, jbh = g.bh;
          if (p.pair) {  // halo column -> (member, column)
            const int m = j / (QP / 2);
            j -= m * (QP / 2);
            jbh = m < 2 ? g.bh + m * p.heads : -1;
          }
          lv[u] = 0.f;
          dv[u] = 0.f;
          if (e < C::QRH * C::LP && i < q_end && j < p.W && jbh >= 0) {
            const size_t qi = ((size_t)jbh * p.q_rows + (i - p.q_row0)) * p.W + j;
            lv[u] = __ldg(&p.lse[qi]);
            dv[u] = __ldg(&p.D[qi]);
          }
        }
#pragma unroll
        for (int u = 0; u < PER_LANE; ++u) {
          const int e = lane + 32 * u;
          if (e < C::QRH * C::LP) {
            lsd[e] = lv[u];
            lsd[C::LD_FLOATS + e] = dv[u];
          }
        }
        mbar_arrive(&full[s]);
      }
      if (lane == 0) ktrace(p, it, 15);
      int nt = 0;
      if (lane == 0) nt = (int)gridDim.x + atomicAdd(p.tile_counter, 1);
      t = __shfl_sync(0xffffffffu, nt, 0);
    }
  } else if (warp == kMmaWarp) {
    // ================= S^T / dP^T issuer: chunk c into TMEM chunk slot c & 1, once the dV/dK MMAs
    // of chunk c - 2 (which read that slot) have completed.  dV/dK have their own issuing warp, so
    // neither stream waits behind the other's dependencies.
    constexpr uint32_t idesc_s = idesc_el<F16>(64, kNCH, false);
    constexpr uint32_t idesc_s2 = idesc_el<F16>(64, 2 * QP, false);  // a chunk of one row pair
    static_assert(kNCH % QP == 0 && (QP * 2) % 16 == 0, "chunk row pairs are whole K-steps of the dV / dK MMAs");
    int c = 0;
    for (int it = 0;; ++it) {
      const int stage = it % kStages;
      mbar_wait(&full_mma[stage], (it / kStages) & 1);
      if (lane == 0) ktrace(p, c, 3);
      const TileInfo &ti = tinfo[stage];
      if (ti.bh < 0) break;
      const int nch = ti.nchunks, row0a = ti.qs_lo[0] - ti.qr0, row0b = ti.qs_lo[1] - ti.qr0;
      const int qn0 = ti.qs_n[0], qn1 = ti.qs_n[1];
      const uint64_t dqs = sdesc_sw<kRB>(smem_u32(smem + stage * C::STAGE_BYTES));
      const uint64_t dkt = dqs + ((2 * C::Q_BYTES) >> 4), dvt = dkt + (C::KT_BYTES >> 4);
      for (int k = 0; k < nch; ++k, ++c) {
        const int x = c & 1;
        // N = the chunk's (even) row count x QP: a full chunk, or 2 (QP = 24) / 2 or 4 (QP = 16) rows
        const int rows_k = chunk_rows_even<C::CR>(qn0, qn1, k);
        const uint32_t ids = rows_k == C::CR ? idesc_s : rows_k == 2 ? idesc_s2 : idesc_el<F16>(64, rows_k * QP, false);
        if (c >= 2) mbar_wait(&slot_free[x], ((c >> 1) - 1) & 1);
        tc_fence_after();
        // descriptors: per-stage bases + immediate offsets (short issue bursts, no per-MMA chains)
        const uint64_t dq0 = dqs + (((row0a + C::CR * k) * QP * kRB) >> 4);
        const uint64_t dq1 = dqs + (((row0b + C::CR * k) * QP * kRB) >> 4);
        const uint32_t s0 = tmem + x * kSlot, s1 = s0 + ((uint32_t)16 << 16);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t ko = (kk * 32) >> 4;
            mma_ss(s0, dkt + ko, dq0 + ko, ids, kk);
            mma_ss(s0 + kNCH, dvt + ko, dq0 + (C::Q_BYTES >> 4) + ko, ids, kk);
            mma_ss(s1, dkt + ((64 * kRB) >> 4) + ko, dq1 + ko, ids, kk);
            mma_ss(s1 + kNCH, dvt + ((64 * kRB) >> 4) + ko, dq1 + (C::Q_BYTES >> 4) + ko, ids, kk);
          }
          mma_commit(&s_full[x]);
        }
        __syncwarp();
        if (lane == 0) ktrace(p, c, 0);
      }
    }
  } else if (warp == kMmaKvWarp) {
    // ================= dV / dK issuer: chunk c once its P^T / dS^T are in TMEM; accumulates in TMEM
    // buffer (tile & 1), so a tile's MMAs never wait for the previous tile's epilogue
    constexpr uint32_t idesc_o = idesc_el<F16>(64, D, true);
    int c = 0;
    for (int it = 0;; ++it) {
      const int stage = it % kStages, b = it % kNacc;
      // the stage cannot advance past this tile before this warp commits its empty[] below
      mbar_wait(&full_mma[stage], (it / kStages) & 1);
      const TileInfo &ti = tinfo[stage];
      if (ti.bh < 0) break;
      const int nch = ti.nchunks, row0a = ti.qs_lo[0] - ti.qr0, row0b = ti.qs_lo[1] - ti.qr0;
      const int qn0 = ti.qs_n[0], qn1 = ti.qs_n[1];
      const uint64_t dqs = sdesc_sw<kRB>(smem_u32(smem + stage * C::STAGE_BYTES));
      const uint32_t o0 = tmem + kACC_COL + b * 2 * D, o1 = o0 + ((uint32_t)16 << 16);
      for (int k = 0; k < nch; ++k, ++c) {
        const int x = c & 1;
        mbar_wait(&ds_full[x], (c >> 1) & 1);
        if (lane == 0) ktrace(p, c, 1);
        if (k == 0) mbar_wait(&acc_free[b], ((it / kNacc) & 1) ^ 1);
        if (lane == 0) ktrace(p, c, 2);
        tc_fence_after();
        const uint64_t dq0 = dqs + (((row0a + C::CR * k) * QP * kRB) >> 4);
        const uint64_t dq1 = dqs + (((row0b + C::CR * k) * QP * kRB) >> 4);
        const uint32_t a0 = tmem + x * kSlot, a1 = a0 + ((uint32_t)16 << 16);
        const uint32_t acc0 = k == 0 ? 0u : 1u;
        const int nks = chunk_rows_even<C::CR>(qn0, qn1, k) * QP / 16;  // K-steps actually holding P / dS
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kNCH / 16; ++ks) {
            if (ks >= nks) break;
            const uint32_t acc = ks == 0 ? acc0 : 1u;
            const uint32_t bo = (ks * 16 * kRB) >> 4, doo = (C::Q_BYTES >> 4) + bo;
            mma_ts(o0, a0 + ks * 8, dq0 + doo, idesc_o, acc);              // dV += P^T dO
            mma_ts(o0 + D, a0 + kNCH + ks * 8, dq0 + bo, idesc_o, acc);    // dK += dS^T Q
            mma_ts(o1, a1 + ks * 8, dq1 + doo, idesc_o, acc);
            mma_ts(o1 + D, a1 + kNCH + ks * 8, dq1 + bo, idesc_o, acc);
          }
          mma_commit(&slot_free[x]);
          if (k == nch - 1) {
            mma_commit(&acc_full[b]);
            mma_commit(&empty[stage]);
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ================= elementwise groups: group grp handles CTA-global chunks c with c % 2 == grp
    const int grp = warp >> 2;
    const int quarter = warp & 3;
    const int half = lane >> 4, r = (lane >> 2) & 3, cc = lane & 3;
    const int Lh = wlen(p.H, L), Lw = wlen(p.W, L);
    const uint32_t lane_q = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = p.scale * log2e;
    // output staging of this warp (dV, dK: two 4x4-key blocks each, SW64 layout of the TMA store)
    uint8_t *ostage = smem + C::OUT_OFF + (grp * 4 + quarter) * C::OUT_W;
    const bool trq = quarter == 2 && lane == 0;
    // ---- epilogue of a tile: dV, dK (scale) from accumulator buffer (tile & 1), TMA-stored via
    // smem.  Deferred until the group has processed its next chunk, so it never waits for the
    // tile's last dV/dK MMAs (the MMA warp needs the buffer again only two tiles later).
    auto epilogue = [&](int eit, int bh, int kr0, int kc0) {
      const int b = eit % kNacc;
      mbar_wait(&acc_full[b], (eit / kNacc) & 1);
      tc_fence_after();
      // pair mode: key columns of member quarter >> 1
      const int ec0 = p.pair ? 4 * (quarter & 1) : kc0 + 4 * quarter, ebh = p.pair ? bh + (quarter >> 1) * p.heads : bh;
      if constexpr (C::EPI_DIRECT) {
        // straight to global memory, 16 head dims at a time: this thread's key (r, cc) of block `half`
        const int pk = kr0 + 4 * half + r, qk = ec0 + cc;
        const bool ok = pk < p.kv_row0 + p.kv_rows && qk < p.W;
        const size_t row = ((size_t)ebh * p.kv_rows + (pk - p.kv_row0)) * p.W + qk;
#pragma unroll
        for (int z16 = 0; z16 < D / 16; ++z16) {
          uint32_t a0[16], a1[16];
          tmem_ld16(lane_q + kACC_COL + b * 2 * D + 16 * z16, a0);
          tmem_ld16(lane_q + kACC_COL + b * 2 * D + D + 16 * z16, a1);
          tc_wait_ld();
          if (ok) {
            uint4 *dv4 = (uint4 *)(p.dv + row * D + 16 * z16), *dk4 = (uint4 *)(p.dk + row * D + 16 * z16);
#pragma unroll
            for (int z = 0; z < 2; ++z) {
              dv4[z] = make_uint4(pack_el<F16>(__uint_as_float(a0[8 * z]), __uint_as_float(a0[8 * z + 1])),
                                  pack_el<F16>(__uint_as_float(a0[8 * z + 2]), __uint_as_float(a0[8 * z + 3])),
                                  pack_el<F16>(__uint_as_float(a0[8 * z + 4]), __uint_as_float(a0[8 * z + 5])),
                                  pack_el<F16>(__uint_as_float(a0[8 * z + 6]), __uint_as_float(a0[8 * z + 7])));
              dk4[z] = make_uint4(
                  pack_el<F16>(__uint_as_float(a1[8 * z]) * p.scale, __uint_as_float(a1[8 * z + 1]) * p.scale),
                  pack_el<F16>(__uint_as_float(a1[8 * z + 2]) * p.scale, __uint_as_float(a1[8 * z + 3]) * p.scale),
                  pack_el<F16>(__uint_as_float(a1[8 * z + 4]) * p.scale, __uint_as_float(a1[8 * z + 5]) * p.scale),
                  pack_el<F16>(__uint_as_float(a1[8 * z + 6]) * p.scale, __uint_as_float(a1[8 * z + 7]) * p.scale));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_free[b]);
      } else {
        uint32_t a0[D], a1[D];
        ld_row<D>(lane_q + kACC_COL + b * 2 * D, a0);
        ld_row<D>(lane_q + kACC_COL + b * 2 * D + D, a1);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_free[b]);
        if (lane == 0) bulk_wait_read0();  // this warp's previous stores have left the staging
        __syncwarp();
        // key (r, cc) of block `half` is row R of its box; 16-byte chunk z at the TMA swizzle position of
        // rows of kRB bytes
        const int R = r * 4 + cc;
        uint8_t *rv = ostage + half * 16 * kRB + R * kRB, *rk = rv + 2 * 16 * kRB;
#pragma unroll
        for (int z = 0; z < D / 8; ++z) {
          const int zz = kRB == 32 ? (z ^ ((R >> 2) & 1)) : kRB == 64 ? (z ^ ((R >> 1) & 3)) : (z ^ (R & 7));
          *(uint4 *)(rv + 16 * zz) = make_uint4(
              pack_el<F16>(__uint_as_float(a0[8 * z]), __uint_as_float(a0[8 * z + 1])),
              pack_el<F16>(__uint_as_float(a0[8 * z + 2]), __uint_as_float(a0[8 * z + 3])),
              pack_el<F16>(__uint_as_float(a0[8 * z + 4]), __uint_as_float(a0[8 * z + 5])),
              pack_el<F16>(__uint_as_float(a0[8 * z + 6]), __uint_as_float(a0[8 * z + 7])));
          *(uint4 *)(rk + 16 * zz) = make_uint4(
              pack_el<F16>(__uint_as_float(a1[8 * z]) * p.scale, __uint_as_float(a1[8 * z + 1]) * p.scale),
              pack_el<F16>(__uint_as_float(a1[8 * z + 2]) * p.scale, __uint_as_float(a1[8 * z + 3]) * p.scale),
              pack_el<F16>(__uint_as_float(a1[8 * z + 4]) * p.scale, __uint_as_float(a1[8 * z + 5]) * p.scale),
              pack_el<F16>(__uint_as_float(a1[8 * z + 6]) * p.scale, __uint_as_float(a1[8 * z + 7]) * p.scale));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {  // out-of-range keys (map / band edge) are clipped by the TMA unit
#pragma unroll
          for (int sb = 0; sb < 2; ++sb) {
            tma_store_4d(&tm_dv, ostage + sb * 16 * kRB, 0, ec0, kr0 - p.kv_row0 + 4 * sb, ebh);
            tma_store_4d(&tm_dk, ostage + (2 + sb) * 16 * kRB, 0, ec0, kr0 - p.kv_row0 + 4 * sb, ebh);
          }
          bulk_commit();
        }
      }
    };
    int cur_head = -1;
    int c = 0;
    int pend_it = -1, pend_bh = 0, pend_kr0 = 0, pend_kc0 = 0;  // deferred epilogue
    for (int it = 0;; ++it) {
      const int stage = it % kStages;
      mbar_wait(&full[stage], (it / kStages) & 1);  // tile description, LSE / D staged
      if (trq) ktrace(p, c, 16 + 4 * grp);
      const TileInfo &ti = tinfo[stage];
      if (ti.bh < 0) break;  // end of work
      const int h = ti.head, bh = ti.bh, kr0 = ti.kr0, kc0 = ti.kc0, qr0 = ti.qr0, qc0 = ti.qc0;
      const int nch = ti.nchunks, qs_lo = ti.qs_lo[half], qs_n = ti.qs_n[half];
      const int qn0 = ti.qs_n[0], qn1 = ti.qs_n[1];
      const int uc = ti.uc[quarter];
      const bool fast = ti.fast[quarter];
      float2 mcol[C::UCW / 2];  // border path: 0 if this lane's key column is in union column z's window
      if (h != cur_head) {  // both groups rebuild the shared table: sync all 256 threads
        named_bar_sync(1, 256);
        const int tid256 = threadIdx.x;
        BiasTable<L>::build_rows(tbl, p.rpb, h, Lw, sl2, tid256, 256);  // (measured fastest here)
        // the all -inf class L and the unmasked class L + 1: one row per thread past the L classes
        for (int row = tid256; row < (L + 2) * C::TROWS; row += 256) {
          if (row < L * C::TROWS) continue;  // a masked class row: built by build_rows
          const int rr = row % C::TROWS;
          const bool live = row >= (L + 1) * C::TROWS && rr < C::TT;
          float b[C::TT];
#pragma unroll
          for (int k2 = 0; k2 < C::TT; ++k2) b[k2] = (p.rpb && live) ? __ldg(&p.rpb[(h * C::TT + rr) * C::TT + k2]) * sl2 : 0.f;
          float *dst = tbl + row * kTblStride;
#pragma unroll
          for (int e = 0; e < kTblStride; ++e) {
            const int cb = e - kTblOff;
            float v = -INFINITY;
#pragma unroll
            for (int k2 = 0; k2 < C::TT; ++k2)
              if (cb == k2 && live) v = b[k2];
            dst[e] = v;
          }
        }
        named_bar_sync(1, 256);
        cur_head = h;
      }
      // this thread's key
      // this thread's key; pair mode: halo column of member quarter >> 1 (bias columns are key - query
      // differences inside one member; mcol masks the other member's columns)
      const int pk = kr0 + 4 * half + r,
                qk = p.pair ? (quarter >> 1) * (QP / 2) + 4 * (quarter & 1) + cc : kc0 + 4 * quarter + cc;
      const float *lsd = (const float *)(smem + stage * C::STAGE_BYTES + 2 * C::Q_BYTES + 2 * C::KT_BYTES);
      const float *tbl_row0 = tbl + kTblOff + qk + L - 1 - (qc0 + uc) + (fast ? C::NS : L + 1) * C::TROWS * kTblStride;
      if (!fast) {
        const int kl = p.pair ? 4 * (quarter & 1) + cc : qk;  // key column inside its map
#pragma unroll
        for (int z = 0; z < C::UCW; z += 2) {
          float mv[2];
#pragma unroll
          for (int o = 0; o < 2; ++o) {
            int j = qc0 + uc + z + o;  // query column (pair mode: inside the quarter's own member)
            bool ok = true;
            if (p.pair) {
              const int m = j / (QP / 2);
              j -= m * (QP / 2);
              ok = m == (quarter >> 1);
            }
            const int ws = wstart(min(j, p.W - 1), p.W, L);
            ok = ok && j < p.W && kl >= ws && kl < ws + Lw;
            mv[o] = ok ? 0.f : -INFINITY;
          }
          mcol[z / 2] = make_float2(mv[0], mv[1]);
        }
      }
      if (trq) ktrace(p, c, 17 + 4 * grp);
      for (int k = 0; k < nch; ++k, ++c) {
        if ((c & 1) != grp) continue;
        const int x = c & 1;
        if (trq) ktrace(p, c, 4);
        mbar_wait(&s_full[x], (c >> 1) & 1);
        if (trq) ktrace(p, c, 5);
        tc_fence_after();
        const int i_base = qs_lo + C::CR * k;  // query row of chunk row 0 (this half)
        const int rows_here = min(qs_n - C::CR * k, q_end - i_base);
        const float *lrow0 = lsd + (i_base - qr0) * C::LP + (qc0 & 3) + uc;
        const uint32_t lane_addr = lane_q + x * kSlot;
        // a quarter whose keys all lie past the map edge only feeds accumulator rows the TMA store
        // clips, so its P / dS columns may hold anything
        if ((p.pair ? 4 * (quarter & 1) : kc0 + 4 * quarter) < p.W) {
          if (fast)
            chunk_rows<L, QP, true, F16>(lane_addr, uc, tbl_row0, mcol, lrow0, pk, i_base, p.H, rows_here, Lh, sl2,
                                    chunk_rows_even<C::CR>(qn0, qn1, k));
          else
            chunk_rows<L, QP, false, F16>(lane_addr, uc, tbl_row0, mcol, lrow0, pk, i_base, p.H, rows_here, Lh, sl2,
                                     chunk_rows_even<C::CR>(qn0, qn1, k));
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[x]);
        if (trq) ktrace(p, c, 6);
        if (lane == 0) ktrace(p, c, 10 + quarter);
        if (pend_it >= 0) {
          epilogue(pend_it, pend_bh, pend_kr0, pend_kc0);
          pend_it = -1;
        }
        if (k == nch - 1) {
          pend_it = it;
          pend_bh = bh;
          pend_kr0 = kr0;
          pend_kc0 = kc0;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);  // done with this stage's LSE / D and TileInfo
    }
    if (pend_it >= 0) epilogue(pend_it, pend_bh, pend_kr0, pend_kc0);
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == kProducerWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
#ifdef NA2D_TRACE
    if (lane == 0 && p.trace) {
      uint64_t gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.trace[17408 + 2 * blockIdx.x + 1] = (long long)gt;
    }
#endif
  }
}

template <int L, int QP, int HD, bool F16>
cudaError_t launch_dkdv_t(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                          const float *lse, const void *dout, const float *D, void *dk, void *dv,
                          const float *drpb_part, int part_ctas, float *drpb, int *tile_counter,
                          cudaStream_t st) {
  using C = CfgK<L, QP, HD>;
  const cudaError_t attr_err = tc::ensure_smem_attr((const void *)na2d_bwd_dkdv_kernel<L, QP, HD, F16>, C::SMEM);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tdo, tk, tv, tdk, tdv;
  const int BH = g.B * g.heads;
  const bool pair = pair_mode(g.B, g.H, g.W, g.q_row0, g.q_rows, g.kv_row0, g.kv_rows);
  if (!(pair ? make_tmap_e16_pair(F16, &tq, q, HD, g.W, g.q_rows, g.heads, BH, QP / 2, C::QRH)
             : make_tmap_e16_4d(F16, &tq, q, HD, g.W, g.q_rows, BH, QP, C::QRH)) ||
      !(pair ? make_tmap_e16_pair(F16, &tdo, dout, HD, g.W, g.q_rows, g.heads, BH, QP / 2, C::QRH)
             : make_tmap_e16_4d(F16, &tdo, dout, HD, g.W, g.q_rows, BH, QP, C::QRH)) ||
      !make_tmap_e16_4d(F16, &tk, k, HD, g.W, g.kv_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tv, v, HD, g.W, g.kv_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tdk, dk, HD, g.W, g.kv_rows, BH, 4, 4) ||
      !make_tmap_e16_4d(F16, &tdv, dv, HD, g.W, g.kv_rows, BH, 4, 4))
    return cudaErrorInvalidValue;
  CUtensorMap tl, td;
  const bool tma_lsd = !pair && (g.W * 4) % 16 == 0 && make_tmap_f32_3d(&tl, lse, g.W, g.q_rows, BH, C::LP, C::QRH) &&
                       make_tmap_f32_3d(&td, D, g.W, g.q_rows, BH, C::LP, C::QRH);
  if (!tma_lsd) tl = td = tq;  // unused
  BwdKParams p;
  p.tma_lsd = tma_lsd ? 1 : 0;
  p.pair = pair ? 1 : 0;
  p.B = pair ? g.B / 2 : g.B;
  p.heads = g.heads;
  p.H = g.H;
  p.W = g.W;
  p.q_rows = g.q_rows;
  p.q_row0 = g.q_row0;
  p.kv_rows = g.kv_rows;
  p.kv_row0 = g.kv_row0;
  p.tiles_h = (g.kv_rows + kTQH - 1) / kTQH;
  p.tiles_w = (g.W + kTQW - 1) / kTQW;
  p.num_tiles = p.B * g.heads * p.tiles_h * p.tiles_w;
  p.shift_cols = 0;
  if (max_query_halo_width(g, false) > QP) p.shift_cols = 1;
  p.scale = g.scale;
  p.rpb = rpb;
  p.lse = lse;
  p.D = D;
  p.tile_counter = tile_counter;
  p.drpb_part = drpb_part;
  p.part_ctas = part_ctas;
  p.drpb = drpb;
  p.dk = (__nv_bfloat16 *)dk;
  p.dv = (__nv_bfloat16 *)dv;
  p.trace = (long long *)debug_trace_buffer();
  const int grid = p.num_tiles < tc::num_sms() ? p.num_tiles : tc::num_sms();
  ProfScope ps("na2d_bwd_dkdv_tc", st);
  const cudaError_t e = launch_pdl(na2d_bwd_dkdv_kernel<L, QP, HD, F16>, grid, kThreads, C::SMEM, st, tq, tdo, tk, tv, tl, td, tdk, tdv, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// widest query halo over the key tile columns (host replica of inv_lo / inv_hi and key_col0), with
// the standard (shift = false) or shifted (shift = true) column origins
int max_query_halo_width(const Geo &g, bool shift) {
  const int L = g.L, W = g.W, len = wlen(W, L), tw = (W + tc::kTQW - 1) / tc::kTQW;
  auto lo = [&](int p) {
    int i = p - L + 1 > 0 ? p - L + 1 : 0;
    while (i < W && wstart(i, W, L) + len - 1 < p) ++i;
    return i;
  };
  auto hi = [&](int p) {
    int i = p + L - 1 < W - 1 ? p + L - 1 : W - 1;
    while (i >= 0 && wstart(i, W, L) > p) --i;
    return i;
  };
  int w = 0;
  for (int t = 0; t < tw; ++t) {
    int c0 = t * tc::kTQW;
    if (shift && t >= tw - 2) c0 = t == tw - 1 ? W - tc::kTQW : W - L - tc::kTQW;
    if (c0 < 0) return 1 << 20;
    const int c1 = c0 + tc::kTQW - 1 < W - 1 ? c0 + tc::kTQW - 1 : W - 1;
    const int ww = hi(c1) - (lo(c0) & ~1) + 1;  // the kernel rounds the halo origin down to even
    w = ww > w ? ww : w;
  }
  return w;
}

bool tc_dkdv_supported(const Geo &g) {
  return max_query_halo_width(g, false) <= 24 || max_query_halo_width(g, true) <= 24;
}


cudaError_t tc_backward_dkdv(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                             const float *lse, const void *dout, const float *D, void *dk, void *dv,
                             const float *drpb_part, int part_ctas, float *drpb, int *tile_counter,
                             cudaStream_t st) {
  // the query halo of a 16-column key tile is at most 16 + 2NS + 1 <= 23 columns away from the right
  // clamp zone; tiles reaching it are shifted (key_col0)
  if (!tc_dkdv_supported(g)) return cudaErrorNotSupported;
  static const bool no_narrow = [] {
    const char *e = getenv("NA2D_NO_NARROW");
    return e && e[0] == '1';
  }();
  // (not in pair mode: measured neutral-to-slower there, stage 4 B2 34.6 -> 35.0 us)
  const bool narrow = !no_narrow && !tc::pair_mode(g.B, g.H, g.W, g.q_row0, g.q_rows, g.kv_row0, g.kv_rows) &&
                      max_query_halo_width(g, false) <= 16;
  auto for_d = [&](auto hd_tag, auto f16_tag) -> cudaError_t {
    constexpr int HD = decltype(hd_tag)::value;
    constexpr bool F16 = decltype(f16_tag)::value;
    // query-halo row pitch 16 when every key tile's query halo fits (maps up to ~16 wide): a 96-query
    // chunk then holds 6 halo rows instead of 4 (NAT stage 3, 14 x 14: B2 62.2 -> 57.6 us)
    if (narrow) switch (g.L) {
      case 3: return launch_dkdv_t<3, 16, HD, F16>(g, q, k, v, rpb, lse, dout, D, dk, dv, drpb_part, part_ctas, drpb, tile_counter, st);
      case 5: return launch_dkdv_t<5, 16, HD, F16>(g, q, k, v, rpb, lse, dout, D, dk, dv, drpb_part, part_ctas, drpb, tile_counter, st);
      case 7: return launch_dkdv_t<7, 16, HD, F16>(g, q, k, v, rpb, lse, dout, D, dk, dv, drpb_part, part_ctas, drpb, tile_counter, st);
    }
    switch (g.L) {
      case 3: return launch_dkdv_t<3, 24, HD, F16>(g, q, k, v, rpb, lse, dout, D, dk, dv, drpb_part, part_ctas, drpb, tile_counter, st);
      case 5: return launch_dkdv_t<5, 24, HD, F16>(g, q, k, v, rpb, lse, dout, D, dk, dv, drpb_part, part_ctas, drpb, tile_counter, st);
      case 7: return launch_dkdv_t<7, 24, HD, F16>(g, q, k, v, rpb, lse, dout, D, dk, dv, drpb_part, part_ctas, drpb, tile_counter, st);
    }
    return cudaErrorInvalidValue;
  };
  using T = std::true_type;
  using Fa = std::false_type;
  const bool f16 = g.dtype == NA2D_F16;
  if (g.d == 16) return f16 ? for_d(std::integral_constant<int, 16>(), T()) : for_d(std::integral_constant<int, 16>(), Fa());
  if (g.d == 32) return f16 ? for_d(std::integral_constant<int, 32>(), T()) : for_d(std::integral_constant<int, 32>(), Fa());
  if (g.d == 64) return f16 ? for_d(std::integral_constant<int, 64>(), T()) : for_d(std::integral_constant<int, 64>(), Fa());
  return cudaErrorInvalidValue;
}

}  // namespace na2d
