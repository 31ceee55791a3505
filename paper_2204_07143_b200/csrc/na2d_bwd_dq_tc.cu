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

constexpr int kStages = 2;
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 elementwise + epilogue
constexpr int kQAcc = 3;       // independent dQ accumulators
constexpr int kDP_COL = 256;   // dP accumulator columns

template <int L>
struct CfgQ {
  static constexpr int HR = kTQH + L - 1;
  static constexpr int UR = 4 + L - 1;
  static constexpr int NSUB = UR * kHCP;
  static constexpr int UCW = L + 5;
  static constexpr int DS_COL = 0;         // dS (bf16 pairs) over consumed S columns
  static constexpr int Q_COL = NSUB / 2;   // dQ partial accumulators in dead S columns
  static_assert(Q_COL + kQAcc * kD <= kDP_COL, "TMEM budget");
  static_assert(kDP_COL + NSUB <= 512, "TMEM budget");
  static constexpr int KV_ROWS = HR * kHCP;
  static constexpr int Q_BYTES = 128 * kRowBytes;
  static constexpr int KV_BYTES = KV_ROWS * kRowBytes;
  static constexpr int STAGE_BYTES = 2 * Q_BYTES + 2 * KV_BYTES;  // Q, dO, K, V
  static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1 KB aligned (swizzled TMA / UMMA)");
  static constexpr int TT = 2 * L - 1;
  static constexpr int TBL_OFF = kStages * STAGE_BYTES;
  static constexpr int DB_OFF = TBL_OFF + BiasTable<L>::FLOATS * 4;
  static constexpr int BAR_OFF = DB_OFF + ((TT * TT * 4 + 255) / 256) * 256;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};

__device__ __forceinline__ TileOrder::Tile decode(const BwdQParams &p, int t) { return p.order.decode(t); }

template <int L>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const BwdQParams p) {
  using C = CfgQ<L>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float *tbl = (float *)(smem + C::TBL_OFF);
  float *s_db = (float *)(smem + C::DB_OFF);
  uint64_t *bars = (uint64_t *)(smem + C::BAR_OFF);
  uint64_t *full = bars, *empty = bars + kStages;
  uint64_t *sp_full = bars + 2 * kStages, *ds_full = sp_full + 1, *dq_full = sp_full + 2, *tmem_free = sp_full + 3;
  uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages + 4);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t_begin = (int)((long)p.num_tiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((long)p.num_tiles * (blockIdx.x + 1) / gridDim.x);
  const int q_end = p.q_row0 + p.q_rows;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(sp_full, 1);
    mbar_init(ds_full, 4);
    mbar_init(dq_full, 1);
    mbar_init(tmem_free, 4);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  for (int c = threadIdx.x; c < C::TT * C::TT; c += kThreads) s_db[c] = 0.f;
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer
    if (elect_one()) {
      int it = 0;
      for (int t = t_begin; t < t_end; ++t, ++it) {
        const int s = it % kStages;
        mbar_wait_sleep(&empty[s], ((it / kStages) & 1) ^ 1, 1024);
        const TileOrder::Tile g = decode(p, t);
        const int hr0 = wstart(g.i0, p.H, L), hc0 = wstart(g.j0, p.W, L);
        uint8_t *st = smem + s * C::STAGE_BYTES;
        mbar_expect_tx(&full[s], C::STAGE_BYTES);
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
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(64, C::NSUB, false);
    constexpr uint32_t idesc_q = idesc_bf16(64, kD, true);
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      const int s = it % kStages;
      const uint32_t ph = it & 1;
      const TileOrder::Tile g = decode(p, t);
      const int hr0 = wstart(g.i0, p.H, L);
      const int rb0 = wstart(min(g.i0, q_end - 1), p.H, L) - hr0;
      const int rb1 = wstart(min(g.i0 + 4, q_end - 1), p.H, L) - hr0;
      mbar_wait_sleep(&full[s], (it / kStages) & 1, 64);
      mbar_wait_sleep(tmem_free, ph ^ 1, 64);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(smem + s * C::STAGE_BYTES);
      const uint32_t do_addr = q_addr + C::Q_BYTES;
      const uint32_t k_addr = q_addr + 2 * C::Q_BYTES;
      const uint32_t v_addr = k_addr + C::KV_BYTES;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kD / 16; ++k)
#pragma unroll
          for (int sb = 0; sb < 2; ++sb) {
            const uint32_t lo = (uint32_t)(16 * sb) << 16;
            const int rb = sb ? rb1 : rb0;
            mma_ss(tmem + lo, sdesc_sw64(q_addr + sb * 4096 + k * 32),
                   sdesc_sw64(k_addr + rb * kHCP * kRowBytes + k * 32), idesc_s, k);
            mma_ss(tmem + lo + kDP_COL, sdesc_sw64(do_addr + sb * 4096 + k * 32),
                   sdesc_sw64(v_addr + rb * kHCP * kRowBytes + k * 32), idesc_s, k);
          }
        mma_commit(sp_full);
      }
      __syncwarp();
      mbar_wait_sleep(ds_full, ph, 64);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < C::NSUB / 16; ++ks)
#pragma unroll
          for (int sb = 0; sb < 2; ++sb) {
            const uint32_t base = tmem + ((uint32_t)(16 * sb) << 16);
            const int rb = sb ? rb1 : rb0;
            mma_ts(base + C::Q_COL + (ks % kQAcc) * kD, base + C::DS_COL + ks * 8,
                   sdesc_sw64(k_addr + rb * kHCP * kRowBytes + ks * 16 * kRowBytes), idesc_q, ks >= kQAcc);
          }
        mma_commit(dq_full);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    // ================= elementwise + epilogue (warps 2..5 -> TMEM lane quarters 2,3,0,1)
    const int quarter = warp & 3;
    const int half = lane >> 4, r = (lane >> 2) & 3, c = lane & 3;
    const int gtid = threadIdx.x - 64;
    const int Lh = wlen(p.H, L), Lw = wlen(p.W, L);
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const float sl2 = p.scale * 1.4426950408889634f;
    // dRPB accumulator in union coordinates for the current (class, head) and its geometry
    float acc[C::UR][C::UCW];
#pragma unroll
    for (int u = 0; u < C::UR; ++u)
#pragma unroll
      for (int z = 0; z < C::UCW; ++z) acc[u][z] = 0.f;
    int cur_key = -1, cur_head = -1;
    int f_wr = 0, f_wc = 0, f_brow = 0, f_bcol = 0;  // geometry of the accumulated class
    auto flush = [&]() {
      // masked to this lane's window; cells (f_brow + u, f_bcol + z)
#pragma unroll
      for (int u = 0; u < C::UR; ++u)
#pragma unroll
        for (int z = 0; z < C::UCW; ++z) {
          if ((unsigned)(u - f_wr) < (unsigned)Lh && (unsigned)(z - f_wc) < (unsigned)Lw)
            atomicAdd(&s_db[(f_brow + u) * C::TT + f_bcol + z], acc[u][z]);
          acc[u][z] = 0.f;
        }
    };
    auto commit_head = [&](int head) {  // per-CTA table -> partials[cta][head]; clear
      named_bar_sync(1, 128);
      if (head >= 0 && p.drpb_part)
        for (int e = gtid; e < C::TT * C::TT; e += 128) {
          float *dst = &p.drpb_part[((size_t)blockIdx.x * p.heads + head) * C::TT * C::TT + e];
          *dst += p.scale * s_db[e];
          s_db[e] = 0.f;
        }
      named_bar_sync(1, 128);
    };
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      const uint32_t ph = it & 1;
      const TileOrder::Tile g = decode(p, t);
      const int h = g.bh % p.heads;
      const int key = g.cls * p.heads + h;
      const int hr0 = wstart(g.i0, p.H, L), hc0 = wstart(g.j0, p.W, L);
      const int i = g.i0 + 4 * half + r, j = g.j0 + 4 * quarter + c;
      const int ic = min(i, q_end - 1), jc = min(j, p.W - 1);
      const int si = wstart(ic, p.H, L), sj = wstart(jc, p.W, L);
      const int rb = wstart(min(g.i0 + 4 * half, q_end - 1), p.H, L) - hr0;
      const int uc = (wstart(min(g.j0 + 4 * quarter, p.W - 1), p.W, L) - hc0) & ~1;
      const int dc = sj - jc + L - 1;
      const int brow0 = hr0 + rb - ic + L - 1, bcol0 = hc0 + uc - jc + L - 1;
      if (key != cur_key) {
        if (p.rpb && cur_key >= 0) flush();
        if (h != cur_head) {
          if (p.rpb) commit_head(cur_head);
          named_bar_sync(1, 128);
          BiasTable<L>::build(tbl, p.rpb, h, Lw, sl2, gtid, 128);
          named_bar_sync(1, 128);
          cur_head = h;
        }
        cur_key = key;
        f_wr = si - hr0 - rb;
        f_wc = sj - hc0 - uc;
        f_brow = brow0;
        f_bcol = bcol0;
      }
      // own query: LSE (log2 units)
      const bool qvalid = i < q_end && j < p.W;
      const size_t qi = ((size_t)g.bh * p.q_rows + (ic - p.q_row0)) * p.W + jc;
      const float lse2 = qvalid ? p.lse[qi] * 1.4426950408889634f : 0.f;
      const float *tcls = tbl + dc * BiasTable<L>::TROWS * kTblStride + kTblOff + bcol0;
      mbar_wait(sp_full, ph);
      tc_fence_after();
      // ---- pass 1: P = exp2(s*scale*log2e + B' - LSE*log2e) (fp32, written over S in place) and
      // D = dO.O = sum_window P dP (exact in fp32: O = sum P V, so dO.O = sum P (dO.v))
      float Dq = 0.f;
#pragma unroll 1
      for (int u = 0; u < C::UR; u += 2) {
        uint32_t sa[16], sb_[16], pa_[16], pb_[16];
        const uint32_t ca = lane_addr + u * kHCP + uc;
        tmem_ld16(ca, sa);
        tmem_ld16(ca + kHCP, sb_);
        tmem_ld16(ca + kDP_COL, pa_);
        tmem_ld16(ca + kDP_COL + kHCP, pb_);
        const int pr = hr0 + rb + u;
        const bool rva = (unsigned)(pr - si) < (unsigned)Lh, rvb = (unsigned)(pr + 1 - si) < (unsigned)Lh;
        const float *ta = tcls + (rva ? pr - ic + L - 1 : C::TT) * kTblStride;
        const float *tb = tcls + (rvb ? pr + 1 - ic + L - 1 : C::TT) * kTblStride;
        tc_wait_ld();
        float da = 0.f, db = 0.f;
#pragma unroll
        for (int z = 0; z < C::UCW; ++z) {
          const float P0 = ex2(fmaf(__uint_as_float(sa[z]), sl2, ta[z]) - lse2);
          const float P1 = ex2(fmaf(__uint_as_float(sb_[z]), sl2, tb[z]) - lse2);
          da = fmaf(P0, __uint_as_float(pa_[z]), da);
          db = fmaf(P1, __uint_as_float(pb_[z]), db);
          sa[z] = __float_as_uint(P0);
          sb_[z] = __float_as_uint(P1);
        }
        Dq += da + db;
        tmem_st16(ca, sa);
        tmem_st16(ca + kHCP, sb_);
      }
      if (qvalid) p.D[qi] = Dq;
      tc_wait_st();
      // ---- pass 2: dS = P (dP - D) -> dRPB accumulators (union coordinates) and bf16 pairs over
      // the consumed S/P columns (the dQ MMA's A operand)
      const int zb = uc >> 1;
#pragma unroll
      for (int u = 0; u < C::UR; u += 2) {
        uint32_t sa[16], sb_[16], pa_[16], pb_[16];
        const uint32_t ca = lane_addr + u * kHCP + uc;
        tmem_ld16(ca, sa);
        tmem_ld16(ca + kHCP, sb_);
        tmem_ld16(ca + kDP_COL, pa_);
        tmem_ld16(ca + kDP_COL + kHCP, pb_);
        tc_wait_ld();
        uint32_t da[C::UCW / 2], db[C::UCW / 2];
#pragma unroll
        for (int z = 0; z < C::UCW; z += 2) {
          float d2[2][2];
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            d2[0][y] = __uint_as_float(sa[z + y]) * (__uint_as_float(pa_[z + y]) - Dq);
            d2[1][y] = __uint_as_float(sb_[z + y]) * (__uint_as_float(pb_[z + y]) - Dq);
            acc[u][z + y] += d2[0][y];
            acc[u + 1][z + y] += d2[1][y];
          }
          da[z / 2] = pack_bf16_alu(d2[0][0], d2[0][1]);
          db[z / 2] = pack_bf16_alu(d2[1][0], d2[1][1]);
        }
        const uint32_t prow = lane_addr + C::DS_COL + u * (kHCP / 2);
        st_zero12(prow);
        st_zero12(prow + kHCP / 2);
        st_row<C::UCW / 2>(prow + zb, da);
        st_row<C::UCW / 2>(prow + kHCP / 2 + zb, db);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      // ---- epilogue: dQ = scale * sum of partial accumulators -> bf16
      mbar_wait(dq_full, ph);
      tc_fence_after();
      uint32_t o[32];
      {
        uint32_t oa[kQAcc][32];
#pragma unroll
        for (int a = 0; a < kQAcc; ++a) tmem_ld32(lane_addr + C::Q_COL + a * kD, oa[a]);
        tc_wait_ld();
#pragma unroll
        for (int z = 0; z < 32; ++z) {
          float s = __uint_as_float(oa[0][z]);
#pragma unroll
          for (int a = 1; a < kQAcc; ++a) s += __uint_as_float(oa[a][z]);
          o[z] = __float_as_uint(s * p.scale);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tmem_free);
      if (qvalid) {
        uint4 *dst = (uint4 *)(p.dq + qi * kD);
#pragma unroll
        for (int z = 0; z < kD; z += 8)
          dst[z / 8] = make_uint4(pack_bf16(__uint_as_float(o[z]), __uint_as_float(o[z + 1])),
                                  pack_bf16(__uint_as_float(o[z + 2]), __uint_as_float(o[z + 3])),
                                  pack_bf16(__uint_as_float(o[z + 4]), __uint_as_float(o[z + 5])),
                                  pack_bf16(__uint_as_float(o[z + 6]), __uint_as_float(o[z + 7])));
      }
    }
    if (p.rpb) {
      if (cur_key >= 0) flush();
      commit_head(cur_head);
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// drpb[h][c] = sum over CTAs of drpb_part[cta][h][c]: one warp per cell, lane l sums CTAs
// l, l+32, ... in order, then a fixed butterfly -- deterministic for a given CTA count.
__global__ void drpb_reduce_kernel(const float *__restrict__ part, int ctas, int n, float *__restrict__ drpb) {
  const int e = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (e >= n) return;
  float s = 0.f;
  for (int b = lane; b < ctas; b += 32) s += part[(size_t)b * n + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) drpb[e] = s;
}

template <int L>
cudaError_t launch_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, const void *out,
                      const float *lse, const void *dout, void *dq, float *drpb, float *D, float *part,
                      cudaStream_t st) {
  using C = CfgQ<L>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(na2d_bwd_dq_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tdo, tk, tv;
  const int BH = g.B * g.heads;
  if (!make_tmap_bf16_4d(&tq, q, kD, g.W, g.q_rows, BH, 4, 4) ||
      !make_tmap_bf16_4d(&tdo, dout, kD, g.W, g.q_rows, BH, 4, 4) ||
      !make_tmap_bf16_4d(&tk, k, kD, g.W, g.kv_rows, BH, kHCP, C::HR) ||
      !make_tmap_bf16_4d(&tv, v, kD, g.W, g.kv_rows, BH, kHCP, C::HR))
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
  const int grid = dq_grid(g);
  const int TT = 2 * L - 1;
  cudaError_t e;
  if (rpb) {
    e = cudaMemsetAsync(part, 0, sizeof(float) * grid * g.heads * TT * TT, st);
    if (e != cudaSuccess) return e;
  }
  {
    ProfScope ps("na2d_bwd_dq_tc", st);
    na2d_bwd_dq_kernel<L><<<grid, kThreads, C::SMEM, st>>>(tq, tdo, tk, tv, p);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess || !rpb) return e;
  {
    ProfScope ps("na2d_bwd_drpb_reduce", st);
    const int n = g.heads * TT * TT;
    drpb_reduce_kernel<<<(n + 3) / 4, 128, 0, st>>>(part, grid, n, drpb);
  }
  return cudaGetLastError();
}

}  // namespace

int dq_grid(const Geo &g) {
  const TileOrder o = make_tile_order(g, g.L);
  return o.num_tiles < tc::num_sms() ? o.num_tiles : tc::num_sms();
}

cudaError_t tc_backward_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                           const void *out, const float *lse, const void *dout, void *dq, float *drpb, float *D,
                           float *part, cudaStream_t st) {
  switch (g.L) {
    case 3: return launch_dq<3>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, st);
    case 5: return launch_dq<5>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, st);
    case 7: return launch_dq<7>(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, part, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace na2d
