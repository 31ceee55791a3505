// na2d_fwd_tc.cu -- NA2D forward on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Eq. 2 for bf16 Q/K/V, head dim 32, L in {3,5,7}:
//   one CTA tile = 8 x 16 queries (M = 128 TMEM lanes).  Their neighbourhoods rho (P:150,
//   P:163-164) all lie inside the halo rows [wstart(i0), +8+L-1) x cols [wstart(j0), +16+L-1)
//   (global clamped coordinates), which TMA stages into shared memory (zero-filled outside the
//   tensor).  The tile x halo products are dense contractions:
//     S = Q K_halo^T      (M=128, N=halo, K=32)   tcgen05.mma SS -> TMEM columns [0, NS)
//     O = P V_halo        (M=128, N=32, K=halo)   tcgen05.mma TS (P from TMEM) -> TMEM
//   Between them four softmax warps (one TMEM lane quarter each, 32 queries = a 4 x 8 query
//   block) read only their block's union of windows (<= (4+L-1) rows x 16 columns of S), add
//   the relative positional bias B[h][p-i+L-1][q-j+L-1] from shared memory, mask the
//   keys outside each query's own window, and compute the exact single-pass softmax (the whole
//   window is in one tile, so no online rescaling): max, exp2, sum, P (bf16) -> TMEM.
//   LSE (natural log) and O / sum are written by the same warps.
// Warp roles (persistent CTAs, one per SM): warp 0 TMA producer (3-stage ring), warp 1 MMA
// issuer, warps 2-5 softmax + epilogue.
#include <math.h>
#include <stdio.h>

#include <mutex>

#include "na2d_internal.cuh"
#include "na2d_profile.cuh"
#include "na2d_sm100.cuh"
#include "na2d_tc.cuh"
#include "na2d_tmap.cuh"

namespace na2d {
namespace {

using namespace sm100;

constexpr int kTQH = 8, kTQW = 16, kM = 128, kD = 32;
constexpr int kStages = 3;
constexpr int kThreads = 192;  // 6 warps
constexpr int kRowBytes = kD * 2;  // 64-byte rows (32 bf16)

template <int L>
struct Cfg {
  static constexpr int HR = kTQH + L - 1, HC = kTQW + L - 1;  // halo extent
  static constexpr int NKEYS = HR * HC;
  static constexpr int NS = (NKEYS + 31) / 32 * 32;          // padded key count (S columns)
  static constexpr int UR = 4 + L - 1;                       // union rows per 4x8 query block
  static constexpr int S_COL = 0, P_COL = NS, O_COL = NS + NS / 2;
  static_assert(O_COL + kD <= 512, "TMEM budget");
  static constexpr int N_HALF = NS > 256 ? NS / 2 : NS;      // MMA N per instruction (<= 256)
  static constexpr int N_PARTS = NS / N_HALF;
  static constexpr int Q_BYTES = kM * kRowBytes;             // 8 KB
  static constexpr int KV_BYTES = NS * kRowBytes;            // padded tile
  static constexpr int KV_TX = NKEYS * kRowBytes;            // bytes TMA delivers
  static constexpr int STAGE_BYTES = Q_BYTES + 2 * KV_BYTES;
  static constexpr int TT = 2 * L - 1;
  // >= 116 KB so that exactly one CTA (owning all 512 TMEM columns) is resident per SM
  static constexpr int SMEM_NEED = kStages * STAGE_BYTES + 1024 /*align*/ + 4096 /*table+bars*/;
  static constexpr int SMEM = SMEM_NEED > 120 * 1024 ? SMEM_NEED : 120 * 1024;
};

struct FwdParams {
  int B, heads, H, W, L, q_rows, q_row0, kv_rows, kv_row0;
  int tiles_h, tiles_w, num_tiles;
  float scale_log2;  // scale * log2(e)
  const float *rpb;  // [heads][TT][TT] or null
  __nv_bfloat16 *out;
  float *lse;
};

template <int L>
__global__ void __launch_bounds__(kThreads, 1)
    na2d_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
  using C = Cfg<L>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *stage_base = smem;
  float *s_table = (float *)(smem + kStages * C::STAGE_BYTES);                 // [TT*TT]
  uint64_t *bars = (uint64_t *)(smem + kStages * C::STAGE_BYTES + 2048);
  uint64_t *full = bars, *empty = bars + kStages;
  uint64_t *s_full = bars + 2 * kStages, *p_full = s_full + 1, *o_full = s_full + 2, *tmem_free = s_full + 3;
  uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages + 4);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // zero the padded key rows of every K/V stage once (TMA never writes them; V pad rows are
  // multiplied by P = 0 and must not hold NaN/Inf garbage)
  for (int s = 0; s < kStages; ++s) {
    uint8_t *kt = stage_base + s * C::STAGE_BYTES + C::Q_BYTES;
    for (int off = C::KV_TX + threadIdx.x * 16; off < C::KV_BYTES; off += kThreads * 16) {
      *(uint4 *)(kt + off) = make_uint4(0, 0, 0, 0);
      *(uint4 *)(kt + C::KV_BYTES + off) = make_uint4(0, 0, 0, 0);
    }
  }
  fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(tmem_free, 4);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int tiles_per_map = p.tiles_h * p.tiles_w;

  if (warp == 0) {
    // ================= TMA producer
    if (elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        const int s = it % kStages;
        mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        const int bh = t / tiles_per_map, rem = t % tiles_per_map;
        const int i0 = p.q_row0 + (rem / p.tiles_w) * kTQH, j0 = (rem % p.tiles_w) * kTQW;
        const int hr0 = wstart(i0, p.H, L), hc0 = wstart(j0, p.W, L);
        uint8_t *st = stage_base + s * C::STAGE_BYTES;
        mbar_expect_tx(&full[s], C::Q_BYTES + 2 * C::KV_TX);
        // Q as four 4x8 query blocks (TMEM lane quarter b <- block b)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          tma_load_4d(st + b * 32 * kRowBytes, &tm_q, &full[s], 0, j0 + 8 * (b & 1), i0 - p.q_row0 + 4 * (b >> 1), bh);
        tma_load_4d(st + C::Q_BYTES, &tm_k, &full[s], 0, hc0, hr0 - p.kv_row0, bh);
        tma_load_4d(st + C::Q_BYTES + C::KV_BYTES, &tm_v, &full[s], 0, hc0, hr0 - p.kv_row0, bh);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    constexpr uint32_t idesc_qk = idesc_bf16(kM, C::N_HALF, false);
    constexpr uint32_t idesc_pv = idesc_bf16(kM, kD, true);
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int s = it % kStages;
      const uint32_t ph = it & 1;
      mbar_wait(&full[s], (it / kStages) & 1);
      mbar_wait(tmem_free, ph ^ 1);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(stage_base + s * C::STAGE_BYTES);
      const uint32_t k_addr = q_addr + C::Q_BYTES;
      const uint32_t v_addr = k_addr + C::KV_BYTES;
      if (elect_one()) {
#pragma unroll
        for (int n = 0; n < C::N_PARTS; ++n)
#pragma unroll
          for (int k = 0; k < kD / 16; ++k)
            mma_ss(tmem + C::S_COL + n * C::N_HALF, sdesc_sw64(q_addr + k * 32),
                   sdesc_sw64(k_addr + n * C::N_HALF * kRowBytes + k * 32), idesc_qk, k);
        mma_commit(s_full);
      }
      __syncwarp();
      mbar_wait(p_full, ph);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll 4
        for (int ks = 0; ks < C::NS / 16; ++ks)
          mma_ts(tmem + C::O_COL, tmem + C::P_COL + ks * 8, sdesc_sw64(v_addr + ks * 16 * kRowBytes), idesc_pv,
                 ks);
        mma_commit(o_full);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  } else {
    // ================= softmax + epilogue (warps 2..5 -> TMEM lane quarters 2,3,0,1)
    const int quarter = warp & 3;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const int TT = C::TT;
    const int Lh = wlen(p.H, L), Lw = wlen(p.W, L);
    const int q_end = p.q_row0 + p.q_rows;
    int cur_head = -1;
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const uint32_t ph = it & 1;
      const int bh = t / tiles_per_map, rem = t % tiles_per_map;
      const int h = bh % p.heads;
      const int i0 = p.q_row0 + (rem / p.tiles_w) * kTQH, j0 = (rem % p.tiles_w) * kTQW;
      const int hr0 = wstart(i0, p.H, L), hc0 = wstart(j0, p.W, L);
      // this thread's query (block `quarter` = rows 4*(quarter>>1).., cols 8*(quarter&1)..)
      const int bi0 = i0 + 4 * (quarter >> 1), bj0 = j0 + 8 * (quarter & 1);
      const int i = bi0 + (lane >> 3), j = bj0 + (lane & 7);
      const int ic = min(i, q_end - 1), jc = min(j, p.W - 1);
      const int ur0 = wstart(min(bi0, q_end - 1), p.H, L) - hr0;
      const int uc0 = (wstart(min(bj0, p.W - 1), p.W, L) - hc0) & ~1;
      const int wr = wstart(ic, p.H, L) - hr0 - ur0;  // window origin inside the union
      const int wc = wstart(jc, p.W, L) - hc0 - uc0;
      // bias cell of union element (u, c): (hr0+ur0+u - ic + L-1, hc0+uc0+c - jc + L-1)
      const int brow0 = hr0 + ur0 - ic + L - 1, bcol0 = hc0 + uc0 - jc + L - 1;
      if (p.rpb && h != cur_head) {  // stage this head's bias table (tile-uniform branch)
        named_bar_sync(1, 128);
        for (int c = threadIdx.x - 64; c < TT * TT; c += 128) s_table[c] = __ldg(&p.rpb[h * TT * TT + c]);
        named_bar_sync(1, 128);
        cur_head = h;
      }
      mbar_wait(s_full, ph);
      tc_fence_after();
      // ---- pass 1: row max over the thread's window (log2 domain)
      float mx = -INFINITY;
      for (int u = 0; u < C::UR; ++u) {
        uint32_t r[16];
        tmem_ld16(lane_addr + C::S_COL + (ur0 + u) * C::HC + uc0, r);
        tc_wait_ld();
        const bool rv = (unsigned)(u - wr) < (unsigned)Lh;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const bool v = rv && (unsigned)(c - wc) < (unsigned)Lw;
          float b = 0.f;
          if (p.rpb && v) b = s_table[(brow0 + u) * TT + bcol0 + c];
          const float x = (__uint_as_float(r[c]) + b) * p.scale_log2;
          mx = v ? fmaxf(mx, x) : mx;
        }
      }
      // ---- zero this lane's P row, then pass 2: P = exp2(x - max) on the window, sum
#pragma unroll
      for (int c = 0; c < C::NS / 2; c += 32) tmem_st32_zero(lane_addr + C::P_COL + c);
      tc_wait_st();
      float sum = 0.f;
      for (int u = 0; u < C::UR; ++u) {
        uint32_t r[16];
        const int col = (ur0 + u) * C::HC + uc0;
        tmem_ld16(lane_addr + C::S_COL + col, r);
        tc_wait_ld();
        const bool rv = (unsigned)(u - wr) < (unsigned)Lh;
        uint32_t pk[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          float e[2];
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            const bool v = rv && (unsigned)(c + z - wc) < (unsigned)Lw;
            float b = 0.f;
            if (p.rpb && v) b = s_table[(brow0 + u) * TT + bcol0 + c + z];
            const float x = (__uint_as_float(r[c + z]) + b) * p.scale_log2;
            e[z] = v ? ex2(x - mx) : 0.f;
            sum += e[z];
          }
          pk[c / 2] = pack_bf16(e[0], e[1]);
        }
        tmem_st8(lane_addr + C::P_COL + col / 2, pk);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // ---- epilogue: O / sum -> bf16, LSE
      mbar_wait(o_full, ph);
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(lane_addr + C::O_COL, o);
      tc_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tmem_free);
      if (i < q_end && j < p.W) {
        const float inv = 1.f / sum;
        const size_t qi = ((size_t)bh * p.q_rows + (i - p.q_row0)) * p.W + j;
        uint4 *dst = (uint4 *)(p.out + qi * kD);
#pragma unroll
        for (int c = 0; c < kD; c += 8)
          dst[c / 8] = make_uint4(pack_bf16(__uint_as_float(o[c]) * inv, __uint_as_float(o[c + 1]) * inv),
                                  pack_bf16(__uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv),
                                  pack_bf16(__uint_as_float(o[c + 4]) * inv, __uint_as_float(o[c + 5]) * inv),
                                  pack_bf16(__uint_as_float(o[c + 6]) * inv, __uint_as_float(o[c + 7]) * inv));
        if (p.lse) p.lse[qi] = (mx + __log2f(sum)) * 0.69314718055994531f;
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int num_sms() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  });
  return n;
}

template <int L>
cudaError_t launch_fwd(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  using C = Cfg<L>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(na2d_fwd_tc_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap tq, tk, tv;
  const int BH = g.B * g.heads;
  if (!make_tmap_bf16_4d(&tq, q, kD, g.W, g.q_rows, BH, 8, 4) ||
      !make_tmap_bf16_4d(&tk, k, kD, g.W, g.kv_rows, BH, C::HC, C::HR) ||
      !make_tmap_bf16_4d(&tv, v, kD, g.W, g.kv_rows, BH, C::HC, C::HR))
    return cudaErrorInvalidValue;
  FwdParams p;
  p.B = g.B;
  p.heads = g.heads;
  p.H = g.H;
  p.W = g.W;
  p.L = L;
  p.q_rows = g.q_rows;
  p.q_row0 = g.q_row0;
  p.kv_rows = g.kv_rows;
  p.kv_row0 = g.kv_row0;
  p.tiles_h = (g.q_rows + kTQH - 1) / kTQH;
  p.tiles_w = (g.W + kTQW - 1) / kTQW;
  p.num_tiles = BH * p.tiles_h * p.tiles_w;
  p.scale_log2 = g.scale * 1.4426950408889634f;
  p.rpb = rpb;
  p.out = (__nv_bfloat16 *)out;
  p.lse = lse;
  const int grid = p.num_tiles < num_sms() ? p.num_tiles : num_sms();
  ProfScope ps("na2d_fwd_tc", st);
  na2d_fwd_tc_kernel<L><<<grid, kThreads, C::SMEM, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace

bool tc_forward_supported(const Geo &g) {
  return g.dtype == NA2D_BF16 && g.d == kD && (g.L == 3 || g.L == 5 || g.L == 7) && tmap_available();
}

cudaError_t tc_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st) {
  switch (g.L) {
    case 3: return launch_fwd<3>(g, q, k, v, rpb, out, lse, st);
    case 5: return launch_fwd<5>(g, q, k, v, rpb, out, lse, st);
    case 7: return launch_fwd<7>(g, q, k, v, rpb, out, lse, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace na2d
