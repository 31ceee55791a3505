// na2d_tc_bwd.cuh -- shared definitions of the tcgen05 backward kernels.
#pragma once

#include <cuda_bf16.h>

#include "na2d_internal.cuh"
#include "na2d_tc_common.cuh"

namespace na2d {

// Tile visiting order grouped by geometry class.  Tile rows (columns) whose 8 (16) query rows
// (columns) are all unclamped and inside the map form one "interior" group; every other tile row
// (column) is a group of its own.  A class is a (row group, column group) pair; consecutive tiles of
// a class share the per-lane union geometry.  Two orders (make_tile_order picks one):
//  * class-major: class, then head, batch, row, column -- when every class holds enough tiles per
//    head that a CTA's contiguous share crosses at most ~4 heads (e.g. NAT-Tiny stage 1: 128 maps
//    per head; ADE 128^2: 16);
//  * interior first: the interior class head-major, then per head every border class in class order
//    -- when the border classes hold only a few tiles per head (few maps, many heads, e.g. the ADE
//    map split into 32 (b,h) units), where class-major would switch heads (bias-table rebuild, dRPB
//    commit) at nearly every border tile.  Measured (cfg2 / cfg4-units B1): class-major 143 / 213 us,
//    interior first 167 / 115 us.
struct TileOrder {
  static constexpr int kMaxGroups = 16;
  int B, heads, q_row0, num_tiles;  // B: maps per head (pair mode: map pairs per head)
  int pair;                         // tc::pair_mode: tile = maps (b, h) and (b + 1, h), b even
  int n_rg, n_cg;
  int int_rg, int_cg;  // the interior row / column group (-1: none)
  int class_major;     // plain class-major order (class, head, batch, row, column)
  int rg_start[kMaxGroups], rg_count[kMaxGroups], cg_start[kMaxGroups], cg_count[kMaxGroups];
  struct Tile {
    int bh, i0, j0, cls;
  };
  __device__ __forceinline__ Tile make(int a, int b, int h, int bb, int rem) const {
    Tile x;
    x.bh = pair ? 2 * bb * heads + h : bb * heads + h;  // (pair mode: member 0)
    x.i0 = q_row0 + (rg_start[a] + rem / cg_count[b]) * tc::kTQH;
    x.j0 = (cg_start[b] + rem % cg_count[b]) * tc::kTQW;
    x.cls = a * n_cg + b;
    return x;
  }
  __device__ __forceinline__ Tile decode(int t) const {
    if (class_major) {
      for (int a = 0; a < n_rg; ++a)
        for (int b = 0; b < n_cg; ++b) {
          const int per_map = rg_count[a] * cg_count[b];
          const int cnt = B * heads * per_map;
          if (t < cnt) {
            const int hb = t / per_map, rem = t - hb * per_map;
            const int h = hb / B;
            return make(a, b, h, hb - h * B, rem);
          }
          t -= cnt;
        }
    }
    if (int_rg >= 0 && int_cg >= 0) {
      const int per_map = rg_count[int_rg] * cg_count[int_cg];
      const int cnt = B * heads * per_map;
      if (t < cnt) {
        const int hb = t / per_map, rem = t - hb * per_map;
        const int h = hb / B;
        return make(int_rg, int_cg, h, hb - h * B, rem);
      }
      t -= cnt;
    }
    int border = 0;  // border tiles per head (all batches)
    for (int a = 0; a < n_rg; ++a)
      for (int b = 0; b < n_cg; ++b)
        if (a != int_rg || b != int_cg) border += B * rg_count[a] * cg_count[b];
    const int h = t / border;
    t -= h * border;
    for (int a = 0; a < n_rg; ++a)
      for (int b = 0; b < n_cg; ++b) {
        if (a == int_rg && b == int_cg) continue;
        const int per_map = rg_count[a] * cg_count[b];
        const int cnt = B * per_map;
        if (t < cnt) {
          const int bb = t / per_map;
          return make(a, b, h, bb, t - bb * per_map);
        }
        t -= cnt;
      }
    return make(0, 0, 0, 0, 0);
  }
};

// Build the class-grouped order for query tiles of a (band of a) map.
TileOrder make_tile_order(const Geo &g, int L);

// B1's contiguous tile ranges: CTA c takes tiles [start[c], start[c + 1]) of the order.  A CTA whose
// range crosses from one (class, head) segment into the next pays a dRPB flush (and on a head
// change a partial-table commit and a bias-table rebuild): traced at ~1.2-1.6 tiles' time each,
// and border-class tiles run slower too (profiles/r02_b1_balance.txt).  The ranges are chosen so
// that tiles + kSwitchCost x switches is balanced across CTAs instead of the tile count alone;
// kSwitchCost = 3 tiles measured best (1.5: B1 cfg2 126.3 us, 3: 124.1 us, 5: 124.2 us).
constexpr int kMaxB1Ctas = 256;
struct B1Ranges {
  int start[kMaxB1Ctas + 1];
};
void make_b1_ranges(const TileOrder &o, const Geo &g, int grid, B1Ranges *r);

struct BwdQParams {
  int heads, H, W, q_rows, q_row0, kv_row0;
  int num_tiles;
  TileOrder order;
  float scale;
  const float *rpb;
  const float *lse;
  const __nv_bfloat16 *out, *dout;
  __nv_bfloat16 *dq;
  float *D;          // [B*heads*q_rows*W] written
  float *drpb_part;  // [grid][heads][TT*TT] partial tables (null if no rpb)
  int *b2_tile_counter;  // zeroed by this kernel for B2's dynamic tile scheduler
  B1Ranges ranges;       // per-CTA tile ranges (make_b1_ranges)
  long long *trace;  // debug timeline (na2d_debug_set_trace) or null
};

int dq_grid(const Geo &g);
int max_query_halo_width(const Geo &g, bool shift);
bool tc_dkdv_supported(const Geo &g);
// drpb_part (may be null): B1's per-CTA dRPB tables [part_ctas][heads][(2L-1)^2]; B2 sums them
// into drpb (fixed CTA order, one warp per cell) before its own work
cudaError_t tc_backward_dkdv(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                             const float *lse, const void *dout, const float *D, void *dk, void *dv,
                             const float *drpb_part, int part_ctas, float *drpb, int *tile_counter,
                             cudaStream_t st);
cudaError_t tc_backward_dq(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                           const void *out, const float *lse, const void *dout, void *dq, float *drpb, float *D,
                           float *part, int *b2_tile_counter, cudaStream_t st);

}  // namespace na2d
