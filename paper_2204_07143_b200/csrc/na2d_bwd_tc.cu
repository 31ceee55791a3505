// na2d_bwd_tc.cu -- tcgen05 backward driver: kernel B1 (dQ, D, dRPB; na2d_bwd_dq_tc.cu) then
// dK/dV, plus the class-grouped tile order shared by the backward kernels.
#include "na2d_internal.cuh"
#include "na2d_tc.cuh"
#include "na2d_tc_bwd.cuh"
#include "na2d_tmap.cuh"

namespace na2d {

TileOrder make_tile_order(const Geo &g, int L) {
  TileOrder o{};
  o.pair = tc::pair_mode(g.B, g.H, g.W, g.q_row0, g.q_rows, g.kv_row0, g.kv_rows);
  o.B = o.pair ? g.B / 2 : g.B;
  o.heads = g.heads;
  o.q_row0 = g.q_row0;
  const int ns = (L - 1) / 2, q_end = g.q_row0 + g.q_rows;
  const int tiles_h = (g.q_rows + tc::kTQH - 1) / tc::kTQH, tiles_w = (g.W + tc::kTQW - 1) / tc::kTQW;
  // groups of tile rows (columns): one run of interior tiles, every other tile alone; returns the count
  // and the interior group's index (-1 if none)
  auto groups = [&](int n, int tile, int first, int end, int axis, int *start, int *count, int *interior_group) {
    int ng = 0;
    int tr = 0;
    *interior_group = -1;
    while (tr < n) {
      auto interior = [&](int t) {
        const int a = first + t * tile, b = a + tile - 1;
        return L < axis && b < end && a - ns >= 0 && b <= axis - 1 - ns;
      };
      if (interior(tr)) {
        int e = tr;
        while (e < n && interior(e)) ++e;
        start[ng] = tr;
        count[ng] = e - tr;
        *interior_group = ng;
        tr = e;
      } else {
        start[ng] = tr;
        count[ng] = 1;
        ++tr;
      }
      ++ng;
    }
    return ng;
  };
  o.n_rg = groups(tiles_h, tc::kTQH, g.q_row0, q_end, g.H, o.rg_start, o.rg_count, &o.int_rg);
  o.n_cg = groups(tiles_w, tc::kTQW, 0, g.W, g.W, o.cg_start, o.cg_count, &o.int_cg);
  o.num_tiles = o.B * g.heads * tiles_h * tiles_w;
  // class-major unless the smallest class holds so few tiles per head that a CTA's contiguous share
  // would cross more than ~4 heads there
  int min_class = 1 << 30;
  for (int a = 0; a < o.n_rg; ++a)
    for (int b = 0; b < o.n_cg; ++b) {
      const int c = o.B * o.rg_count[a] * o.cg_count[b];
      min_class = c < min_class ? c : min_class;
    }
  const int grid = o.num_tiles < tc::num_sms() ? o.num_tiles : tc::num_sms();
  o.class_major = 4 * min_class * grid >= o.num_tiles ? 1 : 0;
  return o;
}

void make_b1_ranges(const TileOrder &o, const Geo &g, int grid, B1Ranges *r) {
  // (class, head) segments of the visiting order (TileOrder::decode), as lengths in tiles
  int seg[2 * TileOrder::kMaxGroups * TileOrder::kMaxGroups * 64];
  int ns = 0;
  const int cap = (int)(sizeof(seg) / sizeof(seg[0]));
  auto per_map = [&](int a, int b) { return o.rg_count[a] * o.cg_count[b]; };
  auto push = [&](int n) {
    if (n > 0 && ns < cap) seg[ns++] = n;
  };
  bool ok = (long)o.n_rg * o.n_cg * g.heads <= cap;
  if (ok && o.class_major) {
    for (int a = 0; a < o.n_rg; ++a)
      for (int b = 0; b < o.n_cg; ++b)
        for (int h = 0; h < g.heads; ++h) push(o.B * per_map(a, b));
  } else if (ok) {
    if (o.int_rg >= 0 && o.int_cg >= 0)
      for (int h = 0; h < g.heads; ++h) push(o.B * per_map(o.int_rg, o.int_cg));
    for (int h = 0; h < g.heads; ++h)
      for (int a = 0; a < o.n_rg; ++a)
        for (int b = 0; b < o.n_cg; ++b)
          if (a != o.int_rg || b != o.int_cg) push(o.B * per_map(a, b));
  }
  const int n = o.num_tiles;
  long sum = 0;
  for (int i = 0; i < ns; ++i) sum += seg[i];
  if (!ok || sum != n || grid <= 1) {
    for (int c = 0; c <= grid; ++c) r->start[c] = (int)((long)n * c / grid);
    return;
  }
  // cost of the order as a line: 4 per tile (quarter-tile units) plus kSwitchCost where a segment
  // starts; CTA c starts at the first tile whose cumulative cost reaches c / grid of the total (a
  // target that falls on a switch lands on the segment's first tile, so that CTA pays no switch)
#ifndef NA2D_B1_SWITCH_COST
#define NA2D_B1_SWITCH_COST 12
#endif
  constexpr long kSwitchCost = NA2D_B1_SWITCH_COST;  // quarter tiles: 3 tiles (1.5 measured 2 us slower at cfg2)
  const long total = 4L * n + kSwitchCost * (ns - 1);
  r->start[0] = 0;
  int c = 1;
  long pre = 0;  // cumulative cost before the current segment's first tile (switch included)
  int s0 = 0;
  for (int i = 0; i < ns && c < grid; ++i) {
    if (i > 0) pre += kSwitchCost;
    const long hi = pre + 4L * seg[i];
    while (c < grid) {
      const long tau = (total * c + grid - 1) / grid;
      if (tau > hi) break;
      const long k = tau <= pre ? 0 : (tau - pre + 3) / 4;  // tiles of this segment before CTA c
      int st = s0 + (int)k;
      if (st < r->start[c - 1]) st = r->start[c - 1];
      r->start[c++] = st;
    }
    pre = hi;
    s0 += seg[i];
  }
  while (c < grid) r->start[c++] = n;
  r->start[grid] = n;
}

bool tc_backward_supported(const Geo &g) {
  if (!((g.dtype == NA2D_BF16 || g.dtype == NA2D_F16) && (g.d == 16 || g.d == 32 || g.d == 64) && (g.L == 3 || g.L == 5 || g.L == 7) &&
        tmap_available()))
    return false;
  const TileOrder o = make_tile_order(g, g.L);
  return o.n_rg <= TileOrder::kMaxGroups && o.n_cg <= TileOrder::kMaxGroups && tc_dkdv_supported(g);
}

size_t tc_backward_scratch_bytes(const Geo &g) {
  const int TT = 2 * g.L - 1;
  return sizeof(float) * (size_t)dq_grid(g) * g.heads * TT * TT + 16;  // + B2 tile counter
}

cudaError_t tc_backward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                        const void *out, const float *lse, const void *dout, void *dq, void *dk, void *dv,
                        float *drpb, float *D, void *scratch, cudaStream_t st) {
  const int TT = 2 * g.L - 1;
  int *counter = (int *)((char *)scratch + sizeof(float) * (size_t)dq_grid(g) * g.heads * TT * TT);
  cudaError_t e = tc_backward_dq(g, q, k, v, rpb, out, lse, dout, dq, drpb, D, (float *)scratch, counter, st);
  if (e != cudaSuccess) return e;
  return tc_backward_dkdv(g, q, k, v, rpb, lse, dout, D, dk, dv, rpb ? (const float *)scratch : nullptr,
                          dq_grid(g), drpb, counter, st);
}

int tc_launches(const Geo &g, int which) {
  if (which == 0) return 1;
  return 2;  // B1 (dQ, D, per-CTA dRPB partials), B2 (dK, dV, and the dRPB partial reduction)
}

}  // namespace na2d
