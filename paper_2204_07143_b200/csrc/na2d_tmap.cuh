// na2d_tmap.cuh -- TMA tensor-map construction (cuTensorMapEncodeTiled through the runtime's
// driver entry point, so libna2d needs no link-time libcuda).
#pragma once

#include <cuda.h>

namespace na2d {

// True if the driver exposes cuTensorMapEncodeTiled.
bool tmap_available();

// 4-D bf16 tensor [outer][rows][W][dim] (dim innermost, contiguous) with a box of
// {dim, box_w, box_h, 1} elements; dim in {16, 32, 64}, i.e. rows of 32 / 64 / 128 bytes with the
// swizzle of that width (one swizzle atom per row: the UMMA K-major / MN-major operand layouts).
// Out-of-bounds box elements are zero-filled by the hardware.  Returns false on failure.
bool make_tmap_bf16_4d(CUtensorMap *m, const void *base, int dim, int W, int rows, int outer, int box_w, int box_h);
// the same for a 16-bit element type: fp16 if f16, else bf16
bool make_tmap_e16_4d(bool f16, CUtensorMap *m, const void *base, int dim, int W, int rows, int outer, int box_w,
                      int box_h);

// Pair layout for small maps (tc::pair_mode): the maps bh and bh + heads side by side.  5-D view
// {dim, col, member, row, bh} with a box of {dim, box_w, 2, box_h, 1}: shared memory receives
// [row][member][col] rows, i.e. a halo of pitch 2 * box_w keys with member m at column m * box_w
// (columns >= W zero-filled).  The caller must only address pairs whose member 1 exists.
bool make_tmap_e16_pair(bool f16, CUtensorMap *m, const void *base, int dim, int W, int rows, int heads, int outer,
                        int box_w, int box_h);

}  // namespace na2d

namespace na2d {
// 3-D fp32 tensor [outer][rows][W] (W innermost) with a box of {box_w, box_h, 1}, no swizzle
// (LSE / D halos).  box_w * 4 must be a multiple of 16 bytes.
bool make_tmap_f32_3d(CUtensorMap *m, const void *base, int W, int rows, int outer, int box_w, int box_h);
}  // namespace na2d
