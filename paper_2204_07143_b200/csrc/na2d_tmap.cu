// na2d_tmap.cu -- see na2d_tmap.cuh.
#include <cuda_runtime.h>

#include <mutex>

#include "na2d_tmap.cuh"

namespace na2d {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

// cuTensorMapEncodeTiled (driver API) needs a current context.  A host thread that has made no
// runtime call that binds one yet (e.g. torch's autograd worker thread, when the kernels'
// one-time attribute setup already ran on another thread) gets CUDA_ERROR_INVALID_CONTEXT:
// bind the primary context of the thread's current device (cudaFree(nullptr) does exactly that).
bool bind_context() { return cudaFree(nullptr) == cudaSuccess; }

}  // namespace

bool tmap_available() { return encode_fn() != nullptr; }

bool make_tmap_bf16_4d(CUtensorMap *m, const void *base, int dim, int W, int rows, int outer, int box_w, int box_h) {
  return make_tmap_e16_4d(false, m, base, dim, W, rows, outer, box_w, box_h);
}

bool make_tmap_e16_4d(bool f16, CUtensorMap *m, const void *base, int dim, int W, int rows, int outer, int box_w,
                      int box_h) {
  EncodeFn fn = encode_fn();
  // rows of dim 16-bit elements: 32 / 64 / 128 bytes, one swizzle atom wide (the UMMA operand layouts)
  if (!fn || (dim != 16 && dim != 32 && dim != 64)) return false;
  const CUtensorMapSwizzle sw = dim == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : dim == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                      : CU_TENSOR_MAP_SWIZZLE_128B;
  const cuuint64_t gdim[4] = {(cuuint64_t)dim, (cuuint64_t)W, (cuuint64_t)rows, (cuuint64_t)outer};
  const cuuint64_t gstride[3] = {(cuuint64_t)dim * 2, (cuuint64_t)W * dim * 2, (cuuint64_t)rows * W * dim * 2};
  const cuuint32_t box[4] = {(cuuint32_t)dim, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  const cuuint32_t estride[4] = {1, 1, 1, 1};
  auto encode = [&] {
    return fn(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base),
              gdim, gstride, box, estride,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUresult r = encode();
  if (r == CUDA_ERROR_INVALID_CONTEXT && bind_context()) r = encode();
  return r == CUDA_SUCCESS;
}

bool make_tmap_e16_pair(bool f16, CUtensorMap *m, const void *base, int dim, int W, int rows, int heads, int outer,
                        int box_w, int box_h) {
  EncodeFn fn = encode_fn();
  if (!fn || (dim != 16 && dim != 32 && dim != 64)) return false;
  const CUtensorMapSwizzle sw = dim == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : dim == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                      : CU_TENSOR_MAP_SWIZZLE_128B;
  const cuuint64_t map = (cuuint64_t)rows * W * dim * 2;  // bytes per (b, h) map
  // dims {dim, col, member, row, bh}: member 1 of the pair at bh is the map bh + heads
  const cuuint64_t gdim[5] = {(cuuint64_t)dim, (cuuint64_t)W, 2, (cuuint64_t)rows, (cuuint64_t)outer};
  const cuuint64_t gstride[4] = {(cuuint64_t)dim * 2, map * heads, (cuuint64_t)W * dim * 2, map};
  const cuuint32_t box[5] = {(cuuint32_t)dim, (cuuint32_t)box_w, 2, (cuuint32_t)box_h, 1};
  const cuuint32_t estride[5] = {1, 1, 1, 1, 1};
  auto encode = [&] {
    return fn(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(base),
              gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUresult r = encode();
  if (r == CUDA_ERROR_INVALID_CONTEXT && bind_context()) r = encode();
  return r == CUDA_SUCCESS;
}

bool make_tmap_f32_3d(CUtensorMap *m, const void *base, int W, int rows, int outer, int box_w, int box_h) {
  EncodeFn fn = encode_fn();
  if (!fn || (box_w * 4) % 16 != 0 || ((size_t)W * 4) % 16 != 0) return false;
  const cuuint64_t gdim[3] = {(cuuint64_t)W, (cuuint64_t)rows, (cuuint64_t)outer};
  const cuuint64_t gstride[2] = {(cuuint64_t)W * 4, (cuuint64_t)rows * W * 4};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  const cuuint32_t estride[3] = {1, 1, 1};
  auto encode = [&] {
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(base), gdim, gstride, box, estride,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUresult r = encode();
  if (r == CUDA_ERROR_INVALID_CONTEXT && bind_context()) r = encode();
  return r == CUDA_SUCCESS;
}

}  // namespace na2d
