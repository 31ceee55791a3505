// na2d_tc_common.cu -- host helpers shared by the tcgen05 kernels.
#include <stdlib.h>

#include <mutex>
#include <set>
#include <utility>

#include "na2d_tc_common.cuh"

namespace na2d {
namespace tc {

// Per device (one process may drive several GPUs): SM count, and which kernels already have their
// dynamic shared-memory limit raised (cudaFuncSetAttribute applies to the current device only).
namespace {
std::mutex g_mu;
std::set<std::pair<const void *, int>> g_attr_done;
int g_sms[64] = {};
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

int num_sms() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return 148;
  if (g_sms[dev] <= 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

cudaError_t ensure_smem_attr(const void *func, int smem_bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_attr_done.count({func, dev})) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e == cudaSuccess) g_attr_done.insert({func, dev});
  return e;
}

bool pair_mode(int B, int H, int W, int q_row0, int q_rows, int kv_row0, int kv_rows) {
  static const bool off = [] {
    const char *e = getenv("NA2D_NO_PAIR");
    return e && e[0] == '1';
  }();
  return !off && B >= 2 && B % 2 == 0 && H <= kTQH && W <= kTQW / 2 && q_row0 == 0 && q_rows == H && kv_row0 == 0 &&
         kv_rows == H;
}

}  // namespace tc
}  // namespace na2d
