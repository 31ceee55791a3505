// na2d_tc_common.cu -- host helpers shared by the tcgen05 kernels.
#include <mutex>

#include "na2d_tc_common.cuh"

namespace na2d {
namespace tc {

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


}  // namespace tc
}  // namespace na2d
