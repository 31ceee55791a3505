// Temporary: tensor-core backward not yet built; dispatcher uses the SIMT backward kernels.
#include "na2d_tc.cuh"

namespace na2d {
bool tc_backward_supported(const Geo &) { return false; }
size_t tc_backward_scratch_bytes(const Geo &) { return 0; }
cudaError_t tc_backward(const Geo &, const void *, const void *, const void *, const float *, const void *,
                        const float *, const void *, void *, void *, void *, float *, float *, void *,
                        cudaStream_t) { return cudaErrorNotSupported; }
int tc_launches(const Geo &, int which) { return which == 0 ? 1 : 0; }
}  // namespace na2d
