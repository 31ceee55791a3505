// Temporary: tensor-core kernels not yet built; dispatcher uses the SIMT kernels.
#include "na2d_tc.cuh"

namespace na2d {
bool tc_forward_supported(const Geo &) { return false; }
bool tc_backward_supported(const Geo &) { return false; }
cudaError_t tc_forward(const Geo &, const void *, const void *, const void *, const float *, void *, float *,
                       cudaStream_t) { return cudaErrorNotSupported; }
size_t tc_backward_scratch_bytes(const Geo &) { return 0; }
cudaError_t tc_backward(const Geo &, const void *, const void *, const void *, const float *, const void *,
                        const float *, const void *, void *, void *, void *, float *, float *, void *,
                        cudaStream_t) { return cudaErrorNotSupported; }
int tc_launches(const Geo &, int) { return 0; }
}  // namespace na2d
