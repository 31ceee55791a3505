// na2d_tc.cuh -- tensor-core (tcgen05 + TMEM + TMA) NA2D kernels for sm_100a.
#pragma once

#include "na2d_internal.cuh"

namespace na2d {

bool tc_forward_supported(const Geo &g);
bool tc_backward_supported(const Geo &g);
cudaError_t tc_forward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb, void *out,
                       float *lse, cudaStream_t st);
size_t tc_backward_scratch_bytes(const Geo &g);
cudaError_t tc_backward(const Geo &g, const void *q, const void *k, const void *v, const float *rpb,
                        const void *out, const float *lse, const void *dout, void *dq, void *dk, void *dv,
                        float *drpb, float *D, void *scratch, cudaStream_t st);
int tc_launches(const Geo &g, int which);

}  // namespace na2d
