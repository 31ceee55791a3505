// na2d_profile.cuh -- optional CUDA-event bracketing of every kernel launch (bench.py roofline).
#pragma once

#include <cuda_runtime.h>

namespace na2d {
// Record the start of launch `name` on stream `st` (no-op unless profiling is enabled).
void prof_begin(const char *name, cudaStream_t st);
// Record the end of the most recent prof_begin on `st`.
void prof_end(cudaStream_t st);

struct ProfScope {
  cudaStream_t st;
  ProfScope(const char *name, cudaStream_t s) : st(s) { prof_begin(name, s); }
  ~ProfScope() { prof_end(st); }
};
}  // namespace na2d
