// na2d_profile.cu -- event pool behind na2d_profile_enable / na2d_profile_read.
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "na2d.h"
#include "na2d_profile.cuh"

namespace na2d {
namespace {

struct Rec {
  const char *name;
  cudaEvent_t a, b;
};

std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void recycle_all() {
  for (auto &r : g_recs) {
    g_pool.push_back(r.a);
    if (r.b) g_pool.push_back(r.b);
  }
  g_recs.clear();
}

}  // namespace

void prof_begin(const char *name, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  Rec r{name, get_event(), nullptr};
  cudaEventRecord(r.a, st);
  g_recs.push_back(r);
}

void prof_end(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on || g_recs.empty() || g_recs.back().b) return;
  g_recs.back().b = get_event();
  cudaEventRecord(g_recs.back().b, st);
}

}  // namespace na2d

using namespace na2d;

namespace na2d {
static void *g_trace = nullptr;
void *debug_trace_buffer() { return g_trace; }
}  // namespace na2d

extern "C" na2d_status na2d_debug_set_trace(void *device_buffer) {
  g_trace = device_buffer;
  return NA2D_OK;
}

extern "C" na2d_status na2d_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  recycle_all();
  g_on = on != 0;
  return NA2D_OK;
}

extern "C" int na2d_profile_read(char *names_out, size_t name_cap, float *total_ms, int *counts, int max_entries) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<std::string> names;
  std::vector<double> tot;
  std::vector<int> cnt;
  for (auto &r : g_recs) {
    if (!r.b) continue;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return -1;
    size_t i = 0;
    while (i < names.size() && names[i] != r.name) ++i;
    if (i == names.size()) {
      names.push_back(r.name);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[i] += ms;
    cnt[i] += 1;
  }
  size_t off = 0;
  int n = 0;
  for (size_t i = 0; i < names.size() && n < max_entries; ++i, ++n) {
    if (names_out) {
      if (off + names[i].size() + 1 > name_cap) return -1;
      memcpy(names_out + off, names[i].c_str(), names[i].size() + 1);
      off += names[i].size() + 1;
    }
    if (total_ms) total_ms[n] = (float)tot[i];
    if (counts) counts[n] = cnt[i];
  }
  return (int)names.size();
}
