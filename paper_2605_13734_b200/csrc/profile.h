// Opt-in per-launch CUDA-event timing (kvc_profile_enable / _collect).
#pragma once
#include <cuda_runtime.h>

namespace kvc {

bool profiling();
// returns an index to pass to prof_end, or -1 when profiling is off
int prof_begin(const char* name, cudaStream_t s);
void prof_end(int idx, cudaStream_t s);

struct ProfScope {
  int idx;
  cudaStream_t s;
  ProfScope(const char* name, cudaStream_t st) : idx(prof_begin(name, st)), s(st) {}
  ~ProfScope() { prof_end(idx, s); }
};

}  // namespace kvc
