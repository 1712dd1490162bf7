// Per-launch event timing for bench.py / the CUDA-event StageTimer.
#include "profile.h"

#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "kvc.h"

namespace kvc {
namespace {

std::atomic<int> g_on{0};

struct Rec {
  const char* name;
  cudaEvent_t a, b;
};

struct Pool {
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> spare;
  cudaEvent_t get() {
    if (!spare.empty()) {
      cudaEvent_t e = spare.back();
      spare.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

thread_local Pool t_pool;

}  // namespace

bool profiling() { return g_on.load(std::memory_order_relaxed) != 0; }

int prof_begin(const char* name, cudaStream_t s) {
  if (!profiling()) return -1;
  Rec r;
  r.name = name;
  r.a = t_pool.get();
  r.b = t_pool.get();
  cudaEventRecord(r.a, s);
  t_pool.recs.push_back(r);
  return (int)t_pool.recs.size() - 1;
}

void prof_end(int idx, cudaStream_t s) {
  if (idx < 0 || idx >= (int)t_pool.recs.size()) return;
  cudaEventRecord(t_pool.recs[idx].b, s);
}

}  // namespace kvc

extern "C" int kvc_profile_enable(int on) {
  kvc::g_on.store(on ? 1 : 0);
  return KVC_OK;
}

extern "C" int kvc_profile_collect(char* names, int64_t names_cap, double* ms, int64_t* launches, int cap) {
  using namespace kvc;
  std::vector<std::string> keys;
  std::vector<double> acc;
  std::vector<int64_t> cnt;
  for (auto& r : t_pool.recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t k = 0;
    for (; k < keys.size(); ++k)
      if (keys[k] == r.name) break;
    if (k == keys.size()) {
      keys.push_back(r.name);
      acc.push_back(0.0);
      cnt.push_back(0);
    }
    acc[k] += t;
    cnt[k] += 1;
    t_pool.spare.push_back(r.a);
    t_pool.spare.push_back(r.b);
  }
  t_pool.recs.clear();
  int n = (int)keys.size() < cap ? (int)keys.size() : cap;
  int64_t pos = 0;
  for (int i = 0; i < n; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = cnt[i];
    if (names) {
      int64_t len = (int64_t)keys[i].size() + 1;
      if (pos + len <= names_cap) {
        memcpy(names + pos, keys[i].c_str(), (size_t)len);
        pos += len;
      }
    }
  }
  cudaGetLastError();
  return n;
}
