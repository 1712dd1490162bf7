// Reciprocal tables for the range coders (see rc_tables.cuh).
#include <mutex>

#include "rc_tables.cuh"

namespace kvc {
namespace {

__device__ uint32_t g_recip[9][kRecipLen];

__global__ void k_build_recip() {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kRecipLen) return;
  for (int w = 1; w <= 8; ++w) g_recip[w][i] = (uint32_t)(0x100000000ull / (uint64_t)((1u << w) + 32u * (uint32_t)i));
}

std::mutex g_mu;
bool g_built[64];

}  // namespace

const uint32_t* recip_tables(cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_recip);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev >= 0 && dev < 64 && !g_built[dev]) {
      k_build_recip<<<kRecipLen / 256, 256, 0, s>>>();
      g_built[dev] = true;
    }
  }
  return reinterpret_cast<const uint32_t*>(p);
}

}  // namespace kvc
