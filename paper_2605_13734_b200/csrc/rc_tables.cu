// Reciprocal tables for the range coders (see rc_tables.cuh).
//
// The tables are computed on the host and copied synchronously (then a
// device synchronize) the first time a plan with an entropy codec is created
// on a device, so no coder launched on any stream -- or captured into a CUDA
// graph -- can read them before they are complete.  The launch paths call
// ensure_recip_tables() again as a guard for plans created while another
// device was current; it is a lock + flag test once the tables exist.
#include <mutex>
#include <vector>

#include "kernels.h"
#include "rc_tables.cuh"

namespace kvc {
namespace {

__device__ uint32_t g_recip[9][kRecipLen];

std::mutex g_mu;
bool g_ready[64];

const std::vector<uint32_t>& host_table() {
  static std::vector<uint32_t> t;
  static std::once_flag once;
  std::call_once(once, [] {
    t.assign((size_t)9 * kRecipLen, 0u);
    for (int w = 1; w <= 8; ++w)
      for (int i = 0; i < kRecipLen; ++i)
        t[(size_t)w * kRecipLen + i] = (uint32_t)(0x100000000ull / (uint64_t)((1u << w) + 32u * (uint32_t)i));
  });
  return t;
}

}  // namespace

cudaError_t ensure_recip_tables() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev >= 0 && dev < 64 && g_ready[dev]) return cudaSuccess;
  const std::vector<uint32_t>& h = host_table();
  if ((e = cudaMemcpyToSymbol(g_recip, h.data(), sizeof(g_recip))) != cudaSuccess) return e;
  if ((e = upload_fused_recip(h.data() + kRecipLen)) != cudaSuccess) return e;      // rows w = 1..4
  if ((e = upload_large_recip(h.data() + 5 * kRecipLen)) != cudaSuccess) return e;  // rows w = 5..8
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
  if (dev >= 0 && dev < 64) g_ready[dev] = true;
  return cudaSuccess;
}

const uint32_t* recip_tables() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_recip);
  return reinterpret_cast<const uint32_t*>(p);
}

}  // namespace kvc
