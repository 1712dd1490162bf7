// Per-position reciprocal tables for the range coders.
//
// Before the first model halving the total at symbol i is A + 32 i
// (codecs.py:227-232), identical for every block; recip(A)[i] =
// floor(2^32 / (A + 32 i)) turns `range // total` into a multiply plus one
// correction.  One table per alphabet size (A = 2..256), built once per
// device, read through the read-only path with a warp-uniform index.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kvc {

constexpr int kRecipLen = 2048;  // >= ceil((65536 - A) / 32) for every A >= 2

// Build the tables on the current device once (host-computed, synchronous
// copy + device synchronize; a lock + flag test afterwards).  kvc_plan_create
// calls it for entropy plans; the launch paths call it again as a guard.
cudaError_t ensure_recip_tables();
// device pointer to the [9][kRecipLen] table (row w = alphabet 2^w)
const uint32_t* recip_tables();
// rows w = 1..4 / 5..8 into the coders' __constant__ copies (synchronous)
cudaError_t upload_fused_recip(const uint32_t* rows_1_to_4);
cudaError_t upload_large_recip(const uint32_t* rows_5_to_8);

__device__ __forceinline__ uint32_t div_recip(uint32_t n, uint32_t d, uint32_t m) {
  // floor(n / d) given m = floor(2^32 / d): the product estimate is q or q-1
  // (PTX: the compiler's form of the correction costs two more instructions)
  uint32_t q;
  asm("{\n\t.reg .u32 r, nd;\n\t.reg .pred p;\n\t"
      "mul.hi.u32 %0, %1, %3;\n\tneg.s32 nd, %2;\n\tmad.lo.u32 r, %0, nd, %1;\n\t"
      "setp.ge.u32 p, r, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
      : "=&r"(q)
      : "r"(n), "r"(d), "r"(m));
  return q;
}

}  // namespace kvc
