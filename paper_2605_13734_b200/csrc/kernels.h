// Kernel argument blocks and launcher declarations.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "kvc_internal.h"

namespace kvc {

struct EncArgs {
  Geo g;
  const void* kv;
  uint8_t* packed;  // packed width streams (the payload for codec none)
  uint8_t* meta;
  const HeadEntry* heads;
  const StreamTab* st;
  uint32_t* status;
  double hk, hc;    // hadamard: 2^896 * RN64(1/sqrt(C)), RN64(sqrt(C))
  float rl[9];      // RN32(1 / (2^w - 1))
  int32_t* fix_rows;    // fused Hadamard encode: rows left to the exact fixup pass
  uint32_t* fix_count;
  uint32_t* fix1_bits;  // certified float32 Hadamard encode: one bit per token row for the float64 pass (or null: fp64 only)
  float hr32;           // RN32(1 / RN64(sqrt C))
  // paged input (kvc_encode_paged): row (lh, t) of kv at out_index(a, lh, t, 0)
  int paged;
  const int32_t* block_table;
  int64_t page_tokens, layer_stride;
};

struct DecArgs {
  Geo g;
  const uint8_t* packed;
  const uint8_t* meta;
  const HeadEntry* heads;
  const StreamTab* st;
  void* out;
  uint32_t* status;
  double hk, hc;
  int paged;
  const int32_t* block_table;
  int64_t page_tokens, layer_stride;
};

#ifdef __CUDACC__
// codec none reads the caller's payload directly: when the length check that
// runs first (k_check_payload) rejected it, the decode kernels read nothing
__device__ __forceinline__ bool payload_rejected(const DecArgs& a) {
  return a.g.codec == C_NONE && (*reinterpret_cast<const volatile uint32_t*>(a.status) & KVC_FLAG_CODEC);
}
#endif

struct ClassBits {
  uint8_t b[4096];
};

// Codec stage (operates on packed width streams).
struct CodecArgs {
  Geo g;
  const StreamTab* st;
  const uint8_t* packed_in;   // encode: packed streams
  uint8_t* packed_out;        // decode: packed streams
  const uint8_t* payload_in;  // decode: payload
  uint8_t* payload_out;       // encode: payload
  uint64_t* offsets;          // nblocks + 1
  const uint64_t* offsets_in;
  uint8_t* slots;             // encode scratch, slot_bytes per block
  uint64_t* sizes;            // encode scratch, per block
  void* scan_tmp;
  size_t scan_bytes;
  int64_t slot_bytes;
  int64_t max_blocks;
  int64_t payload_bytes;      // decode: caller's payload length
  uint32_t* status;
  const uint32_t* recip;      // [9][2048] reciprocal tables (rc_tables.cuh)
};

// Fused quantize + range-code kernels (fused_rc.cu): one thread per codec
// block reads bf16 KV and writes its range-coded block (encode), or decodes a
// block straight to KV (decode); no packed-symbol round trip through HBM.
struct FusedArgs {
  Geo g;
  const void* kv;              // encode input, (L,H,T,C) bf16, contiguous or paged (out_index)
  __half* scales;              // encode: metadata scales / zeros out
  __half* zeros;
  const __half* scales_in;     // decode: metadata in
  const __half* zeros_in;
  uint8_t* slots;              // encode: slot_bytes per block
  uint64_t* sizes;             // encode: per block (max_blocks + 1)
  int64_t slot_bytes, max_blocks;
  const uint8_t* payload_in;   // decode
  const uint64_t* offsets_in;
  int64_t payload_bytes;
  void* out;                   // decode output (contiguous or paged)
  int paged;                   // encode: kv is paged; decode: out is paged
  const int32_t* block_table;
  int64_t page_tokens, layer_stride;
  uint32_t* status;
  const uint32_t* recip;
  float rl[9];
};

// cudaFuncSetAttribute is per device: raise a kernel's dynamic shared memory
// limit once per (kernel, device) of the process
template <auto K>
inline void set_max_dyn_smem(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
}

// element index of (lh, t, c) in the KV cache: contiguous (L,H,T,C), or the
// paged layout [pages, page_tokens, H, C] per layer (the decode output, and
// the encode input of kvc_encode_paged)
template <class A>
__device__ __forceinline__ int64_t out_index(const A& a, int64_t lh, int64_t t, int64_t c) {
  if (!a.paged) return (lh * a.g.T + t) * a.g.C + c;
  const int64_t l = lh / a.g.H, h = lh - l * a.g.H;
  const int64_t page = a.block_table[t / a.page_tokens];
  return l * a.layer_stride + (page * a.page_tokens + t % a.page_tokens) * a.g.H * a.g.C + h * a.g.C + c;
}

cudaError_t launch_setup(const Geo& g, const uint8_t* meta, StreamTab* st, HeadEntry* heads, cudaStream_t s);
cudaError_t launch_write_classmap(const ClassBits& cb, uint8_t* dst, int nbytes, cudaStream_t s);
cudaError_t launch_affine_calibrate(const EncArgs& a, cudaStream_t s);
cudaError_t launch_encode_generic(const EncArgs& a, cudaStream_t s);
cudaError_t launch_encode_fixup(const EncArgs& a, cudaStream_t s);
cudaError_t launch_decode_generic(const DecArgs& a, cudaStream_t s);

// fast head_dim-128 per-token kernels (fast128.cu); return false if not applicable
bool fast128_applicable(const Geo& g);
cudaError_t launch_encode_fast128(const EncArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_decode_fast128(const DecArgs& a, int sm_count, cudaStream_t s);

// per-channel (q=uchan) head_dim-128 kernels (uchan128.cu)
bool uchan128_applicable(const Geo& g);
cudaError_t launch_encode_uchan128(const EncArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_decode_uchan128(const DecArgs& a, int sm_count, cudaStream_t s);

// delta decode, head_dim 128, exact sequential fp64 cumsum (delta128.cu)
bool delta128_applicable(const Geo& g);
int64_t delta128_ws_bytes(const Geo& g);
cudaError_t launch_decode_delta128(const DecArgs& a, void* ws, cudaStream_t s);

// small-alphabet range coder (rc_small.cu), widths 1..4
bool rc_small_supported(int w);
cudaError_t launch_rc_small_encode(const CodecArgs& a, int w, unsigned grid, cudaStream_t s);
cudaError_t launch_rc_small_decode(const CodecArgs& a, int w, unsigned grid, cudaStream_t s);

// large-alphabet range coder (rc_large.cu), widths 5..8
cudaError_t launch_rc_large_encode(const CodecArgs& a, int w, cudaStream_t s);
cudaError_t launch_rc_large_decode(const CodecArgs& a, int w, cudaStream_t s);

// codec stage (codec.cu)
size_t codec_scan_bytes(int64_t max_blocks);
cudaError_t launch_codec_encode(const CodecArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_codec_decode(const CodecArgs& a, int sm_count, cudaStream_t s);
// block offsets (exclusive scan of sizes) + gather of slots into the payload
cudaError_t launch_codec_finish(const CodecArgs& a, cudaStream_t s);
cudaError_t launch_check_payload(const CodecArgs& a, cudaStream_t s);
cudaError_t launch_copy_device_length(void* dst, const void* src, const uint64_t* nbytes_dev, int64_t max_bytes,
                                      cudaStream_t s);
cudaError_t launch_sq_error(const void* a, const void* b, int64_t n, int dtype, double* out, cudaStream_t s);
cudaError_t launch_sq_error_partials(const void* a, const void* b, int64_t n, int dtype, double* partials,
                                     int64_t npartials, cudaStream_t s);
cudaError_t launch_block_crc32(const uint8_t* payload, const uint64_t* offsets, int64_t nblocks, uint32_t* crc,
                               cudaStream_t s);

// fused quantize + range code (fused_rc.cu)
bool fused_rc_applicable(const Geo& g);
cudaError_t launch_fused_rc_encode(const FusedArgs& a, cudaStream_t s);
cudaError_t launch_fused_rc_decode(const FusedArgs& a, cudaStream_t s);

}  // namespace kvc
