// Codec stage over packed width streams: dispatch of the block range coders
// (rc_small.cu: w <= 4, rc_large.cu: w >= 5), PackBits RLE, and the
// block-offset scan + gather.
//
// A width stream (codecs.py:339-345) is cut into blocks of g.block symbols;
// each block is coded independently with the reference's own algorithm so
// decoding is parallel (one thread per block):
//   entropy block = BE32(len) || range_encode(block, 1 << w)  (codecs.py:245-270, :310-317, :364-366)
//   rle block     = rle_encode(packed block bytes)             (codecs.py:112-152)
// Encode writes each block into a worst-case-sized scratch slot, then an
// exclusive scan of the sizes gives block_offsets and a gather kernel packs
// the slots into the payload.
#include <cub/device/device_scan.cuh>

#include "kernels.h"
#include "profile.h"
#include "rc_tables.cuh"

namespace kvc {

namespace {

// ----------------------------------------------------------------- RLE
__device__ void rle_encode_block(const uint8_t* src, int64_t n, uint8_t* slot, int64_t cap, uint64_t* size_out,
                                 uint32_t* status) {
  // greedy PackBits (codecs.py:112-152): runs >= 3 become (128+len-3, byte)
  // in chunks <= 130; everything else is literal in chunks <= 128.
  int64_t pos = 0;
  int64_t i = 0;
  int64_t lit = -1;
  auto emit_lit = [&](int64_t from, int64_t upto) {
    while (from < upto) {
      int64_t ch = upto - from < 128 ? upto - from : 128;
      if (pos + 1 + ch <= cap) {
        slot[pos] = (uint8_t)(ch - 1);
        for (int64_t k = 0; k < ch; ++k) slot[pos + 1 + k] = src[from + k];
      }
      pos += 1 + ch;
      from += ch;
    }
  };
  while (i < n) {
    const uint8_t v = src[i];
    int64_t j = i + 1;
    while (j < n && src[j] == v) ++j;
    int64_t run = j - i;
    if (run >= 3) {
      if (lit >= 0) {
        emit_lit(lit, i);
        lit = -1;
      }
      while (run >= 3) {
        int64_t ch = run < 130 ? run : 130;
        if (pos + 2 <= cap) {
          slot[pos] = (uint8_t)(128 + ch - 3);
          slot[pos + 1] = v;
        }
        pos += 2;
        run -= ch;
      }
      if (run) lit = j - run;
    } else if (lit < 0) {
      lit = i;
    }
    i = j;
  }
  if (lit >= 0) emit_lit(lit, n);
  if (pos > cap) {
    atomicOr(status, KVC_FLAG_CAPACITY);
    pos = 0;
  }
  *size_out = (uint64_t)pos;
}

__device__ __forceinline__ int block_stream(const StreamTab& st, int64_t b) {
  return (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
}

__global__ void __launch_bounds__(128) k_rle_encode(CodecArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > a.max_blocks) return;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) {
    a.sizes[b] = 0;
    return;
  }
  const int si = block_stream(st, b);
  const int w = st.w[si];
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int64_t n = min(a.g.block, st.count[si] - start);
  const uint8_t* src = a.packed_in + st.byte_off[si] + start * w / 8;
  rle_encode_block(src, (n * w + 7) / 8, a.slots + b * a.slot_bytes, a.slot_bytes, a.sizes + b, a.status);
}

__global__ void __launch_bounds__(128) k_rle_decode(CodecArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) return;
  const int si = block_stream(st, b);
  const int w = st.w[si];
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int64_t n = min(a.g.block, st.count[si] - start);
  const int64_t want = (n * w + 7) / 8;
  const uint64_t o0 = a.offsets_in[b], o1 = a.offsets_in[b + 1];
  if (o1 < o0 || (a.payload_bytes >= 0 && (int64_t)o1 > a.payload_bytes)) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  const uint8_t* in = a.payload_in + o0;
  const int64_t len = (int64_t)(o1 - o0);
  uint8_t* out = a.packed_out + st.byte_off[si] + start * w / 8;
  int64_t pos = 0, o = 0;
  bool bad = false;
  while (pos < len) {  // codecs.py:155-174
    uint32_t c = in[pos++];
    if (c < 128) {
      int64_t l = (int64_t)c + 1;
      if (pos + l > len || o + l > want) { bad = true; break; }
      for (int64_t k = 0; k < l; ++k) out[o + k] = in[pos + k];
      o += l;
      pos += l;
    } else {
      if (pos >= len) { bad = true; break; }
      int64_t l = (int64_t)c - 125;
      if (o + l > want) { bad = true; break; }
      const uint8_t v = in[pos++];
      for (int64_t k = 0; k < l; ++k) out[o + k] = v;
      o += l;
    }
  }
  if (bad || o != want) atomicOr(a.status, KVC_FLAG_CODEC);
}

// ---------------------------------------------------------- scan + gather
// one warp per block copies its slot bytes to payload[offsets[b]]: partial
// head / tail words byte by byte (they are shared with the neighbouring
// blocks), the aligned body as 32-bit words funnel-shifted out of the
// 16-byte-aligned slot
__global__ void __launch_bounds__(256) k_gather(CodecArgs a) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const StreamTab& st = *a.st;
  if (b >= st.nblocks) return;
  const uint64_t o0 = a.offsets[b], o1 = a.offsets[b + 1];
  const uint32_t len = (uint32_t)(o1 - o0);
  const uint8_t* src = a.slots + b * a.slot_bytes;
  uint8_t* dst = a.payload_out + o0;
  const uint32_t head = min((uint32_t)((4u - (uint32_t)(o0 & 3u)) & 3u), len);
  const uint32_t words = (len - head) >> 2;
  const uint32_t tail = len - head - 4 * words;
  if (lane < (int)head) dst[lane] = src[lane];
  if (lane < (int)tail) dst[head + 4 * words + lane] = src[head + 4 * words + lane];
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
  const uint32_t sh = 8 * head;  // src byte offset of the body inside its first word
  for (uint32_t w = lane; w < words; w += 32) {
    const uint32_t lo = s32[w];
    const uint32_t v = sh ? __funnelshift_r(lo, s32[w + 1], sh) : lo;
    d32[w] = v;
  }
}

// decode-side checks: offsets[0] == 0, offsets[nblocks] == payload bytes
// (codecs.py:412-413 / :429-430 trailing-byte rule), none: exact length.
__global__ void k_check_payload(CodecArgs a) {
  const StreamTab& st = *a.st;
  if (a.g.codec == C_NONE) {
    if (a.payload_bytes >= 0 && a.payload_bytes != st.packed_bytes) atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  if (a.offsets_in[0] != 0) atomicOr(a.status, KVC_FLAG_CODEC);
  if (a.payload_bytes >= 0 && (int64_t)a.offsets_in[st.nblocks] != a.payload_bytes) atomicOr(a.status, KVC_FLAG_CODEC);
}

void widths_used(const Geo& g, bool used[9]) {
  for (int i = 0; i < 9; ++i) used[i] = false;
  if (g.quant == Q_UNIFORM || g.quant == Q_UCHAN) {
    used[g.bits] = true;
  } else {
    used[g.hi] = used[g.lo] = true;
  }
}

}  // namespace

size_t codec_scan_bytes(int64_t max_blocks) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)(max_blocks + 1));
  return bytes + 256;
}

cudaError_t launch_codec_encode(const CodecArgs& args, int sm_count, cudaStream_t s) {
  (void)sm_count;
  CodecArgs a = args;
  if (a.g.codec == C_ENTROPY) a.recip = recip_tables(s);
  const unsigned grid = (unsigned)((a.max_blocks + 1 + 127) / 128);
  bool used[9];
  widths_used(a.g, used);
  if (a.g.codec == C_ENTROPY) {
    // one launch per width in use; each thread skips blocks of other widths
    for (int w = 1; w <= 8; ++w) {
      if (!used[w]) continue;
      cudaError_t e = w <= 4 ? launch_rc_small_encode(a, w, grid, s) : launch_rc_large_encode(a, w, s);
      if (e != cudaSuccess) return e;
    }
  } else {
    ProfScope ps("rle_encode", s);
    k_rle_encode<<<grid, 128, 0, s>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  size_t tmp = a.scan_bytes;
  {
    ProfScope ps("offset_scan", s);
    e = cub::DeviceScan::ExclusiveSum(a.scan_tmp, tmp, a.sizes, a.offsets, (int)(a.max_blocks + 1), s);
  }
  if (e != cudaSuccess) return e;
  const unsigned ggrid = (unsigned)((a.max_blocks * 32 + 255) / 256 + 1);
  ProfScope ps("gather", s);
  k_gather<<<ggrid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_codec_decode(const CodecArgs& args, int sm_count, cudaStream_t s) {
  (void)sm_count;
  CodecArgs a = args;
  if (a.g.codec == C_ENTROPY) a.recip = recip_tables(s);
  {
    ProfScope ps("check_payload", s);
    k_check_payload<<<1, 1, 0, s>>>(a);
  }
  if (a.g.codec == C_NONE) return cudaGetLastError();
  const unsigned grid = (unsigned)((a.max_blocks + 127) / 128 + 1);
  bool used[9];
  widths_used(a.g, used);
  if (a.g.codec == C_ENTROPY) {
    for (int w = 1; w <= 8; ++w) {
      if (!used[w]) continue;
      cudaError_t e = w <= 4 ? launch_rc_small_decode(a, w, grid, s) : launch_rc_large_decode(a, w, s);
      if (e != cudaSuccess) return e;
    }
  } else {
    ProfScope ps("rle_decode", s);
    k_rle_decode<<<grid, 128, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace kvc
