// Codec stage over packed width streams: per-block adaptive range coding
// (c=entropy) and PackBits RLE (c=rle), plus the block-offset scan.
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
#include "numerics.cuh"
#include "profile.h"

namespace kvc {

namespace {

constexpr uint32_t kTop = 1u << 24;
constexpr uint32_t kBot = 1u << 16;
constexpr uint32_t kStep = 32u;
constexpr uint32_t kLimit = 1u << 16;

// ----------------------------------------------------------- byte streams
struct ByteReader {  // sequential reader over an arbitrarily aligned buffer
  const uint32_t* w;
  uint32_t cur;
  int idx;  // next byte index within cur (0..4)
  __device__ void init(const uint8_t* p) {
    uintptr_t a = reinterpret_cast<uintptr_t>(p);
    w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
    idx = (int)(a & 3);
    cur = __ldg(w);
  }
  __device__ __forceinline__ uint32_t next() {
    if (idx == 4) {
      cur = __ldg(++w);
      idx = 0;
    }
    uint32_t b = (cur >> (idx * 8)) & 0xFFu;
    ++idx;
    return b;
  }
};

struct WordWriter {  // sequential writer into a 4-byte aligned buffer
  uint32_t* w;
  uint32_t acc;
  int n;
  __device__ void init(uint8_t* p) {
    w = reinterpret_cast<uint32_t*>(p);
    acc = 0;
    n = 0;
  }
  __device__ __forceinline__ void put(uint32_t b) {
    acc |= b << (n * 8);
    if (++n == 4) {
      *w++ = acc;
      acc = 0;
      n = 0;
    }
  }
  __device__ void flush() {
    if (n) *w = acc;
  }
};

// symbols of width W read MSB-first from a byte stream
template <int W>
struct SymReader {
  ByteReader br;
  uint32_t buf;
  int nb;
  __device__ void init(const uint8_t* p) {
    br.init(p);
    buf = 0;
    nb = 0;
  }
  __device__ __forceinline__ uint32_t next() {
    if (nb < W) {
      buf = (buf << 8) | br.next();
      nb += 8;
    }
    nb -= W;
    return (buf >> nb) & ((1u << W) - 1u);
  }
};

// ------------------------------------------------------------ order-0 model
// codecs.py:188-242: all frequencies start at 1; +32 per coded symbol; when
// the total reaches 2^16 every frequency becomes max(1, f // 2).
template <int W, bool kSmall = (W <= 4)>
struct Model;

template <int W>
struct Model<W, true> {  // registers, fully unrolled
  static constexpr int A = 1 << W;
  uint32_t f[A];
  uint32_t total;
  __device__ void init() {
#pragma unroll
    for (int i = 0; i < A; ++i) f[i] = 1;
    total = A;
  }
  __device__ __forceinline__ void lookup(uint32_t s, uint32_t& cum, uint32_t& fr) const {
    uint32_t c = 0, r = 0;
#pragma unroll
    for (int i = 0; i < A; ++i) {
      c += (i < (int)s) ? f[i] : 0u;
      r = (i == (int)s) ? f[i] : r;
    }
    cum = c;
    fr = r;
  }
  __device__ __forceinline__ uint32_t find(uint32_t target, uint32_t& cum, uint32_t& fr) const {
    uint32_t c = 0, s = 0, cs = 0, fs = f[0];
#pragma unroll
    for (int i = 0; i < A; ++i) {
      bool ge = target >= c;
      s = ge ? i : s;
      cs = ge ? c : cs;
      fs = ge ? f[i] : fs;
      c += f[i];
    }
    cum = cs;
    fr = fs;
    return s;
  }
  __device__ __forceinline__ void bump(uint32_t s) {
#pragma unroll
    for (int i = 0; i < A; ++i) f[i] += (i == (int)s) ? kStep : 0u;
    total += kStep;
    if (total >= kLimit) {
      uint32_t t = 0;
#pragma unroll
      for (int i = 0; i < A; ++i) {
        uint32_t h = f[i] >> 1;
        f[i] = h ? h : 1u;
        t += f[i];
      }
      total = t;
    }
  }
};

template <int W>
struct Model<W, false> {  // Fenwick tree in local memory (A = 32..256)
  static constexpr int A = 1 << W;
  uint32_t f[A];
  uint32_t tree[A + 1];
  uint32_t total;
  __device__ void rebuild() {
    for (int i = 0; i <= A; ++i) tree[i] = 0;
    for (int i = 1; i <= A; ++i) {
      tree[i] += f[i - 1];
      int j = i + (i & -i);
      if (j <= A) tree[j] += tree[i];
    }
  }
  __device__ void init() {
    for (int i = 0; i < A; ++i) f[i] = 1;
    total = A;
    rebuild();
  }
  __device__ __forceinline__ uint32_t prefix(uint32_t s) const {
    uint32_t c = 0;
    for (int i = (int)s; i > 0; i -= i & -i) c += tree[i];
    return c;
  }
  __device__ __forceinline__ void lookup(uint32_t s, uint32_t& cum, uint32_t& fr) const {
    cum = prefix(s);
    fr = f[s];
  }
  __device__ __forceinline__ uint32_t find(uint32_t target, uint32_t& cum, uint32_t& fr) const {
    int pos = 0;
    uint32_t rem = target;
#pragma unroll
    for (int bit = A; bit; bit >>= 1) {
      int nx = pos + bit;
      if (nx <= A && tree[nx] <= rem) {
        rem -= tree[nx];
        pos = nx;
      }
    }
    cum = target - rem;
    fr = f[pos];
    return (uint32_t)pos;
  }
  __device__ __forceinline__ void bump(uint32_t s) {
    f[s] += kStep;
    for (int i = (int)s + 1; i <= A; i += i & -i) tree[i] += kStep;
    total += kStep;
    if (total >= kLimit) {
      uint32_t t = 0;
      for (int i = 0; i < A; ++i) {
        uint32_t h = f[i] >> 1;
        f[i] = h ? h : 1u;
        t += f[i];
      }
      total = t;
      rebuild();
    }
  }
};

// renormalisation condition of codecs.py:255-261 evaluated without 64-bit
// math: (low ^ (low + range)) < TOP with the carry out of bit 31 counted.
__device__ __forceinline__ bool top_bytes_equal(uint32_t low, uint32_t range) {
  uint32_t s = low + range;
  return s >= low && (low ^ s) < kTop;
}

__device__ __forceinline__ int block_stream(const StreamTab& st, int64_t b) {
  return (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
}

// ------------------------------------------------------------ entropy encode
template <int W>
__device__ void rc_encode_block(const uint8_t* src, int64_t n, uint8_t* slot, int64_t cap, uint64_t* size_out,
                                uint32_t* status) {
  Model<W> m;
  m.init();
  SymReader<W> rd;
  rd.init(src);
  WordWriter wr;
  wr.init(slot + 4);
  uint32_t low = 0, range = 0xFFFFFFFFu;
  int64_t len = 0;
  const int64_t lim = cap - 8;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t s = rd.next();
    uint32_t cum, fr;
    m.lookup(s, cum, fr);
    uint32_t unit = range / m.total;
    low += unit * cum;
    range = unit * fr;
    for (;;) {
      if (top_bytes_equal(low, range)) {
      } else if (range < kBot) {
        range = (0u - low) & (kBot - 1u);
      } else {
        break;
      }
      if (len < lim) wr.put(low >> 24);
      ++len;
      low <<= 8;
      range <<= 8;
    }
    m.bump(s);
  }
  for (int k = 0; k < 4; ++k) {
    if (len < lim) wr.put(low >> 24);
    ++len;
    low <<= 8;
  }
  wr.flush();
  if (len >= lim) {
    atomicOr(status, KVC_FLAG_CAPACITY);
    len = 0;
  }
  uint32_t be = ((uint32_t)len >> 24) | (((uint32_t)len >> 8) & 0xFF00u) | (((uint32_t)len << 8) & 0xFF0000u) |
                ((uint32_t)len << 24);
  *reinterpret_cast<uint32_t*>(slot) = be;
  *size_out = (uint64_t)len + 4;
}

template <int W>
__device__ void rc_decode_block(const uint8_t* src, int64_t avail, uint8_t* dst, int64_t n, uint32_t* status) {
  if (avail < 4) {
    atomicOr(status, KVC_FLAG_CODEC);
    return;
  }
  ByteReader br;
  br.init(src);
  uint32_t hdr = 0;
  for (int k = 0; k < 4; ++k) hdr = (hdr << 8) | br.next();
  if ((int64_t)hdr + 4 != avail) {
    atomicOr(status, KVC_FLAG_CODEC);
    return;
  }
  int64_t left = hdr;
  Model<W> m;
  m.init();
  uint32_t low = 0, range = 0xFFFFFFFFu, code = 0;
  bool bad = false;
  for (int k = 0; k < 4; ++k) {
    uint32_t b = 0;
    if (left > 0) { b = br.next(); --left; } else bad = true;
    code = (code << 8) | b;
  }
  uint32_t acc = 0;
  int nacc = 0;
  uint8_t* o = dst;
  for (int64_t i = 0; i < n && !bad; ++i) {
    uint32_t unit = range / m.total;
    uint32_t s, cum, fr;
    if (code >= low) {
      uint32_t q = (code - low) / unit;
      uint32_t target = q < m.total - 1 ? q : m.total - 1;
      s = m.find(target, cum, fr);
    } else {  // negative target (malformed stream): the reference's search yields 0
      s = 0;
      m.lookup(0, cum, fr);
    }
    low += unit * cum;
    range = unit * fr;
    for (;;) {
      if (top_bytes_equal(low, range)) {
      } else if (range < kBot) {
        range = (0u - low) & (kBot - 1u);
      } else {
        break;
      }
      uint32_t b = 0;
      if (left > 0) { b = br.next(); --left; } else { bad = true; break; }
      code = (code << 8) | b;
      low <<= 8;
      range <<= 8;
    }
    m.bump(s);
    acc = (acc << W) | s;
    nacc += W;
    if (nacc >= 8) {
      nacc -= 8;
      *o++ = (uint8_t)(acc >> nacc);
    }
  }
  if (bad) {
    atomicOr(status, KVC_FLAG_CODEC);
    return;
  }
  if (nacc) *o = (uint8_t)(acc << (8 - nacc));
}

template <int W>
__global__ void __launch_bounds__(128) k_rc_encode(CodecArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > a.max_blocks) return;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) {
    a.sizes[b] = 0;
    return;
  }
  const int si = block_stream(st, b);
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int64_t n = min(a.g.block, st.count[si] - start);
  const uint8_t* src = a.packed_in + st.byte_off[si] + start * W / 8;
  rc_encode_block<W>(src, n, a.slots + b * a.slot_bytes, a.slot_bytes, a.sizes + b, a.status);
}

template <int W>
__global__ void __launch_bounds__(128) k_rc_decode(CodecArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) return;
  const int si = block_stream(st, b);
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int64_t n = min(a.g.block, st.count[si] - start);
  const uint64_t o0 = a.offsets_in[b], o1 = a.offsets_in[b + 1];
  if (o1 < o0 || (a.payload_bytes >= 0 && (int64_t)o1 > a.payload_bytes)) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  rc_decode_block<W>(a.payload_in + o0, (int64_t)(o1 - o0), a.packed_out + st.byte_off[si] + start * W / 8, n,
                     a.status);
}

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
  while (pos < len) {
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
// one warp per block copies its slot bytes to payload[offsets[b]]
__global__ void __launch_bounds__(256) k_gather(CodecArgs a) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const StreamTab& st = *a.st;
  if (b >= st.nblocks) return;
  const uint64_t o0 = a.offsets[b], o1 = a.offsets[b + 1];
  const uint8_t* src = a.slots + b * a.slot_bytes;
  uint8_t* dst = a.payload_out + o0;
  for (uint64_t k = lane; k < o1 - o0; k += 32) dst[k] = src[k];
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

template <int W>
void launch_rc_encode_w(const CodecArgs& a, unsigned grid, cudaStream_t s) {
  ProfScope ps("rc_encode", s);
  k_rc_encode<W><<<grid, 128, 0, s>>>(a);
}
template <int W>
void launch_rc_decode_w(const CodecArgs& a, unsigned grid, cudaStream_t s) {
  ProfScope ps("rc_decode", s);
  k_rc_decode<W><<<grid, 128, 0, s>>>(a);
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

cudaError_t launch_codec_encode(const CodecArgs& a, int sm_count, cudaStream_t s) {
  (void)sm_count;
  const unsigned grid = (unsigned)((a.max_blocks + 1 + 127) / 128);
  bool used[9];
  widths_used(a.g, used);
  if (a.g.codec == C_ENTROPY) {
    // one launch per width in use; each thread skips blocks of other widths
    for (int w = 1; w <= 4; ++w)
      if (used[w]) launch_rc_small_encode(a, w, grid, s);
    if (used[5]) launch_rc_encode_w<5>(a, grid, s);
    if (used[6]) launch_rc_encode_w<6>(a, grid, s);
    if (used[7]) launch_rc_encode_w<7>(a, grid, s);
    if (used[8]) launch_rc_encode_w<8>(a, grid, s);
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

cudaError_t launch_codec_decode(const CodecArgs& a, int sm_count, cudaStream_t s) {
  (void)sm_count;
  {
    ProfScope ps("check_payload", s);
    k_check_payload<<<1, 1, 0, s>>>(a);
  }
  if (a.g.codec == C_NONE) return cudaGetLastError();
  const unsigned grid = (unsigned)((a.max_blocks + 127) / 128 + 1);
  bool used[9];
  widths_used(a.g, used);
  if (a.g.codec == C_ENTROPY) {
    for (int w = 1; w <= 4; ++w)
      if (used[w]) launch_rc_small_decode(a, w, grid, s);
    if (used[5]) launch_rc_decode_w<5>(a, grid, s);
    if (used[6]) launch_rc_decode_w<6>(a, grid, s);
    if (used[7]) launch_rc_decode_w<7>(a, grid, s);
    if (used[8]) launch_rc_decode_w<8>(a, grid, s);
  } else {
    ProfScope ps("rle_decode", s);
    k_rle_decode<<<grid, 128, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace kvc
