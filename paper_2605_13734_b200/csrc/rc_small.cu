// Adaptive range coder, small alphabets (w <= 4 bits, A = 2^w <= 16): the
// c=entropy hot path of the KIVI 2-bit profiles.
//
// Bit-exact with codecs.py:181-331 per block.  One thread codes one block;
// a warp's lanes walk their blocks in lockstep, which makes the first H =
// ceil((65536 - A) / 32) = 2048 symbols special: the model total at symbol i
// is exactly A + 32 i for every lane (codecs.py:227-232: no halving can
// happen before it), so
//   * `range // total` is a multiply by a per-position reciprocal from a
//     global read-only table (rc_tables.cuh, warp-uniform index) plus one
//     correction (div_magic), and
//   * no halving check is needed inside that loop.
// The remainder of a longer block (after the first halving) and short tails
// run a generic per-symbol loop with hardware division.  Cumulative
// frequencies live in registers (16-bit fields of one 64-bit word for
// A <= 4); bytes are emitted / pulled with one funnel shift each.
#include <cstdint>

#include "kernels.h"
#include "profile.h"
#include "rc_tables.cuh"

namespace kvc {
namespace {

constexpr uint32_t kTop = 1u << 24;
constexpr uint32_t kBot = 1u << 16;
constexpr int kH = 2048;  // first halving after symbol kH-1 for every A in 2..16

__device__ __forceinline__ uint32_t div_magic(uint32_t n, uint32_t d, uint32_t m) {
  // floor(n / d) with m = floor(2^32 / d): the estimate is q or q-1
  const uint32_t q = __umulhi(n, m);
  return q + ((n - q * d) >= d ? 1u : 0u);
}

// ----------------------------------------------------------------- models
template <int W, bool kPacked = (W <= 2)>
struct SModel;

template <int W>
struct SModel<W, true> {  // A <= 4: fields [0 | C1 | C2 | C3] of a 64-bit word
  static constexpr int A = 1 << W;
  uint64_t M;
  uint32_t total;
  __device__ void init() {
    M = 0;
#pragma unroll
    for (int k = 1; k < A; ++k) M |= (uint64_t)k << (16 * k);
    total = A;
  }
  __device__ __forceinline__ uint32_t field(int k) const { return (uint32_t)(M >> (16 * k)) & 0xFFFFu; }
  __device__ __forceinline__ void lookup(uint32_t s, uint32_t& lo, uint32_t& hi) const {
    lo = (uint32_t)(M >> (16 * s)) & 0xFFFFu;
    hi = (s == A - 1) ? total : (uint32_t)(M >> (16 * (s + 1))) & 0xFFFFu;
  }
  __device__ __forceinline__ void add(uint32_t s) {
    constexpr uint64_t inc = (A == 4) ? ((32ull << 16) | (32ull << 32) | (32ull << 48)) : (32ull << 16);
    M += inc << (16 * s);
  }
  __device__ void halve() {
    uint32_t prev = 0, t = 0;
    uint64_t nm = 0;
#pragma unroll
    for (int k = 1; k <= A; ++k) {
      const uint32_t ck = (k == A) ? total : field(k);
      uint32_t f = (ck - prev) >> 1;
      f = f ? f : 1u;
      prev = ck;
      t += f;
      if (k < A) nm |= (uint64_t)t << (16 * k);
    }
    M = nm;
    total = t;
  }
  // decode: largest s with C[s]*unit <= x; returns the scaled bounds
  __device__ __forceinline__ uint32_t find(uint32_t x, uint32_t unit, uint32_t& plo, uint32_t& phi) const {
    uint32_t p[A + 1];
    p[0] = 0;
    uint32_t s = 0;
#pragma unroll
    for (int k = 1; k < A; ++k) {
      p[k] = unit * field(k);
      s += (x >= p[k]) ? 1u : 0u;
    }
    p[A] = unit * total;
    plo = 0;
    phi = p[1];
#pragma unroll
    for (int k = 1; k < A; ++k) {
      plo = (s == (uint32_t)k) ? p[k] : plo;
      phi = (s == (uint32_t)k) ? p[k + 1] : phi;
    }
    return s;
  }
};

template <int W>
struct SModel<W, false> {  // A = 8, 16: cumulative counts in registers
  static constexpr int A = 1 << W;
  uint32_t C[A];
  uint32_t total;
  __device__ void init() {
#pragma unroll
    for (int k = 0; k < A; ++k) C[k] = k;
    total = A;
  }
  __device__ __forceinline__ void lookup(uint32_t s, uint32_t& lo, uint32_t& hi) const {
    lo = 0;
    hi = total;
#pragma unroll
    for (int k = 1; k < A; ++k) {
      lo = (s == (uint32_t)k) ? C[k] : lo;
      hi = (s + 1 == (uint32_t)k) ? C[k] : hi;
    }
  }
  __device__ __forceinline__ void add(uint32_t s) {
#pragma unroll
    for (int k = 1; k < A; ++k) C[k] += ((uint32_t)k > s) ? 32u : 0u;
  }
  __device__ void halve() {
    uint32_t prev = 0, t = 0;
#pragma unroll
    for (int k = 1; k <= A; ++k) {
      const uint32_t ck = (k == A) ? total : C[k];
      uint32_t f = (ck - prev) >> 1;
      f = f ? f : 1u;
      prev = ck;
      t += f;
      if (k < A) C[k] = t;
    }
    total = t;
  }
  __device__ __forceinline__ uint32_t find(uint32_t x, uint32_t unit, uint32_t& plo, uint32_t& phi) const {
    uint32_t target = x / unit;
    target = target < total - 1 ? target : total - 1;
    uint32_t s = 0;
#pragma unroll
    for (int k = 1; k < A; ++k) s += (target >= C[k]) ? 1u : 0u;
    uint32_t lo, hi;
    lookup(s, lo, hi);
    plo = unit * lo;
    phi = unit * hi;
    return s;
  }
};

// ----------------------------------------------------------------- encoder
struct Enc {
  uint32_t low, range;
  uint32_t acc;  // pending output bytes, big-endian
  uint32_t n;    // bytes emitted
  uint32_t* out;
  __device__ __forceinline__ void emit() {
    acc = __funnelshift_l(low, acc, 8);  // acc << 8 | low >> 24
    if ((++n & 3u) == 0) out[(n >> 2) - 1] = __byte_perm(acc, 0, 0x0123);
    low <<= 8;
    range <<= 8;
  }
  __device__ __forceinline__ void step(uint32_t unit, uint32_t lo, uint32_t hi) {
    low += unit * lo;
    range = unit * (hi - lo);
    for (;;) {  // codecs.py:255-264, (low ^ (low + range)) < TOP in 33 bits
      const uint32_t t = low + range;
      if (t < low || (low ^ t) >= kTop) {
        if (range >= kBot) break;
        range = (0u - low) & (kBot - 1u);
      }
      emit();
    }
  }
};

template <int W>
__device__ __forceinline__ uint32_t sym_at(const uint32_t* wd, int j) {
  constexpr uint32_t mask = (1u << W) - 1u;
  const int p = j * W, k = p >> 5, off = p & 31;
  if (off + W <= 32) return (wd[k] >> (32 - off - W)) & mask;
  return ((wd[k] << (off + W - 32)) | (wd[k + 1] >> (64 - off - W))) & mask;
}

// symbols per group and words per group: a group is a whole number of words
template <int W>
struct Grp {
  static constexpr int kSyms = (W == 3) ? 32 : 32 / W;
  static constexpr int kWords = (W == 3) ? 3 : 1;
};

template <int W>
__global__ void __launch_bounds__(128) k_rc_small_encode(CodecArgs a) {
  constexpr int A = 1 << W;
  const uint32_t* __restrict__ magic = a.recip + W * kRecipLen;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > a.max_blocks) return;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) {
    a.sizes[b] = 0;
    return;
  }
  const int si = (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int n = (int)min(a.g.block, st.count[si] - start);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(a.packed_in + st.byte_off[si] + start * W / 8);
  uint8_t* slot = a.slots + b * a.slot_bytes;
  SModel<W> m;
  m.init();
  Enc e;
  e.low = 0;
  e.range = 0xFFFFFFFFu;
  e.acc = 0;
  e.n = 0;
  e.out = reinterpret_cast<uint32_t*>(slot + 4);
  constexpr int GS = Grp<W>::kSyms, GW = Grp<W>::kWords;
  const int n1 = min(n, kH) / GS;  // whole groups in the reciprocal-table phase
  for (int gI = 0; gI < n1; ++gI) {
    uint32_t wd[GW];
#pragma unroll
    for (int k = 0; k < GW; ++k) wd[k] = __byte_perm(__ldg(src + gI * GW + k), 0, 0x0123);
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const uint32_t s = sym_at<W>(wd, j);
      const uint32_t unit = div_magic(e.range, m.total, magic[gI * GS + j]);
      uint32_t lo, hi;
      m.lookup(s, lo, hi);
      e.step(unit, lo, hi);
      m.add(s);
      m.total += 32;
    }
  }
  int i = n1 * GS;
  if (i == kH) m.halve();  // total reached A + 32 kH >= 2^16 (codecs.py:231-232)
  if (i < n) {             // phase 2 / tail: generic per-symbol loop
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(src) + (size_t)i * W / 8;
    uint32_t buf = 0;
    int nb = 0, pos = 0;
    for (; i < n; ++i) {
      if (nb < W) {
        buf = (buf << 8) | sb[pos++];
        nb += 8;
      }
      nb -= W;
      const uint32_t s = (buf >> nb) & (A - 1);
      const uint32_t unit = (i < kH) ? div_magic(e.range, m.total, magic[i]) : e.range / m.total;
      uint32_t lo, hi;
      m.lookup(s, lo, hi);
      e.step(unit, lo, hi);
      m.add(s);
      m.total += 32;
      if (m.total >= 65536u) m.halve();
    }
  }
  for (int k = 0; k < 4; ++k) e.emit();  // finish: 4 bytes of low (codecs.py:266-270)
  if (e.n & 3u) e.out[e.n >> 2] = __byte_perm(e.acc << (8 * (4 - (e.n & 3u))), 0, 0x0123);
  const uint32_t len = e.n;  // <= 4 bytes per symbol + 4 < slot capacity
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(len, 0, 0x0123);
  a.sizes[b] = (uint64_t)len + 4;
}

// ----------------------------------------------------------------- decoder
struct Dec {
  uint32_t low, range, code;
  uint32_t cur;  // remaining bytes of the current input word, big-endian aligned at the top
  int avail;     // bytes left in cur
  const uint32_t* p;
  const uint32_t* last;  // last readable word (reads are clamped; overruns are detected by count)
  uint32_t pulled;       // bytes consumed after the 4 priming bytes
  __device__ __forceinline__ uint32_t next_byte() {
    if (avail == 0) {
      p = p < last ? p + 1 : p;
      cur = __byte_perm(__ldg(p), 0, 0x0123);
      avail = 4;
    }
    const uint32_t b = cur >> 24;
    cur <<= 8;
    --avail;
    return b;
  }
  __device__ __forceinline__ void step(uint32_t plo, uint32_t phi) {
    low += plo;
    range = phi - plo;
    for (;;) {
      const uint32_t t = low + range;
      if (t < low || (low ^ t) >= kTop) {
        if (range >= kBot) break;
        range = (0u - low) & (kBot - 1u);
      }
      code = (code << 8) | next_byte();
      ++pulled;
      low <<= 8;
      range <<= 8;
    }
  }
};

template <int W>
__device__ __forceinline__ uint32_t dec_symbol(Dec& d, SModel<W>& m, uint32_t unit) {
  uint32_t s, plo, phi;
  if (d.code >= d.low) {
    s = m.find(d.code - d.low, unit, plo, phi);
  } else {  // malformed stream: the reference's Fenwick search yields symbol 0
    s = 0;
    uint32_t lo, hi;
    m.lookup(0, lo, hi);
    plo = unit * lo;
    phi = unit * hi;
  }
  d.step(plo, phi);
  m.add(s);
  m.total += 32;
  return s;
}

template <int W>
__global__ void __launch_bounds__(128) k_rc_small_decode(CodecArgs a) {
  constexpr int A = 1 << W;
  const uint32_t* __restrict__ magic = a.recip + W * kRecipLen;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) return;
  const int si = (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int n = (int)min(a.g.block, st.count[si] - start);
  const uint64_t o0 = a.offsets_in[b], o1 = a.offsets_in[b + 1];
  if (o1 < o0 + 8 || (a.payload_bytes >= 0 && (int64_t)o1 > a.payload_bytes)) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  const uint8_t* src = a.payload_in + o0;
  uint32_t hdr = 0, code = 0;
  for (int k = 0; k < 4; ++k) hdr = (hdr << 8) | src[k];
  if ((uint64_t)hdr + 4 != o1 - o0) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  for (int k = 4; k < 8; ++k) code = (code << 8) | src[k];
  Dec d;
  d.low = 0;
  d.range = 0xFFFFFFFFu;
  d.code = code;
  d.pulled = 0;
  {
    const uintptr_t q = reinterpret_cast<uintptr_t>(src + 8);
    const uintptr_t e = reinterpret_cast<uintptr_t>(a.payload_in + o1 - 1);
    d.p = reinterpret_cast<const uint32_t*>(q & ~(uintptr_t)3);
    d.last = reinterpret_cast<const uint32_t*>(e & ~(uintptr_t)3);
    if (d.p > d.last) d.p = d.last;
    const int skip = (int)(q & 3);
    d.cur = __byte_perm(__ldg(d.p), 0, 0x0123) << (8 * skip);
    d.avail = 4 - skip;
  }
  SModel<W> m;
  m.init();
  uint8_t* dst = a.packed_out + st.byte_off[si] + start * W / 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 3) == 0;
  constexpr int GS = Grp<W>::kSyms, GW = Grp<W>::kWords;
  const int n1 = aligned ? min(n, kH) / GS : 0;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst);
  for (int gI = 0; gI < n1; ++gI) {
    uint64_t acc = 0;
    int nbits = 0, wi = 0;  // compile-time after unrolling
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const uint32_t unit = div_magic(d.range, m.total, magic[gI * GS + j]);
      acc = (acc << W) | dec_symbol<W>(d, m, unit);
      nbits += W;
      if (nbits >= 32) {
        nbits -= 32;
        dw[gI * GW + wi++] = __byte_perm((uint32_t)(acc >> nbits), 0, 0x0123);
      }
    }
  }
  int i = n1 * GS;
  if (i == kH) m.halve();
  uint64_t acc = 0;
  int nacc = 0, nout = i * W / 8;
  for (; i < n; ++i) {
    const uint32_t unit = (i < kH) ? div_magic(d.range, m.total, magic[i]) : d.range / m.total;
    acc = (acc << W) | dec_symbol<W>(d, m, unit);
    if (m.total >= 65536u) m.halve();
    nacc += W;
    while (nacc >= 8) {
      nacc -= 8;
      dst[nout++] = (uint8_t)(acc >> nacc);
    }
  }
  // reading past the block's bytes is a truncated stream (codecs.py:283-288)
  if ((uint64_t)d.pulled + 8 > o1 - o0) atomicOr(a.status, KVC_FLAG_CODEC);
}

}  // namespace

bool rc_small_supported(int w) { return w >= 1 && w <= 4; }

cudaError_t launch_rc_small_encode(const CodecArgs& a, int w, unsigned grid, cudaStream_t s) {
  ProfScope ps("rc_encode", s);
  switch (w) {
    case 1: k_rc_small_encode<1><<<grid, 128, 0, s>>>(a); break;
    case 2: k_rc_small_encode<2><<<grid, 128, 0, s>>>(a); break;
    case 3: k_rc_small_encode<3><<<grid, 128, 0, s>>>(a); break;
    default: k_rc_small_encode<4><<<grid, 128, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_rc_small_decode(const CodecArgs& a, int w, unsigned grid, cudaStream_t s) {
  ProfScope ps("rc_decode", s);
  switch (w) {
    case 1: k_rc_small_decode<1><<<grid, 128, 0, s>>>(a); break;
    case 2: k_rc_small_decode<2><<<grid, 128, 0, s>>>(a); break;
    case 3: k_rc_small_decode<3><<<grid, 128, 0, s>>>(a); break;
    default: k_rc_small_decode<4><<<grid, 128, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace kvc
