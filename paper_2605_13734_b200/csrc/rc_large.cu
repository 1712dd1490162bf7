// Adaptive range coder, large alphabets (w = 5..8 bits, A = 32..256): the
// c=entropy path of the 8-bit profiles (BASELINE config 5).
//
// Bit-exact with codecs.py:181-331 per block; one thread per block.  The
// order-0 model (codecs.py:188-242) is ONE u16 Fenwick tree of frequencies
// per thread in shared memory (512 B at A = 256), element j of thread t at
// [j][t] so a warp's accesses to the same node are conflict-free; a symbol's
// frequency is a Fenwick point query, so no separate frequency array is kept
// and twice as many blocks fit per SM.  Prefix / point / update paths are
// known from the symbol up front, so their shared loads issue together.
// Node values never exceed the running total (< 2^16): a bump that would
// reach 2^16 takes the halving path (frequencies recovered from the tree,
// incremented, halved, tree rebuilt) before any node is written.  Before the
// first halving `range // total` uses the reciprocal table (rc_tables.cuh).
#include <cstdint>

#include "kernels.h"
#include "profile.h"
#include "rc_coder.cuh"
#include "rc_tables.cuh"

namespace kvc {
namespace {

constexpr int kLThreads = 128;

template <int W>
__host__ __device__ constexpr int halving_at() {
  return (65536 - (1 << W) + 31) / 32;
}

template <int W>
struct LModel {
  static constexpr int A = 1 << W;
  uint16_t* tree;  // node j (1..A) at tree[(j - 1) * kLThreads]
  uint32_t total;
  __device__ __forceinline__ uint32_t T(uint32_t j) const { return tree[(j - 1) * kLThreads]; }
  __device__ __forceinline__ void set(uint32_t j, uint32_t v) { tree[(j - 1) * kLThreads] = (uint16_t)v; }
  __device__ void init(uint16_t* base, int lane) {
    tree = base + lane;
    for (uint32_t j = 1; j <= (uint32_t)A; ++j) set(j, j & (0u - j));  // all frequencies 1
    total = A;
  }
  // sum of f[0..s-1]
  __device__ __forceinline__ uint32_t prefix(uint32_t s) const {
    uint32_t c = 0, i = s;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      c += i ? T(i) : 0u;
      i &= i - 1;
    }
    return c;
  }
  // f[s] = T(s+1) - sum of the nodes between (s+1) - lowbit(s+1) and s
  __device__ __forceinline__ uint32_t freq(uint32_t s) const {
    const uint32_t i = s + 1;
    const uint32_t stop = i - (i & (0u - i));
    uint32_t v = T(i), j = s;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      v -= (j > stop) ? T(j) : 0u;
      j = (j > stop) ? (j & (j - 1)) : j;
    }
    return v;
  }
  // codecs.py:227-242: f[s] += 32, total += 32, halve at 2^16
  __device__ __forceinline__ void bump(uint32_t s) {
    if (total + 32u < 65536u) {
      uint32_t i = s + 1;
#pragma unroll
      for (int k = 0; k <= W; ++k) {
        if (i <= (uint32_t)A) set(i, T(i) + 32u);
        i += i & (0u - i);
      }
      total += 32u;
    } else {
      halve_with(s);
    }
  }
  __device__ void halve_with(uint32_t s) {
    // tree -> frequencies in place (inverse build), bump s, halve, rebuild
    for (uint32_t j = A; j >= 1; --j) {
      const uint32_t p = j + (j & (0u - j));
      if (p <= (uint32_t)A) set(p, T(p) - T(j));
    }
    const uint32_t fs = T(s + 1) + 32u;  // may be 2^16 for A = 32: kept in 32 bits
    uint32_t t = 0;
    for (uint32_t j = 1; j <= (uint32_t)A; ++j) {
      uint32_t h = (j == s + 1 ? fs : T(j)) >> 1;
      h = h ? h : 1u;
      set(j, h);
      t += h;
    }
    total = t;
    for (uint32_t j = 1; j <= (uint32_t)A; ++j) {
      const uint32_t p = j + (j & (0u - j));
      if (p <= (uint32_t)A) set(p, T(p) + T(j));
    }
  }
  // largest s with prefix(s) <= target (codecs.py:214-225); cum = prefix(s)
  __device__ __forceinline__ uint32_t find(uint32_t target, uint32_t& cum) const {
    uint32_t pos = 0, rem = target;
#pragma unroll
    for (uint32_t bit = A / 2; bit; bit >>= 1) {  // node A holds the total > target
      const uint32_t v = T(pos + bit);
      if (v <= rem) {
        rem -= v;
        pos += bit;
      }
    }
    cum = target - rem;
    return pos;
  }
};

template <int W>
__global__ void __launch_bounds__(kLThreads) k_rc_large_encode(CodecArgs a) {
  constexpr int A = 1 << W;
  constexpr int H = halving_at<W>();
  extern __shared__ __align__(16) uint16_t lsm[];
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
  const uint8_t* src = a.packed_in + st.byte_off[si] + start * W / 8;
  uint8_t* slot = a.slots + b * a.slot_bytes;
  uint32_t* out = reinterpret_cast<uint32_t*>(slot + 4);
  LModel<W> m;
  m.init(lsm, threadIdx.x);
  RcEnc e;
  e.init(out);
  uint32_t buf = 0;
  int nb = 0, pos = 0;
  for (int i = 0; i < n; ++i) {
    if (nb < W) {
      buf = (buf << 8) | __ldg(src + pos++);
      nb += 8;
    }
    nb -= W;
    const uint32_t s = (buf >> nb) & (A - 1);
    const uint32_t cum = m.prefix(s);
    const uint32_t fr = m.freq(s);
    const uint32_t unit = (i < H) ? div_recip(e.range, m.total, __ldg(magic + i)) : e.range / m.total;
    e.encode(unit, cum, fr);
    m.bump(s);
  }
  const uint32_t nout = e.finish();
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(nout, 0, 0x0123);
  a.sizes[b] = (uint64_t)nout + 4;
}

template <int W>
__global__ void __launch_bounds__(kLThreads) k_rc_large_decode(CodecArgs a) {
  constexpr int H = halving_at<W>();
  extern __shared__ __align__(16) uint16_t lsm[];
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
  const int64_t len = (int64_t)(o1 - o0);
  uint32_t hdr = 0;
  for (int k = 0; k < 4; ++k) hdr = (hdr << 8) | src[k];
  if ((int64_t)hdr + 4 != len) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  RcDec d;
  d.init(src, src + len);
  LModel<W> m;
  m.init(lsm, threadIdx.x);
  uint8_t* dst = a.packed_out + st.byte_off[si] + start * W / 8;
  uint64_t acc = 0;
  int nacc = 0, nout = 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t unit = (i < H) ? div_recip(d.range, m.total, __ldg(magic + i)) : d.range / m.total;
    uint32_t s, cum;
    if (d.code >= d.low) {
      uint32_t target = (d.code - d.low) / unit;
      target = target < m.total - 1 ? target : m.total - 1;
      s = m.find(target, cum);
    } else {  // malformed stream: the reference's search yields symbol 0
      s = 0;
      cum = 0;
    }
    const uint32_t fr = m.freq(s);
    d.advance(unit * cum, unit * (cum + fr));
    m.bump(s);
    acc = (acc << W) | s;
    nacc += W;
    if (nacc >= 8) {
      nacc -= 8;
      dst[nout++] = (uint8_t)(acc >> nacc);
    }
  }
  // bytes consumed = 4 header + 4 priming + pulled (codecs.py:283-288)
  if ((int64_t)d.pulled() + 8 > len) atomicOr(a.status, KVC_FLAG_CODEC);
}

template <int W>
size_t large_smem() {
  return (size_t)(1 << W) * kLThreads * sizeof(uint16_t);
}

template <int W>
cudaError_t enc_w(const CodecArgs& a, cudaStream_t s) {
  const size_t sm = large_smem<W>();
  cudaFuncSetAttribute(k_rc_large_encode<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const unsigned grid = (unsigned)((a.max_blocks + 1 + kLThreads - 1) / kLThreads);
  k_rc_large_encode<W><<<grid, kLThreads, sm, s>>>(a);
  return cudaGetLastError();
}

template <int W>
cudaError_t dec_w(const CodecArgs& a, cudaStream_t s) {
  const size_t sm = large_smem<W>();
  cudaFuncSetAttribute(k_rc_large_decode<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const unsigned grid = (unsigned)((a.max_blocks + kLThreads - 1) / kLThreads + 1);
  k_rc_large_decode<W><<<grid, kLThreads, sm, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rc_large_encode(const CodecArgs& a, int w, cudaStream_t s) {
  ProfScope ps("rc_encode", s);
  switch (w) {
    case 5: return enc_w<5>(a, s);
    case 6: return enc_w<6>(a, s);
    case 7: return enc_w<7>(a, s);
    default: return enc_w<8>(a, s);
  }
}

cudaError_t launch_rc_large_decode(const CodecArgs& a, int w, cudaStream_t s) {
  ProfScope ps("rc_decode", s);
  switch (w) {
    case 5: return dec_w<5>(a, s);
    case 6: return dec_w<6>(a, s);
    case 7: return dec_w<7>(a, s);
    default: return dec_w<8>(a, s);
  }
}

}  // namespace kvc
