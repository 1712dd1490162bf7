// Adaptive range coder, large alphabets (w = 5..8 bits, A = 32..256): the
// c=entropy path of the 8-bit profiles (BASELINE config 5).
//
// Bit-exact with codecs.py:181-331 per block; one thread per block.  The
// order-0 model (codecs.py:188-242) is a Fenwick tree of u16 counts plus the
// u16 frequencies, in shared memory, element j of thread t at [j][t] so a
// warp's accesses to the same element are conflict-free.  Prefix and update
// paths are known from the symbol up front, so their loads issue together
// instead of as a dependent chain.  Before the first halving (symbol
// H = ceil((65536 - A) / 32)) the total is A + 32 i for every lane and
// `range // total` uses a per-position reciprocal table (as in rc_small.cu).
#include <cstdint>
#include <type_traits>

#include "kernels.h"
#include "profile.h"

namespace kvc {
namespace {

constexpr uint32_t kTop = 1u << 24;
constexpr uint32_t kBot = 1u << 16;
constexpr int kLThreads = 64;
constexpr int kMaxHL = 2048;

template <int W>
__host__ __device__ constexpr int halving_at() {
  return (65536 - (1 << W) + 31) / 32;
}

__device__ __forceinline__ uint32_t div_magic(uint32_t n, uint32_t d, uint32_t m) {
  const uint32_t q = __umulhi(n, m);
  return q + ((n - q * d) >= d ? 1u : 0u);
}

// Frequencies fit u16 for A >= 64 (f + 32 <= 65535 - (A-1) + 32); A = 32 can
// reach 65536 in long blocks, so small alphabets keep u32 (smem is cheap there).
// Tree nodes are only read while total < 2^16, so u16 suffices.
template <int W>
using FreqT = typename std::conditional<(W <= 6), uint32_t, uint16_t>::type;

template <int W>
struct LModel {
  static constexpr int A = 1 << W;
  static constexpr int LOG = W;
  FreqT<W>* f;     // f[j * kLThreads]
  FreqT<W>* tree;  // tree[(j-1) * kLThreads], j = 1..A
  uint32_t total;
  __device__ __forceinline__ uint32_t F(int j) const { return f[j * kLThreads]; }
  __device__ __forceinline__ uint32_t T(int j) const { return tree[(j - 1) * kLThreads]; }
  __device__ void rebuild() {
    for (int j = 1; j <= A; ++j) tree[(j - 1) * kLThreads] = 0;
    for (int j = 1; j <= A; ++j) {
      const uint32_t v = T(j) + F(j - 1);
      tree[(j - 1) * kLThreads] = (FreqT<W>)v;
      const int p = j + (j & -j);
      if (p <= A) tree[(p - 1) * kLThreads] = (FreqT<W>)(T(p) + v);
    }
  }
  __device__ void init(FreqT<W>* base, int lane) {
    f = base + lane;
    tree = base + A * kLThreads + lane;
    for (int j = 0; j < A; ++j) f[j * kLThreads] = 1;
    total = A;
    rebuild();
  }
  // sum of f[0..s-1]: the log2(A)+1 nodes of the path are independent loads
  __device__ __forceinline__ uint32_t prefix(uint32_t s) const {
    uint32_t c = 0;
    uint32_t i = s;
#pragma unroll
    for (int k = 0; k <= LOG; ++k) {
      const uint32_t v = i ? T((int)i) : 0u;
      c += v;
      i &= i - 1;  // clear the lowest set bit
    }
    return c;
  }
  __device__ __forceinline__ void bump(uint32_t s) {
    f[s * kLThreads] = (FreqT<W>)(F((int)s) + 32u);
    uint32_t i = s + 1;
#pragma unroll
    for (int k = 0; k <= LOG; ++k) {
      if (i <= (uint32_t)A) tree[(i - 1) * kLThreads] = (FreqT<W>)(T((int)i) + 32u);
      i += i & (0u - i);
    }
    total += 32;
  }
  __device__ void halve() {  // codecs.py:234-242
    uint32_t t = 0;
    for (int j = 0; j < A; ++j) {
      uint32_t h = F(j) >> 1;
      h = h ? h : 1u;
      f[j * kLThreads] = (FreqT<W>)h;
      t += h;
    }
    total = t;
    rebuild();
  }
  // largest s with prefix(s) <= target (codecs.py:214-225); cum = prefix(s)
  __device__ __forceinline__ uint32_t find(uint32_t target, uint32_t& cum) const {
    uint32_t pos = 0, rem = target;
#pragma unroll
    for (int bit = A; bit; bit >>= 1) {
      const uint32_t nx = pos + bit;
      if (nx <= (uint32_t)A) {
        const uint32_t v = T((int)nx);
        if (v <= rem) {
          rem -= v;
          pos = nx;
        }
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
  extern __shared__ __align__(16) unsigned char lsm_raw[];
  FreqT<W>* lsm = reinterpret_cast<FreqT<W>*>(lsm_raw);
  uint32_t* magic = reinterpret_cast<uint32_t*>(lsm + 2 * A * kLThreads);
  for (int i = threadIdx.x; i < H; i += blockDim.x) magic[i] = (uint32_t)(0x100000000ull / (uint64_t)(A + 32 * i));
  __syncthreads();
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
  uint32_t low = 0, range = 0xFFFFFFFFu, acc = 0, nout = 0;
  uint32_t buf = 0;
  int nb = 0, pos = 0;
  for (int i = 0; i < n; ++i) {
    if (nb < W) {
      buf = (buf << 8) | src[pos++];
      nb += 8;
    }
    nb -= W;
    const uint32_t s = (buf >> nb) & (A - 1);
    const uint32_t cum = m.prefix(s);
    const uint32_t fr = m.F((int)s);
    const uint32_t unit = (i < H) ? div_magic(range, m.total, magic[i]) : range / m.total;
    low += unit * cum;
    range = unit * fr;
    for (;;) {
      const uint32_t t = low + range;
      if (t < low || (low ^ t) >= kTop) {
        if (range >= kBot) break;
        range = (0u - low) & (kBot - 1u);
      }
      acc = __funnelshift_l(low, acc, 8);
      if ((++nout & 3u) == 0) out[(nout >> 2) - 1] = __byte_perm(acc, 0, 0x0123);
      low <<= 8;
      range <<= 8;
    }
    m.bump(s);
    if (m.total >= 65536u) m.halve();
  }
  for (int k = 0; k < 4; ++k) {
    acc = __funnelshift_l(low, acc, 8);
    if ((++nout & 3u) == 0) out[(nout >> 2) - 1] = __byte_perm(acc, 0, 0x0123);
    low <<= 8;
  }
  if (nout & 3u) out[nout >> 2] = __byte_perm(acc << (8 * (4 - (nout & 3u))), 0, 0x0123);
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(nout, 0, 0x0123);
  a.sizes[b] = (uint64_t)nout + 4;
}

template <int W>
__global__ void __launch_bounds__(kLThreads) k_rc_large_decode(CodecArgs a) {
  constexpr int A = 1 << W;
  constexpr int H = halving_at<W>();
  extern __shared__ __align__(16) unsigned char lsm_raw[];
  FreqT<W>* lsm = reinterpret_cast<FreqT<W>*>(lsm_raw);
  uint32_t* magic = reinterpret_cast<uint32_t*>(lsm + 2 * A * kLThreads);
  for (int i = threadIdx.x; i < H; i += blockDim.x) magic[i] = (uint32_t)(0x100000000ull / (uint64_t)(A + 32 * i));
  __syncthreads();
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
  uint32_t hdr = 0, code = 0;
  for (int k = 0; k < 4; ++k) hdr = (hdr << 8) | src[k];
  if ((int64_t)hdr + 4 != len) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  for (int k = 4; k < 8; ++k) code = (code << 8) | src[k];
  int64_t rp = 8;
  bool bad = false;
  LModel<W> m;
  m.init(lsm, threadIdx.x);
  uint8_t* dst = a.packed_out + st.byte_off[si] + start * W / 8;
  uint32_t low = 0, range = 0xFFFFFFFFu;
  uint64_t acc = 0;
  int nacc = 0, nout = 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t unit = (i < H) ? div_magic(range, m.total, magic[i]) : range / m.total;
    uint32_t s, cum;
    if (code >= low) {
      uint32_t target = (code - low) / unit;
      target = target < m.total - 1 ? target : m.total - 1;
      s = m.find(target, cum);
    } else {  // malformed stream: the reference's search yields symbol 0
      s = 0;
      cum = 0;
    }
    const uint32_t fr = m.F((int)s);
    low += unit * cum;
    range = unit * fr;
    for (;;) {
      const uint32_t t = low + range;
      if (t < low || (low ^ t) >= kTop) {
        if (range >= kBot) break;
        range = (0u - low) & (kBot - 1u);
      }
      uint32_t byte = 0;
      if (rp < len) byte = src[rp];
      else bad = true;
      ++rp;
      code = (code << 8) | byte;
      low <<= 8;
      range <<= 8;
    }
    m.bump(s);
    if (m.total >= 65536u) m.halve();
    acc = (acc << W) | s;
    nacc += W;
    if (nacc >= 8) {
      nacc -= 8;
      dst[nout++] = (uint8_t)(acc >> nacc);
    }
  }
  if (bad) atomicOr(a.status, KVC_FLAG_CODEC);
}

template <int W>
size_t large_smem() {
  return (size_t)2 * (1 << W) * kLThreads * sizeof(FreqT<W>) + (size_t)halving_at<W>() * 4;
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
