// Adaptive range coder, large alphabets (w = 5..8 bits, A = 32..256): the
// c=entropy path of the 8-bit profiles (BASELINE config 5).
//
// Bit-exact with codecs.py:181-331 per block; one thread per block.  The
// order-0 model (codecs.py:188-242) is ONE u16 Fenwick tree of frequencies
// per thread in shared memory (512 B at A = 256), node pairs of thread t in
// word [q][t] so a warp's accesses are bank-conflict-free; a symbol's
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
  // nodes j-1 = 2q, 2q+1 of a thread share one 32-bit word, word q of thread
  // t at [q][t]: every lane of a warp hits its own bank whatever node it reads
  uint16_t* tree;
  uint32_t total;
  __device__ __forceinline__ static uint32_t at(uint32_t j) {
    return (((j - 1) >> 1) * kLThreads) * 2 + ((j - 1) & 1);
  }
  __device__ __forceinline__ uint32_t T(uint32_t j) const { return tree[at(j)]; }
  __device__ __forceinline__ void set(uint32_t j, uint32_t v) { tree[at(j)] = (uint16_t)v; }
  __device__ void init(uint16_t* base, int lane) {
    tree = base + 2 * lane;
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
  // Decoder search without the division: the largest s with
  // unit * prefix(s) <= x, which is find(min(x // unit, total - 1))
  // (codecs.py:214-225, :290-292) since a <= x // unit <=> a * unit <= x and
  // prefix(A-1) <= total - 1; plo = unit * prefix(s).  No overflow: partial
  // sums stay <= unit * total <= range.
  //
  // The same descent also yields phi = unit * prefix(s+1) with no frequency
  // query: node T(pos+bit) rejected at the last rejecting level covers
  // [s+1 - lowbit(s+1), s+1) (every later level was accepted, so s+1's low
  // bit is that level), hence unit * prefix(s+1) is exactly the rejected
  // candidate acc + unit * T(pos+bit); with no rejection s = A-1 and
  // prefix(A) = total.
  __device__ __forceinline__ uint32_t find_scaled(uint32_t x, uint32_t unit, uint32_t& plo, uint32_t& phi) const {
    uint32_t pos = 0, acc = 0, rej = unit * total;
#pragma unroll
    for (uint32_t bit = A / 2; bit; bit >>= 1) {
      const uint32_t v = acc + unit * T(pos + bit);
      if (v <= x) {
        acc = v;
        pos += bit;
      } else {
        rej = v;
      }
    }
    plo = acc;
    phi = rej;
    return pos;
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
  // symbols collect in a 64-bit accumulator and leave as big-endian 32-bit
  // words when the destination is word aligned (blocks of a multiple of 32
  // symbols are), else byte by byte
  const bool word_out = (reinterpret_cast<uintptr_t>(dst) & 3u) == 0;
  uint64_t acc = 0;
  int nacc = 0, nout = 0;
  for (int i = 0; i < n; ++i) {
    const unsigned mask = __activemask();
    const uint32_t unit = (i < H) ? div_recip(d.range, m.total, __ldg(magic + i)) : d.range / m.total;
    // code < low only in a malformed stream; offset() reads 0 -> symbol 0
    uint32_t plo, phi;
    const uint32_t s = m.find_scaled(d.offset(), unit, plo, phi);
    d.advance_warp(plo, phi, mask);
    m.bump(s);
    acc = (acc << W) | s;
    nacc += W;
    if (word_out) {
      if (nacc >= 32) {
        nacc -= 32;
        *reinterpret_cast<uint32_t*>(dst + nout) = __byte_perm((uint32_t)(acc >> nacc), 0, 0x0123);
        nout += 4;
      }
    } else if (nacc >= 8) {
      nacc -= 8;
      dst[nout++] = (uint8_t)(acc >> nacc);
    }
  }
  while (nacc >= 8) {  // whole bytes left over (word_out with a ragged tail)
    nacc -= 8;
    dst[nout++] = (uint8_t)(acc >> nacc);
  }
  // bytes consumed = 4 header + 4 priming + pulled (codecs.py:283-288)
  if ((int64_t)d.pulled() + 8 > len) atomicOr(a.status, KVC_FLAG_CODEC);
}

// ------------------------------------------------ two-phase encoder
// The model values the coder needs at position i (cum, freq, total) depend
// only on the block's symbols, not on the coder state, so for blocks of at
// most 2048 symbols they are computed first, a warp per block, and the coder
// threads then run on precomputed (cum << 16 | freq) words:
//   before the first halving (i < H): f[v] = 1 + 32 c_v(i), so
//     cum_i = s + 32 * #{j < i : s_j < s},  freq_i = 1 + 32 * #{j < i : s_j = s}
//   (codecs.py:188-242).  The warp takes 32 positions at a time: counts over
//   earlier chunks come from a shared prefix-count array P, counts among
//   earlier lanes of the chunk from a radix ballot rank.
//   at the halving (after position H-1) f'[v] = max(1, f[v] // 2) =
//   (c_v ? 16 c_v : 1), so the <= 2048 - H tail positions use
//   cum' = 16 P[s] + #{v < s : c_v = 0} plus 32 per earlier smaller tail
//   symbol, and total' = 16 H + #{v : c_v = 0} (+ 32 per tail position).
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// rank of each valid lane's W-bit symbol among the earlier valid lanes:
// less = #{earlier lanes with a smaller symbol}, returns the mask of earlier
// lanes with an equal symbol
template <int W>
__device__ __forceinline__ unsigned ballot_rank(uint32_t s, unsigned earlier, uint32_t& less) {
  unsigned eq = earlier;
  less = 0;
#pragma unroll
  for (int bit = W - 1; bit >= 0; --bit) {
    const bool one = (s >> bit) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, one);
    if (one) {
      less += __popc(eq & ~bb);
      eq &= bb;
    } else {
      eq &= ~bb;
    }
  }
  return eq;
}

template <int W>
__global__ void __launch_bounds__(128) k_rc_large_model(CodecArgs a, int64_t b0, int64_t nb) {
  constexpr int A = 1 << W;
  constexpr int H = halving_at<W>();
  constexpr int K = A / 32;  // counters per lane
  __shared__ __align__(16) uint32_t sP[4][A + 4];
  __shared__ __align__(16) uint32_t sH[4][A + 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bl = (int64_t)blockIdx.x * 4 + warp;
  if (bl >= nb) return;  // whole warp
  const int64_t b = b0 + bl;
  const StreamTab& st = *a.st;
  if (b >= st.nblocks) return;
  const int si = (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int n = (int)min(a.g.block, st.count[si] - start);
  const uint8_t* src = a.packed_in + st.byte_off[si] + start * W / 8;
  uint32_t* P = sP[warp];
  uint32_t* h = sH[warp];
  for (int v = lane; v <= A; v += 32) P[v] = 0;
  for (int v = lane; v < A; v += 32) h[v] = 0;
  __syncwarp();
  uint32_t* out = a.model + bl * a.g.block;
  const unsigned lt = lanemask_lt();
  const int nh = min(n, H);
  auto sym_at = [&](int i) -> uint32_t {
    if constexpr (W == 8) {
      return src[i];
    } else {
      const int64_t p = (int64_t)i * W;
      const uint32_t two = ((uint32_t)src[p >> 3] << 8) | src[(p >> 3) + 1];
      return (two >> (16 - (int)(p & 7) - W)) & (A - 1);
    }
  };
  for (int c0 = 0; c0 < nh; c0 += 32) {
    const int i = c0 + lane;
    const bool valid = i < nh;
    const uint32_t s = valid ? sym_at(i) : 0u;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    uint32_t less;
    const unsigned eq = ballot_rank<W>(s, lt & vmask, less);
    const uint32_t ps = P[s], cs = P[s + 1] - ps;
    if (valid) {
      out[i] = ((s + 32u * (ps + less)) << 16) | (1u + 32u * (cs + __popc(eq)));
      atomicAdd(&h[s], 1u);
    }
    __syncwarp();
    // P[u + 1] += #{chunk symbols <= u}: lane-local inclusive prefix + warp scan
    uint32_t cnt[K], run = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      run += h[lane * K + k];
      cnt[k] = run;
    }
    uint32_t base = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, base, o);
      if (lane >= o) base += t;
    }
    base -= run;  // exclusive
#pragma unroll
    for (int k = 0; k < K; ++k) {
      P[lane * K + k + 1] += base + cnt[k];
      h[lane * K + k] = 0;
    }
    __syncwarp();
  }
  if (n > H) {
    // the halved model (see above); h[v] <- #{u < v : c_u = 0}
    uint32_t z[K], run = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int v = lane * K + k;
      z[k] = run;
      run += (P[v + 1] == P[v]) ? 1u : 0u;
    }
    uint32_t base = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, base, o);
      if (lane >= o) base += t;
    }
    const uint32_t zeros_total = __shfl_sync(0xffffffffu, base, 31);
    base -= run;
#pragma unroll
    for (int k = 0; k < K; ++k) h[lane * K + k] = base + z[k];
    __syncwarp();
    for (int c0 = H; c0 < n; c0 += 32) {  // one pass for block <= 2048
      const int i = c0 + lane;
      const bool valid = i < n;
      const uint32_t s = valid ? sym_at(i) : 0u;
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      uint32_t less;
      const unsigned eq = ballot_rank<W>(s, lt & vmask, less);
      const uint32_t cs = P[s + 1] - P[s];
      const uint32_t f1 = cs ? 16u * cs : 1u;
      if (valid) out[i] = ((16u * P[s] + h[s] + 32u * less) << 16) | (f1 + 32u * __popc(eq));
    }
    if (lane == 0) a.model_total[bl] = 16u * (uint32_t)H + zeros_total;
  }
}

template <int W>
__global__ void __launch_bounds__(128) k_rc_large_code(CodecArgs a, int64_t b0, int64_t nb) {
  constexpr int A = 1 << W;
  constexpr int H = halving_at<W>();
  const uint32_t* __restrict__ magic = a.recip + W * kRecipLen;
  const int64_t bl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (bl >= nb) return;
  const int64_t b = b0 + bl;
  if (b > a.max_blocks) return;
  const StreamTab& st = *a.st;
  if (b >= st.nblocks) {
    a.sizes[b] = 0;
    return;
  }
  const int si = (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int n = (int)min(a.g.block, st.count[si] - start);
  const uint4* mv = reinterpret_cast<const uint4*>(a.model + bl * a.g.block);
  uint8_t* slot = a.slots + b * a.slot_bytes;
  RcEnc e;
  e.init(reinterpret_cast<uint32_t*>(slot + 4));
  const uint32_t tail_total = n > H ? a.model_total[bl] : 0u;
  const int nh = min(n, H) & ~3;  // whole quads before the halving: warp-converged fast loop
  for (int i4 = 0; i4 < nh; i4 += 4) {
    const unsigned mask = __activemask();
    const uint4 q = __ldg(mv + (i4 >> 2));
    const uint32_t qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t i = (uint32_t)(i4 + j);
      const uint32_t unit = div_recip(e.range, (uint32_t)A + 32u * i, __ldg(magic + i));
      e.encode_warp(unit, qv[j] >> 16, qv[j] & 0xFFFFu, mask);
    }
  }
  for (int i = nh; i < n; ++i) {  // the rest (and the tail after the halving)
    const uint32_t v = __ldg(a.model + bl * a.g.block + i);
    const uint32_t unit = i < H ? div_recip(e.range, (uint32_t)A + 32u * (uint32_t)i, __ldg(magic + i))
                                : e.range / (tail_total + 32u * (uint32_t)(i - H));
    e.encode(unit, v >> 16, v & 0xFFFFu);
  }
  const uint32_t len = e.finish();
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(len, 0, 0x0123);
  a.sizes[b] = (uint64_t)len + 4;
}

template <int W>
cudaError_t enc2_w(const CodecArgs& a, cudaStream_t s) {
  const int64_t total = a.max_blocks + 1;  // block ids 0 .. max_blocks
  // equal batches (a small last batch would leave the coder pass at low occupancy)
  const int64_t nbatch = (total + a.model_blocks - 1) / a.model_blocks;
  const int64_t per = (total + nbatch - 1) / nbatch;
  for (int64_t b0 = 0; b0 < total; b0 += per) {
    const int64_t nb = min(per, total - b0);
    k_rc_large_model<W><<<(unsigned)((nb + 3) / 4), 128, 0, s>>>(a, b0, nb);
    k_rc_large_code<W><<<(unsigned)((nb + 127) / 128), 128, 0, s>>>(a, b0, nb);
  }
  return cudaGetLastError();
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
  if (a.model_blocks > 0 && a.g.block <= 2048) {
    switch (w) {
      case 5: return enc2_w<5>(a, s);
      case 6: return enc2_w<6>(a, s);
      case 7: return enc2_w<7>(a, s);
      default: return enc2_w<8>(a, s);
    }
  }
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
