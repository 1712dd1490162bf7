// Adaptive range coder, large alphabets (w = 5..8 bits, A = 32..256): the
// c=entropy path of the 8-bit profiles (BASELINE config 5).
//
// Bit-exact with codecs.py:181-331 per block; one thread per block.  The
// order-0 model (codecs.py:188-242) is ONE u16 Fenwick tree of frequencies
// per thread in shared memory (512 B at A = 256), node pairs of thread t in
// word [q][t] so a warp's accesses are bank-conflict-free.  Every model step
// is a single root-to-leaf descent: the nodes it rejects are exactly the
// nodes the frequency update touches, so the update is a predicated store
// right after each read (LModel::find_scaled_upd / lookup_upd).  The encoder
// walks the symbol's bits (all loads independent); the decoder compares
// against the code and loads both children of the next level while the
// current comparison resolves.  Node values never exceed the running total
// (< 2^16): the bump that reaches 2^16 skips the stores and takes the
// halving path (frequencies recovered from the tree, incremented, halved,
// tree rebuilt).  Before the first halving `range // total` uses the
// reciprocal table (rc_tables.cuh) from constant memory.
#include <cstdint>
#include <mutex>

#include "kernels.h"
#include "profile.h"
#include "rc_coder.cuh"
#include "rc_tables.cuh"

namespace kvc {
namespace {

constexpr int kLThreads = 224;  // 7 warps: two CTAs of 112 KB trees fill the SM (14 warps)

// rows w = 5..8 of the reciprocal tables (rc_tables.cuh) in constant memory:
// read with the warp-uniform position index through the constant cache, off
// the load/store path and the per-symbol critical path
__constant__ uint32_t c_recip_l[4][kRecipLen];

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
  // ---- descent with the update folded in -------------------------------
  // The descent that locates symbol s visits, at each level, the node
  // covering [pos, pos + bit).  It is rejected exactly when s lies inside,
  // and those rejected nodes plus the root are the nodes a Fenwick update of
  // s touches, so f[s] += 32 is a predicated store of (value + 32) right
  // after each rejected node is read: no separate update walk.  The root
  // (node A) is the running total, kept in a register and written back only
  // before a halving.  Node addresses: with pos even, node pos + bit sits at
  // byte pos * 256 + off(bit) of the thread's column (pair layout above).
  __device__ __forceinline__ static constexpr uint32_t off(uint32_t bit) {
    return bit >= 2 ? (bit / 2 - 1) * (4 * kLThreads) + 2 : 0;
  }
  // 32-bit shared-window address of the thread's column (no generic pointer
  // arithmetic in the descents)
  __device__ __forceinline__ uint32_t col() const { return (uint32_t)__cvta_generic_to_shared(tree); }
  // 16-bit nodes moved through 32-bit registers (zero-extended on load,
  // truncated on store): selects between loaded nodes stay plain SELs instead
  // of 16-bit merges plus a mask
  __device__ __forceinline__ static uint32_t lds16(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  }
  __device__ __forceinline__ static void sts16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "r"(v));
  }
  // decoder: s = largest with unit * prefix(s) <= x; plo / phi as find_scaled
  template <bool UPD>
  __device__ __forceinline__ uint32_t find_scaled_upd(uint32_t x, uint32_t unit, uint32_t& plo, uint32_t& phi) {
    // One level of lookahead: while level k's comparison resolves, both
    // candidate nodes of level k-1 (the left child if rejected, the right
    // if accepted) are already being loaded, so the dependent chain per
    // level is compare + select instead of a shared-memory round trip.
    const uint32_t q0 = col();
    uint32_t q = q0;
    uint32_t acc = 0, rej = unit * total;
    uint32_t t = lds16(q + off(A / 2));
#pragma unroll
    for (int k = W - 1; k >= 0; --k) {
      const uint32_t bit = 1u << k;
      uint32_t t_rej = 0, t_acc = 0;
      if (k > 0) {
        t_rej = lds16(q + off(bit / 2));
        t_acc = lds16(q + bit * (2 * kLThreads) + off(bit / 2));
      }
      const uint32_t v = acc + unit * t;
      if (v <= x) {
        acc = v;
        q += bit * (2 * kLThreads);
        t = t_acc;
      } else {
        rej = v;
        if (UPD) sts16(q + off(bit), t + 32u);
        t = t_rej;
      }
    }
    plo = acc;
    phi = rej;
    return (q - q0) / (2 * kLThreads);  // pos
  }
  // encoder: cum = prefix(s), freq = f[s]; the path is s's bits, so every
  // node address is known up front and the loads issue together
  template <bool UPD>
  __device__ __forceinline__ void lookup_upd(uint32_t s, uint32_t& cum, uint32_t& fr) {
    // all loads first, then the stores: the path's nodes are distinct, and a
    // store between two loads would serialize the loads behind its data
    const uint32_t q0 = col();
    uint32_t na[W], t[W];
#pragma unroll
    for (int k = W - 1; k >= 0; --k) {
      const uint32_t bit = 1u << k;
      const uint32_t pre = s & ~(2 * bit - 1);  // pos at this level
      na[k] = q0 + pre * (2 * kLThreads) + off(bit);
      t[k] = lds16(na[k]);
    }
    uint32_t acc = 0, hi = total;
#pragma unroll
    for (int k = W - 1; k >= 0; --k) {
      const uint32_t bit = 1u << k;
      if (s & bit) {
        acc += t[k];
      } else {
        hi = acc + t[k];  // the last rejected node ends at s + 1
        if (UPD) sts16(na[k], t[k] + 32u);
      }
    }
    cum = acc;
    fr = hi - acc;
  }
  // f[s] += 32 after a descent: the total, or the halving (codecs.py:227-242)
  __device__ __forceinline__ void after_upd(uint32_t s, bool halving) {
    if (halving) {
      set(A, total);  // the root, not maintained by the descents
      halve_with(s);
    } else {
      total += 32u;
    }
  }

};

template <int W>
__global__ void __launch_bounds__(kLThreads) k_rc_large_encode(CodecArgs a) {
  constexpr int A = 1 << W;
  constexpr int H = halving_at<W>();
  extern __shared__ __align__(16) uint16_t lsm[];
  const uint32_t* magic = c_recip_l[W - 5];
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
  int i = 0;
  if ((reinterpret_cast<uintptr_t>(src) & 3u) == 0) {
    // positions before the halving: symbols from a 64-bit window refilled
    // with big-endian words loaded one refill ahead (block starts are 4-byte
    // aligned), the model total is 2^W + 32 i (warp-uniform), and the
    // converged-lane coder (votes instead of a divergent underflow branch)
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(src);
    const int nw = (n * W + 31) / 32;
    int wi = 0;
    uint32_t nxt = __ldg(wp);
    uint64_t win = 0;
    int nbits = 0;
    const int n1 = min(n, H - 1);
    if constexpr (W == 8) {
      // four symbols per loaded word (byte j = symbol 4q + j), unrolled; the
      // next word is loaded one step ahead
      const int n4 = n1 & ~3;
      for (; i < n4; i += 4) {
        const unsigned mask = __activemask();  // the same lanes code all four
        const uint32_t cur = nxt;
        nxt = __ldg(wp + min(++wi, nw - 1));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t s = (cur >> (8 * j)) & 0xFFu;
          uint32_t cum, fr;
          m.template lookup_upd<true>(s, cum, fr);
          e.encode_warp(div_recip(e.range, (uint32_t)A + 32u * (uint32_t)(i + j), magic[i + j]), cum, fr, mask);
          m.total += 32u;
        }
      }
      // the word-window loop below continues at word wi (nbits == 0)
    }
    for (; i < n1; ++i) {
      const unsigned mask = __activemask();
      if (nbits < W) {
        win |= (uint64_t)__byte_perm(nxt, 0, 0x0123) << (32 - nbits);
        nbits += 32;
        nxt = __ldg(wp + min(++wi, nw - 1));
      }
      const uint32_t s = (uint32_t)(win >> (64 - W));
      win <<= W;
      nbits -= W;
      uint32_t cum, fr;
      m.template lookup_upd<true>(s, cum, fr);
      e.encode_warp(div_recip(e.range, (uint32_t)A + 32u * (uint32_t)i, magic[i]), cum, fr, mask);
      m.total += 32u;
    }
  }
  // the rest (the halving position and after, or an unaligned block): the
  // byte reader from bit i * W
  const int64_t bit0 = (int64_t)i * W;
  int pos = (int)(bit0 >> 3);
  uint32_t buf = 0;
  int nb = 0;
  if (bit0 & 7) {
    buf = __ldg(src + pos++);
    nb = 8 - (int)(bit0 & 7);
  }
  for (; i < n; ++i) {
    if (nb < W) {
      buf = (buf << 8) | __ldg(src + pos++);
      nb += 8;
    }
    nb -= W;
    const uint32_t s = (buf >> nb) & (A - 1);
    const bool hv = m.total + 32u >= 65536u;  // this bump halves (i == H - 1)
    uint32_t cum, fr;
    if (hv) {
      m.template lookup_upd<false>(s, cum, fr);
    } else {
      m.template lookup_upd<true>(s, cum, fr);
    }
    const uint32_t unit = (i < H) ? div_recip(e.range, m.total, magic[i]) : e.range / m.total;
    e.encode(unit, cum, fr);
    m.after_upd(s, hv);
  }
  const uint32_t nout = e.finish();
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(nout, 0, 0x0123);
  a.sizes[b] = (uint64_t)nout + 4;
}

template <int W>
__global__ void __launch_bounds__(kLThreads) k_rc_large_decode(CodecArgs a) {
  constexpr int A = 1 << W;
  constexpr int H = halving_at<W>();
  extern __shared__ __align__(16) uint16_t lsm[];
  const uint32_t* magic = c_recip_l[W - 5];
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) return;
  const int si = (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
  if (st.w[si] != W) return;
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int n = (int)min(a.g.block, st.count[si] - start);
  const uint64_t o0 = a.offsets_in[b], o1 = a.offsets_in[b + 1];
  if (o1 < o0 || o1 - o0 < 8 || (a.payload_bytes >= 0 && o1 > (uint64_t)a.payload_bytes)) {
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
  int i = 0;
  if (word_out) {
    // positions before the halving: total 2^W + 32 i, reciprocal loaded one
    // symbol ahead, updates folded into the descent, one word out per 32 bits
    const int n1 = min(n, H - 1);
    if constexpr (W == 8) {
      // four symbols per word: unrolled, one store per four
      const int n4 = n1 & ~3;
      for (; i < n4; i += 4) {
        const unsigned mask = __activemask();  // the same lanes decode all four
        uint32_t wd = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t unit = div_recip(d.range, (uint32_t)A + 32u * (uint32_t)(i + j), magic[i + j]);
          uint32_t plo, phi;
          const uint32_t s = m.template find_scaled_upd<true>(d.offset(), unit, plo, phi);
          d.advance_warp(plo, phi, mask);
          m.total += 32u;
          wd |= s << (8 * j);  // little-endian byte j = symbol i + j
        }
        *reinterpret_cast<uint32_t*>(dst + nout) = wd;
        nout += 4;
      }
    }
    for (; i < n1; ++i) {
      const unsigned mask = __activemask();
      const uint32_t unit = div_recip(d.range, (uint32_t)A + 32u * (uint32_t)i, magic[i]);
      uint32_t plo, phi;
      const uint32_t s = m.template find_scaled_upd<true>(d.offset(), unit, plo, phi);
      d.advance_warp(plo, phi, mask);
      m.total += 32u;
      acc = (acc << W) | s;
      nacc += W;
      if (nacc >= 32) {
        nacc -= 32;
        *reinterpret_cast<uint32_t*>(dst + nout) = __byte_perm((uint32_t)(acc >> nacc), 0, 0x0123);
        nout += 4;
      }
    }
  }
  for (; i < n; ++i) {
    const unsigned mask = __activemask();
    const uint32_t unit = (i < H) ? div_recip(d.range, m.total, magic[i]) : d.range / m.total;
    // code < low only in a malformed stream; offset() reads 0 -> symbol 0
    uint32_t plo, phi;
    const bool hv = m.total + 32u >= 65536u;  // this bump halves (uniform: i == H - 1)
    const uint32_t s = hv ? m.template find_scaled_upd<false>(d.offset(), unit, plo, phi)
                          : m.template find_scaled_upd<true>(d.offset(), unit, plo, phi);
    d.advance_warp(plo, phi, mask);
    m.after_upd(s, hv);
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

cudaError_t upload_large_recip(const uint32_t* rows) {
  return cudaMemcpyToSymbol(c_recip_l, rows, sizeof(c_recip_l));
}

cudaError_t launch_rc_large_encode(const CodecArgs& a, int w, cudaStream_t s) {
  if (cudaError_t ce = ensure_recip_tables(); ce != cudaSuccess) return ce;
  ProfScope ps("rc_encode", s);
  switch (w) {
    case 5: return enc_w<5>(a, s);
    case 6: return enc_w<6>(a, s);
    case 7: return enc_w<7>(a, s);
    default: return enc_w<8>(a, s);
  }
}

cudaError_t launch_rc_large_decode(const CodecArgs& a, int w, cudaStream_t s) {
  if (cudaError_t ce = ensure_recip_tables(); ce != cudaSuccess) return ce;
  ProfScope ps("rc_decode", s);
  switch (w) {
    case 5: return dec_w<5>(a, s);
    case 6: return dec_w<6>(a, s);
    case 7: return dec_w<7>(a, s);
    default: return dec_w<8>(a, s);
  }
}

}  // namespace kvc
