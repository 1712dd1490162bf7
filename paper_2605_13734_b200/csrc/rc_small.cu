// Adaptive range coder, small alphabets (w <= 4 bits, A = 2^w <= 16): the
// c=entropy hot path of the KIVI 2-bit profiles.
//
// Bit-exact with codecs.py:181-331 per block.  One thread codes one block;
// a warp's lanes walk their blocks in lockstep, which makes the first H =
// ceil((65536 - A) / 32) = 2048 symbols special: the model total at symbol i
// is exactly A + 32 i for every lane (codecs.py:227-232: no halving can
// happen before it), so
//   * `range // total` is a multiply by a per-position reciprocal from a
//     global read-only table (rc_tables.cuh; each 32-symbol group's entries
//     are prefetched into registers) plus one correction, and
//   * no halving check is needed inside that loop.
// The remainder of a longer block (after the first halving) and short tails
// run a generic per-symbol loop with hardware division.  Cumulative
// frequencies C[1..A-1] live in registers; lookup and update share the
// predicates (s >= k); the decoder's symbol search for A <= 4 is branch-free
// (compare x = code - low against unit * C[k]).  Renormalization moves all
// settled bytes in one branch-free step (rc_coder.cuh).
#include <cstdint>

#include "kernels.h"
#include "profile.h"
#include "rc_coder.cuh"
#include "rc_tables.cuh"

namespace kvc {
namespace {

constexpr int kH = 2048;  // first halving after symbol kH-1 for every A in 2..16

template <int W>
struct SModel {
  static constexpr int A = 1 << W;
  uint32_t C[A];  // C[k] = sum of f[0..k-1] for k = 1..A-1 (C[0] unused)
  uint32_t total;
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int k = 1; k < A; ++k) C[k] = k;
    total = A;
  }
  __device__ __forceinline__ void lookup(uint32_t s, uint32_t& lo, uint32_t& hi) const {
    lo = 0;
    hi = C[1];
#pragma unroll
    for (int k = 1; k < A; ++k) {
      const bool ge = s >= (uint32_t)k;
      lo = ge ? C[k] : lo;
      hi = ge ? (k + 1 < A ? C[k + 1] : total) : hi;
    }
  }
  __device__ __forceinline__ void add(uint32_t s) {  // f[s] += 32 (codecs.py:227-230)
#pragma unroll
    for (int k = 1; k < A; ++k) C[k] += (s < (uint32_t)k) ? 32u : 0u;
    total += 32u;
  }
  __device__ void halve() {  // codecs.py:234-242
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
  // decode: s with C[s] <= target = min(x / unit, total - 1); returns unit*C[s], unit*C[s+1]
  __device__ __forceinline__ uint32_t find(uint32_t x, uint32_t unit, uint32_t& plo, uint32_t& phi) const {
    if constexpr (A <= 4) {
      // x >= unit*C[k]  <=>  floor(x / unit) >= C[k]; the clamp to total-1 never
      // changes the symbol because C[A-1] <= total - 1
      uint32_t s = 0;
      plo = 0;
      phi = unit * C[1];
#pragma unroll
      for (int k = 1; k < A; ++k) {
        const uint32_t pk = unit * C[k];
        const uint32_t pn = unit * (k + 1 < A ? C[k + 1] : total);
        const bool ge = x >= pk;
        s += ge ? 1u : 0u;
        plo = ge ? pk : plo;
        phi = ge ? pn : phi;
      }
      return s;
    } else {
      uint32_t target = x / unit;
      target = target < total - 1 ? target : total - 1;
      uint32_t s = 0, lo = 0, hi = C[1];
#pragma unroll
      for (int k = 1; k < A; ++k) {
        const bool ge = target >= C[k];
        s += ge ? 1u : 0u;
        lo = ge ? C[k] : lo;
        hi = ge ? (k + 1 < A ? C[k + 1] : total) : hi;
      }
      plo = unit * lo;
      phi = unit * hi;
      return s;
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

// a group is a whole number of 32-bit words of symbols
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
  RcEnc e;
  e.init(reinterpret_cast<uint32_t*>(slot + 4));
  constexpr int GS = Grp<W>::kSyms, GW = Grp<W>::kWords;
  const int n1 = min(n, kH) / GS;  // whole groups in the reciprocal-table phase
  for (int gI = 0; gI < n1; ++gI) {
    uint32_t wd[GW], mg[GS];
#pragma unroll
    for (int k = 0; k < GW; ++k) wd[k] = __byte_perm(__ldg(src + gI * GW + k), 0, 0x0123);
#pragma unroll
    for (int j = 0; j < GS; ++j) mg[j] = __ldg(magic + gI * GS + j);
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const uint32_t s = sym_at<W>(wd, j);
      // m.total == A + 32*i until the first halving (warp-uniform)
      const uint32_t unit = div_recip(e.range, m.total, mg[j]);
      uint32_t lo, hi;
      m.lookup(s, lo, hi);
      e.encode(unit, lo, hi - lo);
      m.add(s);
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
      const uint32_t unit = (i < kH) ? div_recip(e.range, m.total, __ldg(magic + i)) : e.range / m.total;
      uint32_t lo, hi;
      m.lookup(s, lo, hi);
      e.encode(unit, lo, hi - lo);
      m.add(s);
      if (m.total >= 65536u) m.halve();
    }
  }
  const uint32_t len = e.finish();  // <= 4 bytes per symbol + 4 < slot capacity
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(len, 0, 0x0123);
  a.sizes[b] = (uint64_t)len + 4;
}

template <int W>
__device__ __forceinline__ uint32_t dec_symbol(RcDec& d, SModel<W>& m, uint32_t unit) {
  // code < low only in a malformed stream; x = 0 then yields symbol 0 with
  // the same bounds the reference's search gives for a negative target
  const uint32_t x = d.offset();
  uint32_t plo, phi;
  const uint32_t s = m.find(x, unit, plo, phi);
  d.advance(plo, phi);
  m.add(s);
  return s;
}

template <int W>
__global__ void __launch_bounds__(128) k_rc_small_decode(CodecArgs a) {
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
  uint32_t hdr = 0;
  for (int k = 0; k < 4; ++k) hdr = (hdr << 8) | src[k];
  if ((uint64_t)hdr + 4 != o1 - o0) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  RcDec d;
  d.init(src, a.payload_in + o1);
  SModel<W> m;
  m.init();
  uint8_t* dst = a.packed_out + st.byte_off[si] + start * W / 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 3) == 0;
  constexpr int GS = Grp<W>::kSyms, GW = Grp<W>::kWords;
  const int n1 = aligned ? min(n, kH) / GS : 0;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst);
  for (int gI = 0; gI < n1; ++gI) {
    uint32_t mg[GS];
#pragma unroll
    for (int j = 0; j < GS; ++j) mg[j] = __ldg(magic + gI * GS + j);
    uint64_t acc = 0;
    int nbits = 0, wo = 0;  // compile-time after unrolling
#pragma unroll
    for (int j = 0; j < GS; ++j) {
      const uint32_t unit = div_recip(d.range, m.total, mg[j]);
      acc = (acc << W) | dec_symbol<W>(d, m, unit);
      nbits += W;
      if (nbits >= 32) {
        nbits -= 32;
        dw[gI * GW + wo++] = __byte_perm((uint32_t)(acc >> nbits), 0, 0x0123);
      }
    }
  }
  int i = n1 * GS;
  if (i == kH) m.halve();
  uint64_t acc = 0;
  int nacc = 0, nout = i * W / 8;
  for (; i < n; ++i) {
    const uint32_t unit = (i < kH) ? div_recip(d.range, m.total, __ldg(magic + i)) : d.range / m.total;
    acc = (acc << W) | dec_symbol<W>(d, m, unit);
    if (m.total >= 65536u) m.halve();
    nacc += W;
    while (nacc >= 8) {
      nacc -= 8;
      dst[nout++] = (uint8_t)(acc >> nacc);
    }
  }
  // bytes consumed = 4 header + 4 priming + pulled; pulling past the block is
  // a truncated stream (codecs.py:283-288)
  if ((uint64_t)d.pulled() + 8 > o1 - o0) atomicOr(a.status, KVC_FLAG_CODEC);
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
