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
#include "rc_model.cuh"
#include "rc_tables.cuh"

namespace kvc {
namespace {

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
  // whole groups in the reciprocal-table phase, read as words when the stream
  // is word aligned (the second width stream of a mixed tensor need not be)
  const bool aligned = (reinterpret_cast<uintptr_t>(src) & 3) == 0;
  const int n1 = aligned ? min(n, kH) / GS : 0;
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
  if (o1 < o0 || o1 - o0 < 8 || (a.payload_bytes >= 0 && o1 > (uint64_t)a.payload_bytes)) {
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
      acc = (acc << W) | dec_symbol_small<W>(d, m, unit);
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
    acc = (acc << W) | dec_symbol_small<W>(d, m, unit);
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
