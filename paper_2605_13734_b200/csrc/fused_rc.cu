// Fused quantize + range-code kernels for the entropy profiles (KIVI-style
// 2-bit K/V, BASELINE config 2): one thread per codec block.
//
// The unfused path quantizes into a packed symbol stream in HBM (one kernel,
// HBM-bound), then range-codes it (another kernel, issue-bound), and the two
// barely overlap because each fills every SM.  Here the coder thread produces
// its own symbols: it reads the block's bf16 values, computes each group's
// scale / zero exactly as quantize.py:146-154 (numerics.cuh), and feeds the
// symbols straight into the adaptive range coder (rc_model.cuh, rc_coder.cuh).
// The HBM traffic (bf16 in, coded bytes out) is spread over the coder's run
// time instead of being a separate pass.  Decode is the mirror image: decoded
// symbols are dequantized in registers and written as KV.
//
// Payload bytes, block sizes, scales and zeros are identical to the unfused
// path (and the reference): a block is the same 2048 consecutive symbols of
// the single width stream (codecs.py:339-345), coded independently.
//
// Two layouts:
//   * per-token groups (q=uniform): block b = rows [16b, 16b+16) of the
//     (L*H*T, 128) matrix; the thread walks its rows group by group.
//   * per-channel groups (q=uchan): the stream is the (L,H,C,T) transpose, so
//     block b = (head, channel, token chunk).  Threads are assigned so the 32
//     lanes of a warp take 32 adjacent channels of the same head and token
//     chunk; each 32-token group is loaded as a coalesced 32x32 tile and
//     transposed through shared memory (decode: the reverse).
//
// Requirements (fused_rc_applicable): entropy codec, one width w <= 4,
// identity transform, head_dim 128, groups of 32, bf16 input, block <= 2048
// (no model halving inside a block), and for uchan T % block == 0.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <mutex>

#include "kernels.h"
#include "numerics.cuh"
#include "profile.h"
#include "rc_coder.cuh"
#include "rc_model.cuh"
#include "rc_tables.cuh"

namespace kvc {
namespace {

constexpr int kFThreads = 128;
__device__ const uint32_t kZeroBlock[4] = {0, 0, 0, 0};

// floor(2^32 / (2^w + 32 i)) for w = 1..4, i < kH: the per-position
// reciprocals of rc_tables.cuh in constant memory, so the coder loops read
// them with a warp-uniform index straight from the constant cache (no vector
// registers, no LSU instruction)
__constant__ uint32_t c_recip[4][kRecipLen];

// bf16 pair helpers (NaN-propagating min / max of packed pairs)
__device__ __forceinline__ uint32_t bmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint16_t half_at(uint2 v, int k) {
  const uint32_t w = (k & 2) ? v.y : v.x;
  return (uint16_t)(w >> (16 * (k & 1)));
}
// packed fp32x2 add / multiply in PTX with an explicit .rn (never contracted
// into an FFMA2)
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// min / max of 32 bf16 values packed in 16 words (exact; a NaN propagates)
__device__ __forceinline__ void minmax_words(const uint32_t* w, float& mn, float& mx) {
  uint32_t lo = w[0], hi = w[0];
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    lo = bmin2(lo, w[k]);
    hi = bmax2(hi, w[k]);
  }
  mn = fminf(bf16_lo(lo), bf16_hi(lo));
  mx = fmaxf(bf16_lo(hi), bf16_hi(hi));
  if (!(isfinite(bf16_lo(lo)) && isfinite(bf16_hi(lo)) && isfinite(bf16_lo(hi)) && isfinite(bf16_hi(hi))))
    mn = __int_as_float(0x7FC00000);  // surfaces as NaN below
}

// 32 symbols of one group (quantize.py:146-154) from bf16 values given as
// value(i), packed as nibbles (symbol j at bits 4(j%8) of word j/8) so the
// coder loop walks them with static shifts.
//
// The packing is an IMAD chain over the magic-rounded floats' bit patterns
// (their low bits are the symbols; the constant magic part is subtracted once
// per word), so it issues on the FMA pipe.  When every lane's group needs no
// clipping -- the exact quotients of its min and max already round into
// [0, levels], which by monotonicity covers the whole group -- the clip is
// skipped (rint of anything in [-0.5, levels + 0.5) lands in range).
template <class Val>
__device__ __forceinline__ void quant32(Val&& value, float mn, float mx, int w, float rl, __half& s16, __half& z16,
                                        uint32_t& flags, uint32_t* nib, unsigned mask) {
  GroupQ q = group_setup(mn, mx, w, rl, s16, z16, flags);
  constexpr uint32_t kFix = kMagicBits * 0x11111111u;  // sum of kMagicBits << 4j, j < 8 (mod 2^32)
  bool easy = false;
  if (q.mode == 0) {
    auto quo = [&](float v) {  // the exact fp32 quotient (v - z) / s
      const float d = __fsub_rn(v, q.z);
      const float q0 = __fmul_rn(d, q.r);
      return __fmaf_rn(__fmaf_rn(-q0, q.s, d), q.r, q0);
    };
    easy = quo(mn) >= -0.5f && quo(mx) < q.lv + 0.5f;
  }
  if (__all_sync(mask, easy)) {
    // two values per FADD2 / FMUL2 / FFMA2 (lane-wise the scalar roundings)
    const float2 nz = make_float2(-q.z, -q.z), r2 = make_float2(q.r, q.r), ns = make_float2(-q.s, -q.s);
    const float2 mg = make_float2(kMagicRound, kMagicRound);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 d = f2add(make_float2(value(8 * k + j), value(8 * k + j + 1)), nz);
        const float2 q0 = f2mul(d, r2);
        const float2 q1 = f2add(__ffma2_rn(__ffma2_rn(q0, ns, d), r2, q0), mg);
        acc += __float_as_uint(q1.x) * (1u << (4 * j)) + __float_as_uint(q1.y) * (1u << (4 * j + 4));
      }
      nib[k] = acc - kFix;
    }
  } else if (q.mode == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += __float_as_uint(quant_magic(value(8 * k + j), q)) * (1u << (4 * j));
      nib[k] = acc - kFix;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) nib[k] = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) nib[i >> 3] |= quant_one(value(i), q) << (4 * (i & 7));
  }
}

__device__ __forceinline__ uint32_t pick4(const uint32_t* v, int k) {
  return k == 0 ? v[0] : k == 1 ? v[1] : k == 2 ? v[2] : v[3];
}

// range-code the 32 symbols of one group at block positions i0 .. i0+31
// (i0 + 32 <= kH: the model total is the warp-uniform 2^W + 32 i)
template <int W>
__device__ __forceinline__ void encode32(RcEnc& e, SModel<W>& m, int i0, const uint32_t* nib, unsigned mask) {
  const uint32_t* tab = c_recip[W - 1] + i0;
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    const uint32_t cur = pick4(nib, k);
    const uint32_t base = (1u << W) + 32u * (uint32_t)(i0 + 8 * k);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t t = cur << (28 - 4 * j);  // symbol j in the top nibble
      const uint32_t tot = base + 32u * j;
      const uint32_t unit = div_recip(e.range, tot, tab[8 * k + j]);
      uint32_t lo, hi;
      m.step_top(t, tot, lo, hi);
      e.encode_warp(unit, lo, hi - lo, mask);
    }
  }
}

// decode 32 symbols of one group, dequantize (quantize.py:178) and hand each
// run of 8 values to sink(k, v) (values 8k .. 8k+7)
template <int W, class Sink>
__device__ __forceinline__ void decode32(RcDec& d, SModel<W>& m, int i0, float s, float z, unsigned mask,
                                         Sink&& sink) {
  const uint32_t* tab = c_recip[W - 1] + i0;
  float val[W <= 2 ? (1 << W) : 1];  // dequantized value of each symbol (quantize.py:178)
  if constexpr (W <= 2) {
#pragma unroll
    for (int q = 0; q < (1 << W); ++q) val[q] = dequant((uint32_t)q, s, z);
  }
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    const uint32_t base = (1u << W) + 32u * (uint32_t)(i0 + 8 * k);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t tot = base + 32u * j;
      const uint32_t unit = div_recip(d.range, tot, tab[8 * k + j]);
      uint32_t plo, phi;
      // code < low only in a malformed stream; offset() reads 0 then
      if constexpr (W <= 2) {
        v[j] = m.dstep(d.offset(), unit, tot, val, plo, phi);
      } else {
        const uint32_t sym = m.find_t(d.offset(), unit, tot, plo, phi);
        m.add_only(sym);
        v[j] = dequant(sym, s, z);
      }
      d.advance_warp(plo, phi, mask);
    }
    sink(k, v);
  }
}

// store a warp's 32 staged rows (row l of the tile = 32 values for lane l's
// destination `dst`) so each 16-byte store instruction covers whole 32-byte
// sectors: lanes 4r..4r+3 (bf16) or 8r..8r+7 (f32) write row r together
template <typename Tout, int kStride>
__device__ __forceinline__ void store_rows(const uint8_t* tile, Tout* dst, int lane, bool live) {
  constexpr int kPer = 32 * (int)sizeof(Tout) / 16;  // 16-byte chunks per row: 4 or 8
  constexpr int kRowsPer = 32 / kPer;                // rows per instruction
  const uint64_t mine = reinterpret_cast<uint64_t>(dst);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int rr = k * kRowsPer + lane / kPer, ch = lane % kPer;
    const uint64_t p = __shfl_sync(0xffffffffu, mine, rr);
    const bool ok = __shfl_sync(0xffffffffu, live, rr);
    // streaming stores (evict-first): the decoded KV is written once and must not
    // push the coded blocks, still being read, out of L2
    if (ok) __stcs(reinterpret_cast<uint4*>(p) + ch, *reinterpret_cast<const uint4*>(tile + rr * kStride + 16 * ch));
  }
}

constexpr int kTileStrideB = 80;   // 32 bf16 + 16 B pad: conflict-free 16 B row access
constexpr int kTileStrideF = 144;  // 32 f32 + 16 B pad

template <typename Tout>
__device__ __forceinline__ void stage_value(uint8_t* tile, int row, int col, int stride, float v) {
  if constexpr (sizeof(Tout) == 2)
    *reinterpret_cast<__nv_bfloat16*>(tile + row * stride + 2 * col) = __float2bfloat16_rn(v);
  else
    *reinterpret_cast<float*>(tile + row * stride + 4 * col) = v;
}

// ------------------------------------------------------------- per token
// one block's groups; FULL = every lane of the warp codes a full block (the
// warp-uniform votes then use a constant mask, with no divergence checks)
template <int W, bool FULL, bool PAGED>
__device__ __forceinline__ void tok_encode_groups(const FusedArgs& a, const uint4* src, int64_t r0, int ngr, RcEnc& e,
                                                  SModel<W>& m, uint32_t& flags, bool& nonfinite) {
  const float rl = a.rl[W];
  uint64_t sacc = 0, zacc = 0;
  const uint4* rp = src;  // PAGED: the current token row, from its page
#pragma unroll 1
  for (int gi = 0; gi < ngr; ++gi) {
    const unsigned mask = FULL ? 0xffffffffu : __activemask();
    if constexpr (FULL) __syncwarp();  // proves convergence: no BRA.DIV before each vote
    if (PAGED && (gi & 3) == 0) {
      const int64_t r = r0 + (gi >> 2), lh = r / a.g.T;
      rp = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.kv) + out_index(a, lh, r - lh * a.g.T, 0));
    }
    const uint4* gp = PAGED ? rp + (gi & 3) * 4 : src + gi * 4;
    uint32_t wv[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = __ldcs(gp + k);  // read once: evict-first, keeps the coded slots in L2
      wv[4 * k] = v.x; wv[4 * k + 1] = v.y; wv[4 * k + 2] = v.z; wv[4 * k + 3] = v.w;
    }
    if (gi + 1 < ngr && (!PAGED || (gi & 3) != 3)) {  // next group's 64 bytes (paged: within the row)
      prefetch_l1(gp + 4);
      prefetch_l1(gp + 6);
    }
    float mn, mx;
    minmax_words(wv, mn, mx);
    nonfinite |= isnan(mn);
    __half s16, z16;
    uint32_t nib[4];
    quant32([&](int i) { return (i & 1) ? bf16_hi(wv[i >> 1]) : bf16_lo(wv[i >> 1]); }, mn, mx, W, rl, s16, z16, flags,
            nib, mask);
    sacc = (sacc >> 16) | ((uint64_t)__half_as_ushort(s16) << 48);
    zacc = (zacc >> 16) | ((uint64_t)__half_as_ushort(z16) << 48);
    if ((gi & 3) == 3) {  // a row's four groups: scales[row*4 .. +3]
      *reinterpret_cast<uint64_t*>(a.scales + r0 * 4 + gi - 3) = sacc;
      *reinterpret_cast<uint64_t*>(a.zeros + r0 * 4 + gi - 3) = zacc;
    }
    encode32<W>(e, m, gi * 32, nib, mask);
  }
}

template <int W>
__global__ void __launch_bounds__(kFThreads, 8) k_fused_tok_encode(const FusedArgs a) {
  const Geo& g = a.g;
  const int64_t gt = (int64_t)blockIdx.x * kFThreads + threadIdx.x;
  if (gt > a.max_blocks) return;
  const int64_t nrows = g.LH * g.T;
  const int R = (int)(g.block / 128);
  const int64_t nblocks = (nrows + R - 1) / R;
  if (gt >= nblocks) {
    a.sizes[gt] = 0;
    return;
  }
  // paged input with whole blocks per head: threads take blocks token-range
  // major (l, token block, head), so a warp reads every head of its tokens
  // (whole 2 KB rows of the page pool); block b's output is b's either way
  int64_t b = gt;
  if (a.paged && g.T % R == 0) {
    const int64_t nbh = g.T / R, per_layer = g.H * nbh, l = gt / per_layer, rem = gt - l * per_layer;
    const int64_t tb = rem / g.H, h = rem - tb * g.H;
    b = (l * g.H + h) * nbh + tb;
  }
  const int64_t r0 = b * R;
  const int nr = (int)min((int64_t)R, nrows - r0);
  const uint4* src = reinterpret_cast<const uint4*>(a.kv) + r0 * 16;
  uint8_t* slot = a.slots + b * a.slot_bytes;
  RcEnc e;
  e.init(reinterpret_cast<uint32_t*>(slot + 4));
  SModel<W> m;
  m.init();
  uint32_t flags = 0;
  bool nonfinite = false;
  // only the warp holding the ragged last block (or lanes past the end) runs
  // the activemask variant
  const int64_t wlast = b - (threadIdx.x & 31) + 31;
  const bool full = wlast < nblocks - 1 || (wlast == nblocks - 1 && nrows % R == 0);
  if (a.paged)
    tok_encode_groups<W, false, true>(a, src, r0, nr * 4, e, m, flags, nonfinite);
  else if (full)
    tok_encode_groups<W, true, false>(a, src, r0, nr * 4, e, m, flags, nonfinite);
  else
    tok_encode_groups<W, false, false>(a, src, r0, nr * 4, e, m, flags, nonfinite);
  const uint32_t len = e.finish();
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(len, 0, 0x0123);
  a.sizes[b] = (uint64_t)len + 4;
  if (nonfinite) flags |= KVC_FLAG_NONFINITE_INPUT;
  if (flags) atomicOr(a.status, flags);
}

// header / bounds checks shared by the decoders; false = malformed block,
// which then decodes a zero stream (so warp-cooperative stores stay intact)
__device__ __forceinline__ bool open_block(const FusedArgs& a, int64_t b, RcDec& d, int64_t& avail) {
  const uint64_t o0 = a.offsets_in[b], o1 = a.offsets_in[b + 1];
  bool ok = o1 >= o0 && o1 - o0 >= 8 && (a.payload_bytes < 0 || o1 <= (uint64_t)a.payload_bytes);
  if (ok) {
    const uint8_t* src = a.payload_in + o0;
    const uint32_t hdr = ((uint32_t)src[0] << 24) | ((uint32_t)src[1] << 16) | ((uint32_t)src[2] << 8) | src[3];
    ok = (uint64_t)hdr + 4 == o1 - o0;
    if (ok) {
      d.init(src, a.payload_in + o1);
      avail = (int64_t)(o1 - o0);
      return true;
    }
  }
  const uint8_t* z = reinterpret_cast<const uint8_t*>(kZeroBlock);
  d.init(z, z + 16);
  avail = 16;
  return false;
}

template <int W, typename Tout>
__global__ void __launch_bounds__(kFThreads) k_fused_tok_decode(const FusedArgs a) {
  constexpr int kStride = sizeof(Tout) == 2 ? kTileStrideB : kTileStrideF;
  __shared__ __align__(16) uint8_t tiles[kFThreads / 32][32 * kStride];
  const Geo& g = a.g;
  const int64_t b = (int64_t)blockIdx.x * kFThreads + threadIdx.x;
  const int64_t nrows = g.LH * g.T;
  const int R = (int)(g.block / 128);
  const int64_t nblocks = (nrows + R - 1) / R;
  const int64_t wb0 = b - (threadIdx.x & 31);
  if (wb0 >= nblocks) return;  // whole warp idle
  const int lane = threadIdx.x & 31;
  uint8_t* tile = tiles[threadIdx.x >> 5];
  const bool real = b < nblocks;
  RcDec d;
  int64_t blen = 16;
  uint32_t flags = 0;
  if (real) {
    if (!open_block(a, b, d, blen)) flags |= KVC_FLAG_CODEC;
  } else {
    const uint8_t* z = reinterpret_cast<const uint8_t*>(kZeroBlock);
    d.init(z, z + 16);
  }
  const int64_t r0 = b * R;
  const int nr = real ? (int)min((int64_t)R, nrows - r0) : 0;
  int64_t lh = real ? r0 / g.T : 0, t = real ? r0 - lh * g.T : 0;
  SModel<W> m;
  m.init();
  float chk = 0.0f;
  uint32_t pulled = 0;
  const uint2* sp = reinterpret_cast<const uint2*>(a.scales_in) + (real ? r0 : 0);
  const uint2* zp = reinterpret_cast<const uint2*>(a.zeros_in) + (real ? r0 : 0);
  uint2 s4 = __ldg(sp), z4 = __ldg(zp);
#pragma unroll 1
  for (int row = 0; row < R; ++row) {  // warp-uniform trip count; rows >= nr store nothing
    const bool live = row < nr;
    Tout* orow = reinterpret_cast<Tout*>(a.out) + (live ? out_index(a, lh, t, 0) : 0);
    const uint2 s4n = (row + 1 < nr) ? __ldg(sp + row + 1) : s4;  // next row's scales, early
    const uint2 z4n = (row + 1 < nr) ? __ldg(zp + row + 1) : z4;
#pragma unroll 1
    for (int gq = 0; gq < 4; ++gq) {
      const float s = __half2float(__ushort_as_half(half_at(s4, gq)));
      const float z = __half2float(__ushort_as_half(half_at(z4, gq)));
      // z + sym*s is non-finite for some symbol iff s or z is (|z|, s <= 65504,
      // sym <= 15: no fp32 overflow; 0*inf is NaN), so one check per group
      if (live && !(isfinite(s) && isfinite(z))) chk = 1.0f;
      decode32<W>(d, m, row * 128 + gq * 32, s, z, 0xffffffffu, [&](int k, const float* v) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          stage_value<Tout>(tile, lane, 8 * k + i, kStride, v[i]);
        }
      });
      __syncwarp();
      store_rows<Tout, kStride>(tile, orow + gq * 32, lane, live);
      __syncwarp();
    }
    if (live) pulled = d.pulled();
    s4 = s4n;
    z4 = z4n;
    if (++t == g.T) {
      t = 0;
      ++lh;
    }
  }
  if (chk != 0.0f) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
  // bytes consumed = 4 header + 4 priming + pulled (codecs.py:283-288)
  if (real && !(flags & KVC_FLAG_CODEC) && (int64_t)pulled + 8 > blen) flags |= KVC_FLAG_CODEC;
  if (flags) atomicOr(a.status, flags);
}

// ----------------------------------------------------------- per channel
// global thread gt -> (head lh, token chunk tc, channel c): a warp = 32
// adjacent channels of one head and chunk; block id b = (lh*128 + c)*nbt + tc
struct ChanMap {
  int64_t lh, tc, b;
  int c;
};
__device__ __forceinline__ ChanMap chan_map(int64_t gt, int64_t nbt) {
  ChanMap r;
  r.lh = gt / (128 * nbt);
  const int64_t rem = gt - r.lh * 128 * nbt;
  r.tc = rem >> 7;
  r.c = (int)(rem & 127);
  r.b = (r.lh * 128 + r.c) * nbt + r.tc;
  return r;
}

template <int W, bool PAGED>
__global__ void __launch_bounds__(kFThreads, 8) k_fused_chan_encode(const FusedArgs a) {
  __shared__ __align__(16) uint8_t tiles[kFThreads / 32][32 * kTileStrideB];
  const Geo& g = a.g;
  const int64_t gt = (int64_t)blockIdx.x * kFThreads + threadIdx.x;
  const int64_t nbt = g.T / g.block;
  const int64_t nblocks = g.LH * 128 * nbt;  // a multiple of the CTA size
  if (gt >= nblocks) {
    if (gt <= a.max_blocks) a.sizes[gt] = 0;
    return;
  }
  // paged input: (l, token chunk, head, channel) order -- the warps in flight
  // cover every head of a token range (whole 2 KB rows of the page pool)
  int64_t gm = gt;
  if (PAGED) {
    const int64_t c = gt & 127, q = gt >> 7, h = q % g.H, q2 = q / g.H, tc = q2 % nbt, l = q2 / nbt;
    gm = ((l * g.H + h) * nbt + tc) * 128 + c;
  }
  const ChanMap cm = chan_map(gm, nbt);
  const int lane = threadIdx.x & 31;
  const int c0 = cm.c - lane;
  uint8_t* tile = tiles[threadIdx.x >> 5];
  const int64_t t0 = cm.tc * g.block;
  // lane's token row for group gi: token t0 + 32 gi + lane, channels c0 .. c0+31
  const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.kv) +
                                                    ((cm.lh * g.T + t0 + lane) * 128 + c0));
  // paged cache: lane's token row of group gi from its page
  const auto paged_row = [&](int gi) {
    return reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.kv) +
                                          out_index(a, cm.lh, t0 + (int64_t)gi * 32 + lane, c0));
  };
  uint8_t* slot = a.slots + cm.b * a.slot_bytes;
  RcEnc e;
  e.init(reinterpret_cast<uint32_t*>(slot + 4));
  SModel<W> m;
  m.init();
  const float rl = a.rl[W];
  uint32_t flags = 0;
  bool nonfinite = false;
  const int ngr = (int)(g.block / 32);
  const int64_t gbase = (cm.lh * 128 + cm.c) * g.G + t0 / 32;  // first scale of the block
  uint64_t sacc = 0, zacc = 0;
#pragma unroll 1
  for (int gi = 0; gi < ngr; ++gi) {
    const uint4* rowp = PAGED ? paged_row(gi) : src + (int64_t)gi * 32 * 16;  // 32 tokens = 32 * 256 B
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(rowp + k);  // read once (evict-first)
    if (gi + 1 < ngr) {
      const uint4* nx = PAGED ? paged_row(gi + 1) : rowp + 32 * 16;
      prefetch_l1(nx);
      prefetch_l1(nx + 2);
    }
    // transpose through shared memory: lane l holds token l's 32 channels and
    // writes them down column l; row c then holds channel c0+c's 32 tokens
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t wk[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = 8 * k + 2 * q;
        *reinterpret_cast<uint16_t*>(tile + c * kTileStrideB + 2 * lane) = (uint16_t)wk[q];
        *reinterpret_cast<uint16_t*>(tile + (c + 1) * kTileStrideB + 2 * lane) = (uint16_t)(wk[q] >> 16);
      }
    }
    __syncwarp();
    uint32_t wv[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 r = *reinterpret_cast<const uint4*>(tile + lane * kTileStrideB + 16 * k);
      wv[4 * k] = r.x; wv[4 * k + 1] = r.y; wv[4 * k + 2] = r.z; wv[4 * k + 3] = r.w;
    }
    float mn, mx;
    minmax_words(wv, mn, mx);
    nonfinite |= isnan(mn);
    auto value = [&](int i) { return (i & 1) ? bf16_hi(wv[i >> 1]) : bf16_lo(wv[i >> 1]); };
    __half s16, z16;
    uint32_t nib[4];
    quant32(value, mn, mx, W, rl, s16, z16, flags, nib, 0xffffffffu);
    sacc = (sacc >> 16) | ((uint64_t)__half_as_ushort(s16) << 48);
    zacc = (zacc >> 16) | ((uint64_t)__half_as_ushort(z16) << 48);
    if ((gi & 3) == 3) {
      *reinterpret_cast<uint64_t*>(a.scales + gbase + gi - 3) = sacc;
      *reinterpret_cast<uint64_t*>(a.zeros + gbase + gi - 3) = zacc;
    }
    encode32<W>(e, m, gi * 32, nib, 0xffffffffu);
  }
  const uint32_t len = e.finish();
  *reinterpret_cast<uint32_t*>(slot) = __byte_perm(len, 0, 0x0123);
  a.sizes[cm.b] = (uint64_t)len + 4;
  if (nonfinite) flags |= KVC_FLAG_NONFINITE_INPUT;
  if (flags) atomicOr(a.status, flags);
}

template <int W, typename Tout>
__global__ void __launch_bounds__(kFThreads) k_fused_chan_decode(const FusedArgs a) {
  constexpr int kStride = sizeof(Tout) == 2 ? kTileStrideB : kTileStrideF;
  __shared__ __align__(16) uint8_t tiles[kFThreads / 32][32 * kStride];
  const Geo& g = a.g;
  const int64_t gt = (int64_t)blockIdx.x * kFThreads + threadIdx.x;
  const int64_t nbt = g.T / g.block;
  const int64_t nblocks = g.LH * 128 * nbt;
  if (gt >= nblocks) return;  // whole CTAs
  const ChanMap cm = chan_map(gt, nbt);
  const int lane = threadIdx.x & 31;
  const int c0 = cm.c - lane;
  uint8_t* tile = tiles[threadIdx.x >> 5];
  const int64_t t0 = cm.tc * g.block;
  RcDec d;
  int64_t blen;
  uint32_t flags = open_block(a, cm.b, d, blen) ? 0u : (uint32_t)KVC_FLAG_CODEC;
  SModel<W> m;
  m.init();
  float chk = 0.0f;
  const int ngr = (int)(g.block / 32);
  const int64_t gbase = (cm.lh * 128 + cm.c) * g.G + t0 / 32;
  uint2 s4 = make_uint2(0, 0), z4 = make_uint2(0, 0);
#pragma unroll 1
  for (int gi = 0; gi < ngr; ++gi) {
    if ((gi & 3) == 0) {
      s4 = __ldg(reinterpret_cast<const uint2*>(a.scales_in + gbase + gi));
      z4 = __ldg(reinterpret_cast<const uint2*>(a.zeros_in + gbase + gi));
    }
    const float s = __half2float(__ushort_as_half(half_at(s4, gi & 3)));
    const float z = __half2float(__ushort_as_half(half_at(z4, gi & 3)));
    // this lane's destination row: token t0 + 32 gi + lane, channels c0 .. c0+31
    Tout* mine = reinterpret_cast<Tout*>(a.out) + out_index(a, cm.lh, t0 + gi * 32 + lane, c0);
    if (!(isfinite(s) && isfinite(z))) chk = 1.0f;  // see k_fused_tok_decode
    decode32<W>(d, m, gi * 32, s, z, 0xffffffffu, [&](int k, const float* v) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        stage_value<Tout>(tile, 8 * k + i, lane, kStride, v[i]);
      }
    });
    __syncwarp();
    store_rows<Tout, kStride>(tile, mine, lane, true);
    __syncwarp();
  }
  if (chk != 0.0f) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
  if (!(flags & KVC_FLAG_CODEC) && (int64_t)d.pulled() + 8 > blen) flags |= KVC_FLAG_CODEC;
  if (flags) atomicOr(a.status, flags);
}

template <int W>
cudaError_t enc_w(const FusedArgs& a, cudaStream_t s) {
  const Geo& g = a.g;
  if (g.uchan) {
    const int64_t nblocks = g.LH * 128 * (g.T / g.block);
    const int64_t threads = nblocks > a.max_blocks + 1 ? nblocks : a.max_blocks + 1;
    const unsigned grid = (unsigned)((threads + kFThreads - 1) / kFThreads);
    if (a.paged)
      k_fused_chan_encode<W, true><<<grid, kFThreads, 0, s>>>(a);
    else
      k_fused_chan_encode<W, false><<<grid, kFThreads, 0, s>>>(a);
  } else {
    k_fused_tok_encode<W><<<(unsigned)((a.max_blocks + 1 + kFThreads - 1) / kFThreads), kFThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

template <int W, typename Tout>
cudaError_t dec_w(const FusedArgs& a, cudaStream_t s) {
  const Geo& g = a.g;
  if (g.uchan) {
    const int64_t nblocks = g.LH * 128 * (g.T / g.block);
    k_fused_chan_decode<W, Tout><<<(unsigned)((nblocks + kFThreads - 1) / kFThreads), kFThreads, 0, s>>>(a);
  } else {
    const int64_t nrows = g.LH * g.T, R = g.block / 128;
    const int64_t nblocks = (nrows + R - 1) / R;
    k_fused_tok_decode<W, Tout><<<(unsigned)((nblocks + kFThreads - 1) / kFThreads), kFThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

template <typename Tout>
cudaError_t dec_t(const FusedArgs& a, cudaStream_t s) {
  switch (a.g.bits) {
    case 1: return dec_w<1, Tout>(a, s);
    case 2: return dec_w<2, Tout>(a, s);
    case 3: return dec_w<3, Tout>(a, s);
    default: return dec_w<4, Tout>(a, s);
  }
}

bool fused_rc_applicable_impl(const Geo& g) {
  if (g.codec != C_ENTROPY || g.transform != T_IDENTITY || g.C != 128 || g.group != 32) return false;
  if (g.quant != Q_UNIFORM && g.quant != Q_UCHAN) return false;
  if (g.bits < 1 || g.bits > 4 || g.in_dtype != KVC_DTYPE_BF16) return false;
  if (g.block > kH || g.block % 128 != 0) return false;
  if (g.uchan && (g.T % g.block != 0)) return false;
  return g.E < (1ll << 40);
}

}  // namespace

cudaError_t upload_fused_recip(const uint32_t* rows) { return cudaMemcpyToSymbol(c_recip, rows, sizeof(c_recip)); }

bool fused_rc_applicable(const Geo& g) { return fused_rc_applicable_impl(g); }

cudaError_t launch_fused_rc_encode(const FusedArgs& args, cudaStream_t s) {
  FusedArgs a = args;
  cudaError_t ce = ensure_recip_tables();
  if (ce != cudaSuccess) return ce;
  ProfScope ps("fused_encode", s);
  switch (a.g.bits) {
    case 1: return enc_w<1>(a, s);
    case 2: return enc_w<2>(a, s);
    case 3: return enc_w<3>(a, s);
    default: return enc_w<4>(a, s);
  }
}

cudaError_t launch_fused_rc_decode(const FusedArgs& args, cudaStream_t s) {
  FusedArgs a = args;
  cudaError_t ce = ensure_recip_tables();
  if (ce != cudaSuccess) return ce;
  ProfScope ps("fused_decode", s);
  return a.g.out_dtype == KVC_DTYPE_BF16 ? dec_t<__nv_bfloat16>(a, s) : dec_t<float>(a, s);
}

}  // namespace kvc
