// Fused head_dim-128 per-token kernels: the hot path for bf16 serving caches.
//
// Encode (kernel 1 of the north star): one CTA streams tiles of 64 token rows
// (16 KB bf16) through a 4-deep TMA ring (cp.async.bulk.tensor, 128B swizzle,
// mbarrier completion).  Two threads own a row, one 64-channel half each:
//   transform -> group min/max -> fp16 scale/zero -> symbols -> MSB-first
//   bit packing straight into the width stream (codecs.py:79-87, :339-345).
// Hadamard runs as a float64 butterfly in registers in the reference's stage
// order (h = 1..32 in-thread, h = 64 as one shuffle exchange), then the exact
// RN32(RN64(S / sqrt 128)) rounding of numerics.cuh.
// Decode (kernel 3): packed stream -> dequantize -> inverse transform (fp32,
// within the reference's tolerance) -> bf16 rows, contiguous or paged.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>

#include "kernels.h"
#include "numerics.cuh"
#include "profile.h"
#include "rowpos.cuh"

namespace kvc {
namespace {

constexpr int kThreads = 128;            // 64 rows per tile
constexpr int kRows = kThreads / 2;
constexpr int kStages = 3;
constexpr int kTileBytes = kThreads * 128;  // one 128 B half-row per thread

enum Mode { M_IDENTITY = 0, M_DELTA = 1, M_HADAMARD = 2, M_AFFINE = 3 };

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// paged cache view (64 ch, half, head, token row, layer), as make_paged_map:
// one box = a run of tokens of one head inside one page
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int h, int r, int l, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(0), "r"(0), "r"(h), "r"(r), "r"(l), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ----------------------------------------------------------- bit packing
// Pack 32 symbols (low byte of the magic-rounded floats) at width W,
// MSB-first (codecs.py:79-87), and store the 4W bytes at dst (4-byte aligned).
template <int W>
__device__ __forceinline__ void pack32_store(const float* q, uint8_t* dst) {
  uint32_t be[W];
  if constexpr (32 % W == 0) {
    // whole symbols per word: an IMAD chain over the magic floats' bit
    // patterns (kMagicBits + symbol), the constant part removed once per word
    constexpr int per = 32 / W;
    constexpr uint32_t fix = kMagicBits * (0xFFFFFFFFu / ((1u << W) - 1u));
#pragma unroll
    for (int k = 0; k < W; ++k) {
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < per; ++j) acc += __float_as_uint(q[k * per + j]) * (1u << (32 - W * (j + 1)));
      be[k] = acc - fix;
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) be[k] = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t s = __float_as_uint(q[i]) & ((1u << W) - 1u);
      const int p = i * W, k = p >> 5, off = p & 31;
      if (off + W <= 32) {
        be[k] |= s << (32 - off - W);
      } else {
        be[k] |= s >> (off + W - 32);
        be[k + 1] |= s << (64 - off - W);
      }
    }
  }
  uint32_t wd[W];
#pragma unroll
  for (int k = 0; k < W; ++k) wd[k] = __byte_perm(be[k], 0, 0x0123);
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int k = 0; k < W; k += 4) *reinterpret_cast<uint4*>(dst + 4 * k) = make_uint4(wd[k], wd[k + 1], wd[k + 2], wd[k + 3]);
  } else if constexpr (W % 2 == 0) {
#pragma unroll
    for (int k = 0; k < W; k += 2) *reinterpret_cast<uint2*>(dst + 4 * k) = make_uint2(wd[k], wd[k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) reinterpret_cast<uint32_t*>(dst)[k] = wd[k];
  }
}

__device__ __forceinline__ void pack32_dispatch(int w, const float* q, uint8_t* dst) {
  switch (w) {
    case 1: pack32_store<1>(q, dst); break;
    case 2: pack32_store<2>(q, dst); break;
    case 3: pack32_store<3>(q, dst); break;
    case 4: pack32_store<4>(q, dst); break;
    case 5: pack32_store<5>(q, dst); break;
    case 6: pack32_store<6>(q, dst); break;
    case 7: pack32_store<7>(q, dst); break;
    default: pack32_store<8>(q, dst); break;
  }
}

// Unpack 32 symbols of width W from src (4-byte aligned) into floats
// (RAW: the magic floats 2^23 + symbol, the 2^23 removed by the caller).
template <int W, bool RAW = false>
__device__ __forceinline__ void unpack32(const uint8_t* src, float* v) {
  uint32_t be[W];
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int k = 0; k < W; k += 4) {
      uint4 t = *reinterpret_cast<const uint4*>(src + 4 * k);
      be[k] = t.x; be[k + 1] = t.y; be[k + 2] = t.z; be[k + 3] = t.w;
    }
  } else if constexpr (W % 2 == 0) {
#pragma unroll
    for (int k = 0; k < W; k += 2) {
      uint2 t = *reinterpret_cast<const uint2*>(src + 4 * k);
      be[k] = t.x; be[k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) be[k] = reinterpret_cast<const uint32_t*>(src)[k];
  }
#pragma unroll
  for (int k = 0; k < W; ++k) be[k] = __byte_perm(be[k], 0, 0x0123);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int p = i * W, k = p >> 5, off = p & 31;
    uint32_t s;
    if (off + W <= 32) {
      s = (be[k] >> (32 - off - W)) & ((1u << W) - 1u);
    } else {
      s = ((be[k] << (off + W - 32)) | (be[k + 1] >> (64 - off - W))) & ((1u << W) - 1u);
    }
    v[i] = RAW ? __uint_as_float(0x4B000000u | s) : __uint_as_float(0x4B000000u | s) - 8388608.0f;
  }
}

template <bool RAW = false>
__device__ __forceinline__ void unpack32_dispatch(int w, const uint8_t* src, float* v) {
  switch (w) {
    case 1: unpack32<1, RAW>(src, v); break;
    case 2: unpack32<2, RAW>(src, v); break;
    case 3: unpack32<3, RAW>(src, v); break;
    case 4: unpack32<4, RAW>(src, v); break;
    case 5: unpack32<5, RAW>(src, v); break;
    case 6: unpack32<6, RAW>(src, v); break;
    case 7: unpack32<7, RAW>(src, v); break;
    default: unpack32<8, RAW>(src, v); break;
  }
}

// packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2: two IEEE round-to-nearest
// operations per instruction, lane-wise identical to the scalar ones).  PTX
// with an explicit .rn: never contracted into an FFMA2 (the __fadd2_rn /
// __fmul2_rn intrinsics are, which would break quantize.py:178's unfused
// multiply-then-add).
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
#define KVC_F2OP(name, op)                                                                               \
  __device__ __forceinline__ float2 name(float2 a, float2 b) {                                          \
    float2 d;                                                                                            \
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t" op      \
        " rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"                                                  \
        : "=f"(d.x), "=f"(d.y)                                                                           \
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                                      \
    return d;                                                                                            \
  }
KVC_F2OP(f2add, "add.rn.f32x2")
KVC_F2OP(f2mul, "mul.rn.f32x2")
#undef KVC_F2OP
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) { return f2add(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// ------------------------------------------------------------ group stats
// min / max of 32 fp32 values
__device__ __forceinline__ void minmax32(const float* y, float& mn, float& mx) {
  mn = y[0];
  mx = y[0];
#pragma unroll
  for (int i = 1; i < 32; ++i) {
    mn = fminf(mn, y[i]);
    mx = fmaxf(mx, y[i]);
  }
}

// min / max of 32 bf16 values packed in 16 words: two per HMNMX2, exact, and
// NaN-propagating so a NaN input surfaces in the group stats (the reference
// rejects non-finite values, tensors.py:41-42)
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
__device__ __forceinline__ void minmax32_bf16(const uint32_t* w, float& mn, float& mx) {
  uint32_t lo = w[0], hi = w[0];
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    lo = bmin2(lo, w[k]);
    hi = bmax2(hi, w[k]);
  }
  lo = bmin2(lo, __byte_perm(lo, 0, 0x1032));  // both halves now hold the min
  hi = bmax2(hi, __byte_perm(hi, 0, 0x1032));
  mn = __uint_as_float(lo << 16);
  mx = __uint_as_float(hi << 16);
}

// Quantize the thread's 64 values (two chunks of 32 at channel bases cb0,
// cb1) given each chunk's min/max; G in {32, 64, 128}: a 64-group is both
// chunks (natural layout) or chunk c of both threads of the row (hadamard
// layout); a 128-group is the whole row across the thread pair.
template <int G>
__device__ __forceinline__ void quantize64(float* y, float mn0, float mx0, float mn1, float mx1, int cb0, int cb1,
                                           int w, float rl, int64_t grow, __half* scales, __half* zeros,
                                           bool hadlayout, int half, uint32_t& flags) {
  static_assert(G == 32 || G == 64 || G == 128, "fused path groups");
  {
    float gmn[2], gmx[2];
    if (G == 32) {
      gmn[0] = mn0; gmx[0] = mx0;
      gmn[1] = mn1; gmx[1] = mx1;
    } else if (G == 128) {
      float mn = fminf(mn0, mn1), mx = fmaxf(mx0, mx1);
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      gmn[0] = gmn[1] = mn;
      gmx[0] = gmx[1] = mx;
    } else if (!hadlayout) {  // natural layout: both chunks form the group
      gmn[0] = gmn[1] = fminf(mn0, mn1);
      gmx[0] = gmx[1] = fmaxf(mx0, mx1);
    } else {  // hadamard layout: chunk c of both threads forms group c
      gmn[0] = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, 1));
      gmx[0] = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      gmn[1] = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, 1));
      gmx[1] = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      __half s16, z16;
      GroupQ q = group_setup(gmn[c], gmx[c], w, rl, s16, z16, flags);
      const int64_t gi = grow + (c ? cb1 : cb0) / G;
      // one writer per group
      const bool writer = (G == 32) ? true : (G == 128) ? (half == 0 && c == 0) : (!hadlayout ? c == 0 : (half == c));
      if (writer && scales) {
        scales[gi] = s16;
        zeros[gi] = z16;
      }
      float* yy = y + c * 32;
      // no clip needed when the exact quotients of the group's min and max
      // already round into [0, levels] (monotone in v); decided per warp
      bool easy = false;
      if (q.mode == 0) {
        const float dl = __fsub_rn(gmn[c], q.z), dh = __fsub_rn(gmx[c], q.z);
        const float l0 = __fmul_rn(dl, q.r), h0 = __fmul_rn(dh, q.r);
        const float l1 = __fmaf_rn(__fmaf_rn(-l0, q.s, dl), q.r, l0);
        const float h1 = __fmaf_rn(__fmaf_rn(-h0, q.s, dh), q.r, h0);
        easy = l1 >= -0.5f && h1 < q.lv + 0.5f;
      }
      if (__all_sync(0xffffffffu, easy)) {
        // two values per FADD2 / FMUL2 / FFMA2, the same roundings as the
        // scalar sequence of quant_magic (minus the clip)
        float2* y2 = reinterpret_cast<float2*>(yy);
        const float2 nz = f2(-q.z, -q.z), r2 = f2(q.r, q.r), ns = f2(-q.s, -q.s), mg = f2(kMagicRound, kMagicRound);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 d = f2add(y2[i], nz);
          const float2 q0 = f2mul(d, r2);
          y2[i] = f2add(f2fma(f2fma(q0, ns, d), r2, q0), mg);
        }
      } else if (q.mode == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) yy[i] = quant_magic(yy[i], q);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) yy[i] = __uint_as_float(kMagicBits + quant_one(yy[i], q));
      }
    }
  }
}

// paged input (thread 0): the 64-token tile as one 5D box per page run; out
// of line so the contiguous kernels' main loop is unchanged
__device__ __noinline__ void issue_paged_tile(uint8_t* dst, const CUtensorMap* map, int64_t tile, int64_t T, int64_t H,
                                              int64_t page_tokens, const int32_t* block_table, uint64_t* bar) {
  const int64_t r0 = tile * kRows, lh = r0 / T, t0 = r0 - lh * T;
  const int l = (int)(lh / H), h = (int)(lh - (int64_t)l * H);
  const int bt = page_tokens < kRows ? (int)page_tokens : kRows;
  for (int j = 0; j < kRows; j += bt) {
    const int64_t t = t0 + j;
    const int64_t prow = (int64_t)block_table[t / page_tokens] * page_tokens + t % page_tokens;
    tma_load_5d(dst + j * 256, map, h, (int)prow, l, bar);
  }
}

// float32 bit pattern of local value i: w[] holds 32 bf16 pairs or 64 fp32
// bit patterns of this thread's half row
template <bool F32>
__device__ __forceinline__ uint32_t vbits_of(const uint32_t* w, int i) {
  if constexpr (F32) return w[i];
  return (i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16);
}

// Hadamard of one row held by a thread pair (this thread: channels
// 64*half..+63 in wv), float64 butterfly in the reference's stage order
// (transforms.py:41-46), then RN32(RN64(S / sqrt 128)).  Leaves this thread's
// 64 outputs in y (chunk 0: channels 32*half.., chunk 1: 64 + 32*half..) and
// returns true when the row must be re-encoded exactly (k_encode_fixup).
template <bool F32>
__device__ __forceinline__ bool had64_row(const uint32_t* wv, int half, const EncArgs& a, float* y, float& nanacc) {
  // Input range of the whole row (this half and the partner's): with every
  // |x| in [2^-100, 2^101) no Hadamard output can overflow f32 or be a
  // nonzero f32 subnormal, so the rounding below needs only the
  // near-midpoint test.  NaN / inf inputs (which the 2^-896
  // reinterpretation would turn into finite doubles) show up here too
  // (tensors.py:41-42).  Zeros, extreme magnitudes and near-midpoint
  // results send the row to the exact fixup pass (k_encode_fixup).
  bool row_ok;
  if constexpr (F32) {  // |x| as unsigned bit patterns order like the floats
    uint32_t amx = wv[0] & 0x7FFFFFFFu, amn = amx;
#pragma unroll
    for (int k = 1; k < 64; ++k) {
      const uint32_t aw = wv[k] & 0x7FFFFFFFu;
      amx = max(amx, aw);
      amn = min(amn, aw);
    }
    if (amx >= 0x7F800000u) nanacc = 1.0f;
    amx = max(amx, (uint32_t)__shfl_xor_sync(0xffffffffu, amx, 1));
    amn = min(amn, (uint32_t)__shfl_xor_sync(0xffffffffu, amn, 1));
    const uint32_t emax = (amx >> 23) & 0xFFu, emin = (amn >> 23) & 0xFFu;
    row_ok = emax <= 127u + 100u && emin >= 127u - 100u;
  } else {
    uint32_t amx = wv[0] & 0x7FFF7FFFu, amn = amx;
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const uint32_t aw = wv[k] & 0x7FFF7FFFu;
      amx = bmax2(amx, aw);
      amn = bmin2(amn, aw);
    }
    amx = bmax2(amx, __byte_perm(amx, 0, 0x1032));
    amn = bmin2(amn, __byte_perm(amn, 0, 0x1032));
    if ((amx & 0x7F80u) == 0x7F80u) nanacc = 1.0f;
    amx = bmax2(amx, __shfl_xor_sync(0xffffffffu, amx, 1));
    amn = bmin2(amn, __shfl_xor_sync(0xffffffffu, amn, 1));
    const uint32_t emax = (amx >> 7) & 0xFFu, emin = (amn >> 7) & 0xFFu;
    row_ok = emax <= 127u + 100u && emin >= 127u - 100u;
  }
  double f[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) f[i] = f32bits_scaled_f64(vbits_of<F32>(wv, i));
  // stages h = 1..32 (transforms.py:41-46 order), in registers.  At h = 32
  // thread B (half 1) writes its two outputs swapped (u - v at i, u + v at
  // i + 32; the same roundings, as one DFMA with -1 each), so afterwards
  // both threads hold the value the partner needs at local 32 + k and the
  // one they keep at local k: the h = 64 exchange below needs no selects.
  const double sgn = half ? -1.0 : 1.0;
#pragma unroll
  for (int h = 1; h < 64; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if ((i & h) == 0) {
        const double u = f[i], v = f[i + h];
        if (h == 32) {
          f[i] = __fma_rn(v, sgn, u);
          f[i + h] = __fma_rn(v, -sgn, u);
        } else {
          f[i] = u + v;
          f[i + h] = u - v;
        }
      }
    }
  }
  // stage h = 64 across the thread pair: A (half 0) keeps outputs 0..31 and
  // 64..95, B keeps 32..63 and 96..127.  A's local k / 32 + k hold its
  // T[k] / T[32 + k]; B's hold T[32 + k] / T[k].  Each sends local 32 + k
  // and forms (own + r, own - r): A gets out[k], out[64 + k]; B gets
  // out[32 + k] (a + b = b + a) and -out[96 + k] (own - r = -(r - own),
  // negated back through the sign of the scale below).
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double send = f[32 + k];
    const int lo = __shfl_xor_sync(0xffffffffu, __double2loint(send), 1);
    const int hi = __shfl_xor_sync(0xffffffffu, __double2hiint(send), 1);
    const double r = __hiloint2double(hi, lo);
    const double u = f[k];
    f[k] = u + r;
    f[32 + k] = u - r;
  }
  // RN32(RN64(S / sqrt n)) as one F2F of RN64(S * RN64(1/sqrt n)); the two
  // differ only within 4 ulp64 of an f32 rounding midpoint (numerics.cuh).
  // B's second half is scaled by -hk (RN is sign-symmetric; an exact zero
  // comes out as -0 there, made +0 in the group min / max below).
  const double hk2 = half ? -a.hk : a.hk;
  bool mid = false;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const double q = f[i] * (i < 32 ? a.hk : hk2);
    mid |= ((uint32_t)__double2loint(q) & 0x1FFFFFFFu) - 0x0FFFFFFCu <= 8u;
    y[i] = __double2float_rn(q);
  }
  bool need_fix = !row_ok || mid;
  need_fix |= __shfl_xor_sync(0xffffffffu, (int)need_fix, 1) != 0;
  return need_fix;
}

// ---------------------------------------------------------------------------
// Certified float32 Hadamard encode (bf16 or float32 input, 32- / 64- /
// 128-channel groups; bf16 at 32 is the reference default profile,
// transforms.py:62 + quantize.py:142-154).
//
// The reference's y = RN32(RN64(S / c)) (S the float64 butterfly sum,
// c = RN64(sqrt 128)) reaches the payload only through three decisions, each
// monotone in y: the fp16 zero RN16(min y), the fp16 scale
// RN16(RN64(RN32(max y - min y) / levels)) and each symbol
// clip(rint(RN32(RN32(y - z) / s))).  So the butterfly runs in float32 (two
// values per FADD2) with a rigorous bound on every output, u = 2^-24:
//  * exact rows -- bf16 inputs are multiples of 2^(emin-7) and every partial
//    sum is below 2^(es1+1) (es1: exponent of Sum|x|), so with
//    es1 <= emin + 16 all seven stages are exact in float32 (any order); what
//    remains is RN32 of S RN32(1/c) (RN32(1/c) is within 0.287u of 1/c) and
//    the reference's own RN32: |y_hat - y| <= 2.3u |y|, so a group's min is
//    within 2.3u |min|, its max within 2.3u |max|;
//  * other rows (and float32 inputs): gamma_7 Sum|x| for any depth-7
//    summation tree plus those roundings, D = 9.3u Sum|x| / c;
//  * both: + 2^-140 for subnormal intermediates.
// A group is certified when every decision is constant on the intervals: the
// zero and the scale are evaluated at both ends (directed rounding; the
// scale's own float32 roundings covered by 1 -+ 2^-22), and every quotient
// RN(RN(S sc - z) r) must lie farther than tau = D / s + 2^-21 (|t| + 1)
// from its rounding boundary.  A certified row's bytes equal the reference's;
// a row with an uncertified group is flagged in a bitmap for the float64 pass
// (k_had64_list, the reference's butterfly in stage order), and rows with
// non-finite or huge inputs go straight to the exact fixup pass
// (k_encode_fixup).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// min / max of 32 floats, two new values per FMNMX3
__device__ __forceinline__ void minmax32_3(const float* y, float& mn, float& mx) {
  mn = fminf(y[0], y[1]);
  mx = fmaxf(y[0], y[1]);
#pragma unroll
  for (int i = 2; i < 32; i += 2) {
    mn = min3f(mn, y[i], y[i + 1]);
    mx = max3f(mx, y[i], y[i + 1]);
  }
}
__device__ __forceinline__ unsigned short rn16(float v) { return __half_as_ushort(__float2half_rn(v)); }

// Float32 Hadamard of the row held by a thread pair (this thread: channels
// 64*half..+63 as bf16 pairs in wv).  y gets this thread's 64 unscaled sums
// S (chunk 0: channels 32*half.., chunk 1: 64 + 32*half.., the same layout
// as had64_row; B's chunk 1 negated).  Returns the
// row's bound D, or -1 when every stage was exact (the caller then bounds
// each group by 2.3u |y| of its extremes: only the scaling and the
// reference's roundings remain).  row_ok: finite inputs with Sum|x| < 2^100
// (no float32 overflow anywhere in the butterfly).
template <bool F32>
__device__ __forceinline__ float had32_row(const uint32_t* wv, int half, const EncArgs& a, float* y, bool& row_ok) {
  // P[m] = (local m, local m + 32): stages h = 1..16 pair P[m] with P[m + h]
  float2 P[32];
#pragma unroll
  for (int m = 0; m < 32; ++m)
    P[m] = make_float2(__uint_as_float(vbits_of<F32>(wv, m)), __uint_as_float(vbits_of<F32>(wv, m + 32)));
  // min |x| (three per FMNMX3, |.| free): the inputs' 2^(emin-7) grid (bf16;
  // float32 inputs carry 24-bit significands and take the gamma_7 bound)
  float amn = 0.0f;
  if constexpr (!F32) {
    amn = fminf(fabsf(P[0].x), fabsf(P[0].y));
#pragma unroll
    for (int m = 1; m < 32; ++m) amn = min3f(amn, fabsf(P[m].x), fabsf(P[m].y));
  }
  // h = 1, and Sum|x| as max(|a + b|, |a - b|) = |a| + |b| per pair (a NaN
  // input makes the sum NaN)
  float2 sa = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int m = 0; m < 32; m += 2) {
    const float2 s = f2add(P[m], P[m + 1]), d = f2sub(P[m], P[m + 1]);
    sa = f2add(sa, make_float2(fmaxf(fabsf(s.x), fabsf(d.x)), fmaxf(fabsf(s.y), fabsf(d.y))));
    P[m] = s;
    P[m + 1] = d;
  }
#pragma unroll
  for (int h = 2; h < 32; h <<= 1) {
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      if ((m & h) == 0) {
        const float2 s = f2add(P[m], P[m + h]), d = f2sub(P[m], P[m + h]);
        P[m] = s;
        P[m + h] = d;
      }
    }
  }
  // h = 32 inside each pair; thread B keeps local 32 + m and sends local m
  // (one FFMA by -+1 each, the same roundings), as had64_row
  const float sg = half ? -1.0f : 1.0f;
  float K[32], Y[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    K[m] = __fmaf_rn(P[m].y, sg, P[m].x);
    Y[m] = __fmaf_rn(P[m].y, -sg, P[m].x);
  }
  // h = 64 across the pair: the unscaled sums S (B's chunk 1 as -S); the
  // scaling by RN32(1/c) happens inside the quantizer (cert_group)
#pragma unroll
  for (int m = 0; m < 32; m += 2) {
    const float2 rv = make_float2(__shfl_xor_sync(0xffffffffu, Y[m], 1), __shfl_xor_sync(0xffffffffu, Y[m + 1], 1));
    const float2 kv = make_float2(K[m], K[m + 1]);
    const float2 s = f2add(kv, rv), d = f2sub(kv, rv);
    y[m] = s.x;
    y[m + 1] = s.y;
    y[32 + m] = d.x;
    y[33 + m] = d.y;
  }
  float s1 = sa.x + sa.y;
  s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
  if constexpr (!F32) amn = fminf(amn, __shfl_xor_sync(0xffffffffu, amn, 1));
  // a NaN / inf input (or a sum near the float32 range) makes s1 NaN / huge:
  // the row goes to the exact fixup pass, which also raises the input flag
  row_ok = s1 < 0x1p100f;
  // Exact stages: inputs are multiples of 2^(emin-7); every partial sum is
  // below 2^(es1+1) (es1: exponent of an upper bound of Sum|x|), so all
  // seven stages are exact when es1 <= emin + 16 (24 bits); other rows take
  // the gamma_7 bound
  if constexpr (!F32) {
    const int emin = (int)(__float_as_uint(amn) >> 23);
    const int es1 = (int)(__float_as_uint(s1 * 1.0000153f) >> 23);  // s1 (1 + 2^-16) >= Sum|x|
    if (es1 <= emin + 16) return -1.0f;
  }
  // (7 + 2.3) u / c: gamma_7 Sum|x| for the butterfly, 2.29u |S| / c for the
  // two float32 scalings and the reference's rounding; 1.002 covers the
  // float32 evaluation of Sum|x| and of this coefficient
  return __fmaf_ru(s1, 9.3f * 0x1p-24f * a.hr32 * 1.002f, 0x1p-140f);
}

// Quantize one certified group of 32 unscaled sums (y = S sc, sc = +-RN32(1/c);
// yy -> magic floats 1.5 2^23 + symbol, as quantize64) with fp16 scale /
// zero s16 / z16; mn / mx: min / max of y.  Returns
// false when a decision is not constant over +-D (the row is then re-encoded
// by the float64 pass, which also rewrites s16 / z16).
__device__ __forceinline__ bool cert_group(float* yy, float sc, float mn, float mx, float D, int w, float rl,
                                           unsigned short& s16, unsigned short& z16) {
  const float lv = (float)((1 << w) - 1);
  // exact butterfly: each output is off by at most 2.29u |y| (RN32 of S
  // RN32(1/c), whose error is 0.287u, and the reference's own RN32): the
  // group's min within 2.3u |mn|, its max within 2.3u |mx| (the bound of the
  // extreme element bounds every element beyond it), any value within
  // 2.3u max(|mn|, |mx|)
  float Dz = D, Dx = D;
  if (D < 0.0f) {
    Dz = __fmaf_ru(fabsf(mn), 2.3f * 0x1p-24f, 0x1p-140f);
    Dx = __fmaf_ru(fabsf(mx), 2.3f * 0x1p-24f, 0x1p-140f);
    D = fmaxf(Dz, Dx);
  }
  // zero RN16(min y), min y in [mn - Dz, mn + Dz]
  const unsigned short zl = rn16(__fsub_rd(mn, Dz)), zh = rn16(__fadd_ru(mn, Dz));
  // scale RN16(RN64(RN32(max - min) / lv)), RN32(max - min) in [dl, dh]
  const float Dd = __fadd_ru(Dz, Dx);
  const float dl = __fsub_rd(__fsub_rd(mx, mn), Dd), dh = __fadd_ru(__fsub_ru(mx, mn), Dd);
  // (1 -+ 2^-22: the three float32 roundings of d rl (1 -+ 2^-22) stay on the
  // safe side of d / lv)
  const unsigned short sl = rn16(__fmul_rn(__fmul_rn(dl, rl), 0.999999761581420898f));
  const unsigned short sh = rn16(__fmul_rn(__fmul_rn(dh, rl), 1.000000238418579102f));
  s16 = sl;
  z16 = zl;
  const float s = __half2float(__ushort_as_half(sl)), z = __half2float(__ushort_as_half(zl));
  bool ok = zl == zh && sl == sh && dl > 0.0f && !isinf(s) && !isinf(z);
  // s == 0: r = 0 turns every quotient into 0 (symbol 0, quantize.py:154)
  const float r = s > 0.0f ? __frcp_rn(s) : 0.0f;
  const float dlo = __fsub_rn(mn, z), dhi = __fsub_rn(mx, z);
  const float l0 = __fmul_rn(dlo, r), h0 = __fmul_rn(dhi, r);
  const float l1 = __fmaf_rn(__fmaf_rn(-l0, s, dlo), r, l0);
  const float h1 = __fmaf_rn(__fmaf_rn(-h0, s, dhi), r, h0);
  // tau >= D / s + 5.1u |t| (+ margin): the distance any quotient may move
  const float tau = __fmaf_ru(D, r * 1.0001f, 0x1p-21f * (fmaxf(fabsf(l1), fabsf(h1)) + 1.0f));
  const bool easy = l1 >= -0.5f && h1 < lv + 0.5f;
  float racc = 0.0f;
  float2* y2 = reinterpret_cast<float2*>(yy);
  const float2 nz = f2(-z, -z), rr = f2(r, r), sc2 = f2(sc, sc), mg = f2(kMagicRound, kMagicRound);
  const float2 nmg = f2(-kMagicRound, -kMagicRound);
  // symbols rint(RN(RN(S sc - z) r)): within D / s + 5.1u |t| of the
  // reference's rint(RN(RN(y - z) / s)) argument (D covers the scaling),
  // inside tau, so a quotient farther than tau from its rounding boundary
  // needs no Markstein correction (quant_magic) to round like the reference
  if (__all_sync(0xffffffffu, easy)) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 q = f2mul(f2fma(y2[i], sc2, nz), rr);
      const float2 m = f2add(q, mg);
      const float2 rho = f2sub(q, f2add(m, nmg));
      racc = max3f(racc, fabsf(rho.x), fabsf(rho.y));
      y2[i] = m;
    }
  } else {
    const float top = kMagicRound + lv;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 q = f2mul(f2fma(y2[i], sc2, nz), rr);
      const float2 m = f2add(q, mg);
      const float2 rho = f2sub(q, f2add(m, nmg));
      racc = max3f(racc, fabsf(rho.x), fabsf(rho.y));
      y2[i] = f2(fminf(fmaxf(m.x, kMagicRound), top), fminf(fmaxf(m.y, kMagicRound), top));
    }
  }
  return ok && racc < 0.5f - tau;
}

// ------------------------------------------------------------ encode kernel
// W = compile-time symbol width (uniform strategies), 0 = per-row runtime width
// F32: float32 input (the reference's own corpora): the tile is 64 rows x
// 512 B read as 128-byte quarter rows (2 stages of 32 KB keep 3 CTAs/SM), and
// every mode reads each value's float32 bit pattern instead of unpacking bf16.
template <bool F32>
__host__ __device__ constexpr int enc_stages() {
  return F32 ? 2 : kStages;
}
template <bool F32>
__host__ __device__ constexpr int enc_tile_bytes() {
  return F32 ? 2 * kTileBytes : kTileBytes;
}
template <bool F32>
__host__ __device__ constexpr int enc_smem_bytes() {
  return enc_stages<F32>() * enc_tile_bytes<F32>() + 1024 + 128;
}

// PAGED: bf16 input read from a paged cache (5D boxes per page run); a
// separate instantiation so the contiguous kernels keep their exact code
// CERT: the certified float32 Hadamard (bf16 input) with the float64 pass
// behind it for the rows it cannot certify
// (4 CTAs per SM; 5, with a 2-stage ring and 96 registers, measured the same)
template <int MODE, int G, int W, bool F32 = false, bool PAGED = false, int CERT = 0>
__global__ void __launch_bounds__(kThreads, ((MODE == M_HADAMARD && !CERT) || MODE == M_DELTA) ? 3 : 4)
    k_enc128(const __grid_constant__ CUtensorMap tmap, const EncArgs a) {
  static_assert(!(F32 && PAGED), "paged input is bf16");
  static_assert(CERT == 0 || MODE == M_HADAMARD, "certified path: Hadamard");
  constexpr int NS = enc_stages<F32>(), TB = enc_tile_bytes<F32>();
  // certified path: a slot is refilled by the last warp to copy it out (a
  // per-slot arrival counter) instead of after a CTA barrier
  __shared__ uint32_t slot_arrivals[NS];
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned (128B swizzle atoms), indexed off smem_raw so the compiler keeps the
  // shared address space (LDS / STS rather than generic loads)
  uint8_t* tiles = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tiles + NS * TB);
  const Geo& g = a.g;
  const int64_t nrows = g.LH * g.T;
  const int64_t ntiles = (nrows + kRows - 1) / kRows;
  const int tid = threadIdx.x, half = tid & 1, warp = tid >> 5, lane = tid & 31;
  // certified contiguous bf16 path: every warp streams its own 16-row tiles
  // through its own 3-slot ring (4 KB boxes, its own mbarriers), so no warp
  // ever waits for another one (the map's box is 32 half rows)
  constexpr bool WR = CERT != 0 && !PAGED && !F32;
  constexpr int WTB = 16 * 256;
  const int64_t nwt = (nrows + 15) / 16;

  // tensor-map coordinate of a tile: 128-byte box rows (bf16 half rows,
  // fp32 quarter rows)
  constexpr int kBoxRows = F32 ? 4 * kRows : 2 * kRows;
  if constexpr (WR) {
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) mbar_init(&full[warp * NS + s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  } else if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      slot_arrivals[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // one tile into ring slot s (thread 0): a 2D box, or for a paged cache
  // (bf16, whole 64-token tiles of one head) one 5D box per page run of bt
  // tokens -- the same 128B-swizzled half rows, at 1 KB-aligned offsets
  auto issue = [&](int s, int64_t tile) {
    mbar_expect_tx(&full[s], TB);
    if constexpr (PAGED)
      issue_paged_tile(tiles + s * TB, &tmap, tile, g.T, g.H, a.page_tokens, a.block_table, &full[s]);
    else
      tma_load_2d(tiles + s * TB, &tmap, 0, (int)(tile * kBoxRows), &full[s]);
  };
  auto issue_w = [&](int s, int64_t wt) {  // one warp tile into this warp's slot s
    uint64_t* b = &full[warp * NS + s];
    mbar_expect_tx(b, WTB);
    tma_load_2d(tiles + (warp * NS + s) * WTB, &tmap, 0, (int)(wt * 32), b);
  };
  const int64_t t_begin = WR ? (int64_t)blockIdx.x * (kThreads / 32) + warp : (int64_t)blockIdx.x;
  const int64_t t_end = WR ? nwt : ntiles;
  const int64_t t_step = WR ? (int64_t)gridDim.x * (kThreads / 32) : (int64_t)gridDim.x;
  if constexpr (WR) {
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) {
        const int64_t wt = t_begin + (int64_t)s * t_step;
        if (wt < t_end) issue_w(s, wt);
      }
    }
  } else if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < ntiles) issue(s, tile);
    }
  }
  __half* scales = reinterpret_cast<__half*>(a.meta);
  __half* zeros = scales + g.ngroups;
  uint32_t flags = 0;
  float nanacc = 0.0f;
  int it = 0;
  // this thread's values from a tile row (swizzled 128-byte box rows); w[]
  // holds 32 bf16 pairs or 64 fp32 bit patterns
  auto load_half = [&](const uint8_t* tb, int r, uint32_t* w) {
    constexpr int kBoxPer = F32 ? 2 : 1;  // 128-byte box rows per half row
#pragma unroll
    for (int q = 0; q < kBoxPer; ++q) {
      const int br = kBoxPer * r + q;
      const uint32_t bsw = (uint32_t)(br & 7);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint4 c = *reinterpret_cast<const uint4*>(tb + br * 128 + (((uint32_t)k ^ bsw) << 4));
        w[32 * q + 4 * k] = c.x; w[32 * q + 4 * k + 1] = c.y; w[32 * q + 4 * k + 2] = c.z; w[32 * q + 4 * k + 3] = c.w;
      }
    }
  };
  constexpr int NW = F32 ? 64 : 32;
  // float32 bit pattern of local value i
  auto vbits = [&](const uint32_t* w, int i) -> uint32_t {
    if constexpr (F32) return w[i];
    return (i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16);
  };
  for (int64_t tile = t_begin; tile < t_end; tile += t_step, ++it) {
    const int s = it % NS;
    mbar_wait(WR ? &full[warp * NS + s] : &full[s], (uint32_t)((it / NS) & 1));
    const uint8_t* tb = WR ? tiles + (warp * NS + s) * WTB : tiles + s * TB;
    uint32_t wv[NW];
    load_half(tb, WR ? lane : tid, wv);
    const int64_t row = WR ? tile * 16 + (lane >> 1) : tile * kRows + (tid >> 1);
    const bool valid = row < nrows;
    // (layer*head, token) of the row: not needed for uniform compile-time
    // widths (the row's stream bit is row * 128 * W) outside delta / affine
    constexpr bool kNeedLH = W == 0 || MODE == M_DELTA || MODE == M_AFFINE;
    const int64_t lh = (kNeedLH && valid) ? row / g.T : 0;
    const int64_t t = (kNeedLH && valid) ? row - lh * g.T : 0;
    uint32_t pv[NW];  // delta: previous row's half
    if (MODE == M_DELTA) {
      if (tid >= 2) {
        load_half(tb, tid - 2, pv);
      } else if (valid && t > 0) {
        const int64_t prev = PAGED ? out_index(a, lh, t - 1, half * 64) : (row - 1) * 128 + half * 64;
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(a.kv) +
                                                          prev * (F32 ? 4 : 2));
#pragma unroll
        for (int k = 0; k < NW / 4; ++k) {
          uint4 c = __ldg(src + k);
          pv[4 * k] = c.x; pv[4 * k + 1] = c.y; pv[4 * k + 2] = c.z; pv[4 * k + 3] = c.w;
        }
      }
    }
    if constexpr (WR) {
      // this warp's half rows are in registers: refill its slot
      __syncwarp();
      if (lane == 0) {
        const int64_t next = tile + (int64_t)NS * t_step;
        if (next < t_end) {
          fence_proxy_async();
          issue_w(s, next);
        }
      }
    } else if constexpr (CERT != 0) {
      // this warp's half rows are in registers; the warp completing the
      // slot's four arrivals (a monotonic count) refills it
      __syncwarp();
      if ((tid & 31) == 0) {
        __threadfence_block();
        if ((atomicAdd(&slot_arrivals[s], 1u) & (kThreads / 32 - 1)) == kThreads / 32 - 1) {
          __threadfence_block();
          const int64_t next = tile + (int64_t)NS * gridDim.x;
          if (next < ntiles) {
            fence_proxy_async();
            issue(s, next);
          }
        }
      }
    } else {
      __syncthreads();  // every thread has its half-row in registers: slot s is free
      if (tid == 0) {
        const int64_t next = tile + (int64_t)NS * gridDim.x;
        if (next < ntiles) {
          fence_proxy_async();
          issue(s, next);
        }
      }
    }
    // invalid tail rows run the same code (shuffles need the full warp) but
    // store nothing

    __align__(8) float y[64];
    int cb0, cb1;
    bool hadlayout = false;
    bool need_fix = false;  // Hadamard: this row is re-encoded exactly by k_encode_fixup
    bool row_ok = true;     // certified path: finite inputs below 2^101
    float Dcert = 0.0f;     // certified path: error bound of the float32 outputs
    const uint32_t flags_before = flags;
    if (MODE == M_HADAMARD) {
      if constexpr (CERT) {
        Dcert = had32_row<F32>(wv, half, a, y, row_ok);
      } else {
        need_fix = had64_row<F32>(wv, half, a, y, nanacc);
        if (need_fix && half == 0 && valid) a.fix_rows[atomicAdd(a.fix_count, 1u)] = (int32_t)row;
      }
      cb0 = 32 * half;
      cb1 = 64 + 32 * half;
      hadlayout = true;
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) y[i] = __uint_as_float(vbits(wv, i));
      if (MODE == M_DELTA && t > 0) {
#pragma unroll
        for (int i = 0; i < 64; ++i) y[i] = __fsub_rn(y[i], __uint_as_float(vbits(pv, i)));
      }
      if (MODE == M_AFFINE) {
        const uint4* mu = reinterpret_cast<const uint4*>(a.meta + g.meta_affine_off + (lh * 128 + half * 64) * 2);
        const uint4* sc = reinterpret_cast<const uint4*>(a.meta + g.meta_affine_off + (g.LH * 128 + lh * 128 + half * 64) * 2);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          uint4 m4 = __ldg(mu + k), s4 = __ldg(sc + k);
          const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w}, sw4[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 mf = __half22float2(*reinterpret_cast<const __half2*>(&mw[q]));
            const float2 sf = __half22float2(*reinterpret_cast<const __half2*>(&sw4[q]));
            const int i = 8 * k + 2 * q;
            y[i] = __fmul_rn(__fsub_rn(y[i], mf.x), sf.x);
            y[i + 1] = __fmul_rn(__fsub_rn(y[i + 1], mf.y), sf.y);
          }
        }
      }
      if (MODE == M_DELTA || MODE == M_AFFINE) {
        // a non-finite input or transform result (tensors.py:41-42) shows up here
        float chk = 0.0f;
#pragma unroll
        for (int i = 0; i < 64; ++i) chk = __fmaf_rn(y[i], 0.0f, chk);
        if (chk != 0.0f) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
      }
      cb0 = 64 * half;
      cb1 = 64 * half + 32;
    }
    float mn0, mx0, mn1, mx1;
    if constexpr (CERT) {
      // min / max of y = RN(S sc): RN is monotone, so scale the extremes of S
      // (B's chunk 1 holds -S: its scale -RN32(1/c) swaps them)
      float sn0, sx0, sn1, sx1;
      minmax32_3(y, sn0, sx0);
      minmax32_3(y + 32, sn1, sx1);
      const float sc0 = a.hr32, sc1 = half ? -a.hr32 : a.hr32;
      mn0 = __fmul_rn(sn0, sc0);
      mx0 = __fmul_rn(sx0, sc0);
      mn1 = __fadd_rn(__fmul_rn(half ? sx1 : sn1, sc1), 0.0f);  // -0 from the negation -> +0
      mx1 = __fadd_rn(__fmul_rn(half ? sn1 : sx1, sc1), 0.0f);
      if constexpr (G == 64) {  // group c = chunk c of both threads
        mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      } else if constexpr (G == 128) {  // one group per row
        mn0 = fminf(mn0, mn1);
        mx0 = fmaxf(mx0, mx1);
        mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mn1 = mn0;
        mx1 = mx0;
      }
      int w;
      int64_t bit;
      if constexpr (W != 0) {
        w = W;
        bit = row * (128 * W);
      } else {
        token_row_pos(g, a.heads, lh, t, w, bit);
      }
      unsigned short s0, z0, s1, z1;
      bool ok = cert_group(y, sc0, mn0, mx0, Dcert, w, a.rl[w], s0, z0);
      ok = cert_group(y + 32, sc1, mn1, mx1, Dcert, w, a.rl[w], s1, z1) && ok;
      if (valid) {  // one writer per group (both threads hold the same scale / zero)
        if constexpr (G == 32) {
          scales[row * 4 + half] = __ushort_as_half(s0);
          zeros[row * 4 + half] = __ushort_as_half(z0);
          scales[row * 4 + 2 + half] = __ushort_as_half(s1);
          zeros[row * 4 + 2 + half] = __ushort_as_half(z1);
        } else if constexpr (G == 64) {
          scales[row * 2 + half] = __ushort_as_half(half ? s1 : s0);
          zeros[row * 2 + half] = __ushort_as_half(half ? z1 : z0);
        } else if (half == 0) {
          scales[row] = __ushort_as_half(s0);
          zeros[row] = __ushort_as_half(z0);
        }
      }
      const int pok = __shfl_xor_sync(0xffffffffu, (int)ok, 1);  // every lane shuffles (no short circuit)
      ok = ok && pok != 0;
      // uncertified rows to the float64 pass (one atomic per warp), rows
      // with non-finite / huge inputs to the exact fixup pass
      // uncertified rows: one bit each in fix1_bits (the warp's 16 rows are
      // 16 consecutive bits of one word; a fire-and-forget atomic OR)
      {
        uint32_t m = __ballot_sync(0xffffffffu, row_ok && !ok && valid) & 0x55555555u;  // even lanes
        m = (m | (m >> 1)) & 0x33333333u;
        m = (m | (m >> 2)) & 0x0F0F0F0Fu;
        m = (m | (m >> 4)) & 0x00FF00FFu;
        m = (m | (m >> 8)) & 0x0000FFFFu;
        const int64_t row0 = WR ? tile * 16 : tile * kRows + (tid & ~31) / 2;
        if ((tid & 31) == 0 && m) atomicOr(a.fix1_bits + (row0 >> 5), m << (row0 & 31));
      }
      if (!row_ok && half == 0 && valid) a.fix_rows[atomicAdd(a.fix_count, 1u)] = (int32_t)row;
      need_fix = !row_ok || !ok;
      if (valid) {
        uint8_t* out = a.packed + (bit >> 3);
        if constexpr (W == 0) {
          pack32_dispatch(w, y, out + cb0 * w / 8);
          pack32_dispatch(w, y + 32, out + cb1 * w / 8);
        } else {
          pack32_store<W>(y, out + cb0 * W / 8);
          pack32_store<W>(y + 32, out + cb1 * W / 8);
        }
      }
      if (need_fix) flags = flags_before;
      continue;
    }
    if (MODE == M_IDENTITY && !F32) {
      // exact bf16 min/max, two per instruction; NaN / inf surface here
      minmax32_bf16(wv, mn0, mx0);
      minmax32_bf16(wv + 16, mn1, mx1);
      if (!(isfinite(mn0) && isfinite(mx0) && isfinite(mn1) && isfinite(mx1))) nanacc = 1.0f;
    } else if (MODE == M_IDENTITY) {
      minmax32(y, mn0, mx0);
      minmax32(y + 32, mn1, mx1);
      uint32_t amx = 0;  // fminf / fmaxf drop NaNs: test the bit patterns
#pragma unroll
      for (int i = 0; i < 64; ++i) amx = max(amx, wv[i] & 0x7FFFFFFFu);
      if (amx >= 0x7F800000u) nanacc = 1.0f;
    } else {
      minmax32(y, mn0, mx0);
      minmax32(y + 32, mn1, mx1);
      if (MODE == M_HADAMARD) {  // -0 from the negated half -> +0 (x + 0 = x otherwise)
        mn1 = __fadd_rn(mn1, 0.0f);
        mx1 = __fadd_rn(mx1, 0.0f);
      }
    }

    int w;
    int64_t bit;
    if constexpr (W != 0) {
        w = W;
        bit = row * (128 * W);
      } else {
        token_row_pos(g, a.heads, lh, t, w, bit);
      }
    quantize64<G>(y, mn0, mx0, mn1, mx1, cb0, cb1, w, a.rl[w], row * (128 / G), valid ? scales : nullptr, zeros,
                  hadlayout, half, flags);
    if (valid) {
      uint8_t* out = a.packed + (bit >> 3);
      if constexpr (W == 0) {
        pack32_dispatch(w, y, out + cb0 * w / 8);
        pack32_dispatch(w, y + 32, out + cb1 * w / 8);
      } else {
        pack32_store<W>(y, out + cb0 * W / 8);
        pack32_store<W>(y + 32, out + cb1 * W / 8);
      }
    }
    if (need_fix) flags = flags_before;  // the fixup pass sets this row's flags exactly
  }
  if (nanacc != 0.0f) flags |= KVC_FLAG_NONFINITE_INPUT;
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// The float64 pass behind the certified encoder: the rows it flagged in
// fix1_bits re-encoded with had64_row -- the reference's butterfly in stage
// order and the exact rounding of the uncertified kernel -- read straight
// from global memory.  Each warp scans 32 bitmap words (1024 rows) at a
// time, collects the flagged rows in shared memory and encodes them 16 at a
// time (a thread pair per row); rows this pass cannot prove exact go on to
// k_encode_fixup.
template <int G, int W, bool F32>
__global__ void __launch_bounds__(kThreads, 3) k_had64_list(const EncArgs a) {
  // per warp: rows carried over from the last window (< 16) + one window's
  __shared__ int32_t rows_s[kThreads / 32][1024 + 16];
  const Geo& g = a.g;
  const int tid = threadIdx.x, half = tid & 1, lane = tid & 31, warp = tid >> 5;
  const int64_t nrows = g.LH * g.T, nwords = (nrows + 31) / 32;
  __half* scales = reinterpret_cast<__half*>(a.meta);
  __half* zeros = scales + g.ngroups;
  uint32_t flags = 0;
  float nanacc = 0.0f;
  int32_t* list = rows_s[warp];
  // encode list[j0 .. j0 + 16) (rows past `total` repeat row j0 and store nothing)
  auto enc_batch = [&](int j0, int total) {
    const int j = j0 + (lane >> 1);
    const bool valid = j < total;
    const int64_t row = list[valid ? j : j0];
    const int64_t lh = row / g.T, t = row - lh * g.T;
    const int64_t eoff = a.paged ? out_index(a, lh, t, half * 64) : row * 128 + half * 64;
    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(a.kv) + eoff * (F32 ? 4 : 2));
    constexpr int NW = F32 ? 64 : 32;
    uint32_t wv[NW];
#pragma unroll
    for (int k = 0; k < NW / 4; ++k) {
      const uint4 cc = __ldg(src + k);
      wv[4 * k] = cc.x; wv[4 * k + 1] = cc.y; wv[4 * k + 2] = cc.z; wv[4 * k + 3] = cc.w;
    }
    const uint32_t flags_before = flags;
    __align__(8) float y[64];
    const bool need_fix = had64_row<F32>(wv, half, a, y, nanacc);
    if (need_fix && half == 0 && valid) a.fix_rows[atomicAdd(a.fix_count, 1u)] = (int32_t)row;
    float mn0, mx0, mn1, mx1;
    minmax32(y, mn0, mx0);
    minmax32(y + 32, mn1, mx1);
    mn1 = __fadd_rn(mn1, 0.0f);
    mx1 = __fadd_rn(mx1, 0.0f);
    int w;
    int64_t bit;
    token_row_pos(g, a.heads, lh, t, w, bit);
    const int cb0 = 32 * half, cb1 = 64 + 32 * half;
    quantize64<G>(y, mn0, mx0, mn1, mx1, cb0, cb1, w, a.rl[w], row * (128 / G), valid ? scales : nullptr, zeros,
                  true, half, flags);
    if (valid) {
      uint8_t* out = a.packed + (bit >> 3);
      if constexpr (W == 0) {
        pack32_dispatch(w, y, out + cb0 * w / 8);
        pack32_dispatch(w, y + 32, out + cb1 * w / 8);
      } else {
        pack32_store<W>(y, out + cb0 * W / 8);
        pack32_store<W>(y + 32, out + cb1 * W / 8);
      }
    }
    if (need_fix) flags = flags_before;
  };
  const int64_t stride = (int64_t)gridDim.x * (kThreads / 32) * 32;
  int q = 0;  // rows queued in list[0 .. q)
  for (int64_t w0 = ((int64_t)blockIdx.x * (kThreads / 32) + warp) * 32; w0 < nwords; w0 += stride) {
    const int64_t wi = w0 + lane;
    uint32_t bits = wi < nwords ? __ldcs(a.fix1_bits + wi) : 0u;
    const int c = __popc(bits);
    int off = c;  // inclusive scan of the counts over the warp
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off += q - c;
    while (bits) {
      const int64_t r = wi * 32 + __ffs(bits) - 1;
      list[off++] = (int32_t)r;
      // the row's bytes into L2 ahead of its encode
      const int64_t lh = r / g.T;
      const uint8_t* p0 = reinterpret_cast<const uint8_t*>(a.kv) +
                          (a.paged ? out_index(a, lh, r - lh * g.T, 0) : r * 128) * (F32 ? 4 : 2);
#pragma unroll
      for (int qq = 0; qq < (F32 ? 4 : 2); ++qq) asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + 128 * qq));
      bits &= bits - 1;
    }
    __syncwarp();
    q += total;
    // full batches of 16 rows now; fewer than 16 wait for the next window
    int j0 = 0;
    for (; j0 + 16 <= q; j0 += 16) enc_batch(j0, q);
    const int rem = q - j0;
    const int32_t carry = lane < rem ? list[j0 + lane] : 0;
    __syncwarp();
    if (lane < rem) list[lane] = carry;
    __syncwarp();
    q = rem;
  }
  if (q > 0) enc_batch(0, q);
  if (nanacc != 0.0f) flags |= KVC_FLAG_NONFINITE_INPUT;
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// ------------------------------------------------------------ decode kernel
// Dequantize + inverse transform of the thread's 64 values (hadamard layout:
// chunks at channels 32*half and 64 + 32*half; natural: 64*half, +32), one
// group per 32-value chunk (G >= 32).  y holds the magic floats 2^23 + symbol.
// zero + symbol * scale (quantize.py:178) is one FFMA2 per two values: the
// product of a symbol (<= 8 bits) and an fp16 scale (11-bit significand) is
// exact in fp32, so the fused and the reference's separate multiply and add
// round identically.  Returns false if a group's scale or zero is not finite
// -- the only way a dequantized or Hadamard-mixed value can be non-finite.
template <int MODE, int G>
__device__ __forceinline__ bool dec_core(float* y, const float* sc, const float* zr, int half, int64_t lh,
                                         const DecArgs& a, const float* aff_rc = nullptr,
                                         const float* aff_mu = nullptr, const float* aff_a = nullptr) {
  static_assert(G >= 32, "fast path groups");
  const Geo& g = a.g;
  bool groups_finite = true;
  float2* Y = reinterpret_cast<float2*>(y);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    groups_finite &= isfinite(sc[c]) && isfinite(zr[c]);
    const float2 s2 = f2(sc[c], sc[c]), z2 = f2(zr[c], zr[c]), m2 = f2(-8388608.0f, -8388608.0f);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float2& v = Y[16 * c + i];
      v = f2fma(f2add(v, m2), s2, z2);
    }
  }
  if (MODE == M_HADAMARD) {
    // inverse = the same orthonormal WHT (transforms.py:73-75), in fp32
    // (decode is held to tolerance), two values per FADD2: in-thread stages
    // over channel bits 0-4 and 6, one pair exchange for bit 5.  At the
    // bit-6 stage B (half 1) writes its outputs swapped (one FFMA2 by -1 each,
    // same roundings) so both threads send local 32 + k and keep local k.
#pragma unroll
    for (int i = 0; i < 32; ++i) {  // h = 1: the two lanes of one pair
      const float u = Y[i].x, v = Y[i].y;
      Y[i] = f2(u + v, u - v);
    }
#pragma unroll
    for (int h = 1; h < 16; h <<= 1) {  // h = 2..16 in float2 units
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if ((i & h) == 0) {
          const float2 u = Y[i], v = Y[i + h];
          Y[i] = f2add(u, v);
          Y[i + h] = f2sub(u, v);
        }
      }
    }
    const float sg = half ? -1.0f : 1.0f;
    const float2 sp = f2(sg, sg), sn = f2(-sg, -sg);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 u = Y[i], v = Y[16 + i];
      Y[i] = f2fma(v, sp, u);
      Y[16 + i] = f2fma(v, sn, u);
    }
    // A: local k = channel k, 32 + k = channel 32 + k; B: local k = channel
    // 64 + k, 32 + k = -(channel 96 + k) (own - r = -(r - own)), restored by
    // the sign of the final scale
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float2 send = Y[16 + k];
      const float2 r = f2(__shfl_xor_sync(0xffffffffu, send.x, 1), __shfl_xor_sync(0xffffffffu, send.y, 1));
      const float2 u = Y[k];
      Y[k] = f2add(u, r);
      Y[16 + k] = f2sub(u, r);
    }
    const float c = 0.08838834764831845f;  // RN32(1/sqrt(128))
    const float2 c0 = f2(c, c), c1 = half ? f2(-c, -c) : c0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      Y[i] = f2mul(Y[i], c0);
      Y[16 + i] = f2mul(Y[16 + i], c1);
    }
  } else if (MODE == M_AFFINE) {
    // x = y / a + mu with the division correctly rounded (div_by_rcp)
    if (aff_rc) {  // the tile's per-channel a, RN(1/a) and mu from shared memory
      const float4* rc4 = reinterpret_cast<const float4*>(aff_rc + half * 64);
      const float4* mu4 = reinterpret_cast<const float4*>(aff_mu + half * 64);
      const float4* a4 = reinterpret_cast<const float4*>(aff_a + half * 64);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float4 r = rc4[k], m = mu4[k], av = a4[k];
        y[4 * k] = __fadd_rn(div_by_rcp(y[4 * k], av.x, r.x), m.x);
        y[4 * k + 1] = __fadd_rn(div_by_rcp(y[4 * k + 1], av.y, r.y), m.y);
        y[4 * k + 2] = __fadd_rn(div_by_rcp(y[4 * k + 2], av.z, r.z), m.z);
        y[4 * k + 3] = __fadd_rn(div_by_rcp(y[4 * k + 3], av.w, r.w), m.w);
      }
    } else {
      const __half* mu = reinterpret_cast<const __half*>(a.meta + g.meta_affine_off) + lh * 128 + half * 64;
      const __half* scl = mu + g.LH * 128;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float av = __half2float(scl[i]);
        y[i] = __fadd_rn(div_by_rcp(y[i], av, __frcp_rn(av)), __half2float(mu[i]));
      }
    }
  }
  return groups_finite;
}

// bf16-pack 8 values
__device__ __forceinline__ uint4 pack_bf16x8(const float* y) {
  uint32_t p[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat162 b = __floats2bfloat162_rn(y[2 * q], y[2 * q + 1]);
    p[q] = *reinterpret_cast<uint32_t*>(&b);
  }
  return make_uint4(p[0], p[1], p[2], p[3]);
}

template <int MODE>
__device__ __forceinline__ void dec_flags(const float* y, bool groups_finite, uint32_t& flags) {
  if (MODE == M_AFFINE) {  // y * (1/a) + mu can overflow for a tiny fp16 a
    float chk = 0.0f;
#pragma unroll
    for (int i = 0; i < 64; ++i) chk = __fmaf_rn(y[i], 0.0f, chk);
    if (chk != 0.0f) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
  } else if (!groups_finite) {
    flags |= KVC_FLAG_NONFINITE_TRANSFORM;
  }
}

// Direct decode: any width layout, contiguous or paged output, bf16 or fp32.
template <int MODE, typename Tout, int G, int W>
__global__ void __launch_bounds__(kThreads, 4) k_dec128(const DecArgs a) {
  if (payload_rejected(a)) return;
  const Geo& g = a.g;
  const int64_t nrows = g.LH * g.T;
  const int64_t ntiles = (nrows + kRows - 1) / kRows;
  const int tid = threadIdx.x, half = tid & 1;
  const __half* scales = reinterpret_cast<const __half*>(a.meta);
  const __half* zeros = scales + g.ngroups;
  uint32_t flags = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kRows + (tid >> 1);
    const bool valid = row0 < nrows;
    const int64_t row = valid ? row0 : nrows - 1;  // tail lanes mirror a real row, store nothing
    const int64_t lh = row / g.T;
    const int64_t t = row - lh * g.T;
    int w;
    int64_t bit;
    token_row_pos(g, a.heads, lh, t, w, bit);
    constexpr bool had = MODE == M_HADAMARD;
    const int cb0 = had ? 32 * half : 64 * half;
    const int cb1 = had ? 64 + 32 * half : 64 * half + 32;
    const uint8_t* src = a.packed + (bit >> 3);
    if constexpr (W != 0) {
      // uniform width: the next tile's packed half-row and scales are at a
      // fixed stride; pull them into L1 while this tile computes
      const int64_t nrow = row + (int64_t)gridDim.x * kRows;
      if (nrow < nrows) {
        const uint8_t* np = src + (nrow - row) * 128 * W / 8;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(np + cb0 * W / 8));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(np + cb1 * W / 8));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(scales + nrow * (128 / G)));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(zeros + nrow * (128 / G)));
      }
    }
    __align__(8) float y[64];
    if constexpr (W == 0) {
      unpack32_dispatch<true>(w, src + cb0 * w / 8, y);
      unpack32_dispatch<true>(w, src + cb1 * w / 8, y + 32);
    } else {
      unpack32<W, true>(src + cb0 * W / 8, y);
      unpack32<W, true>(src + cb1 * W / 8, y + 32);
    }
    const int64_t gi0 = row * (128 / G) + cb0 / G, gi1 = row * (128 / G) + cb1 / G;
    const float sc[2] = {__half2float(scales[gi0]), __half2float(scales[gi1])};
    const float zr[2] = {__half2float(zeros[gi0]), __half2float(zeros[gi1])};
    const bool groups_finite = dec_core<MODE, G>(y, sc, zr, half, lh, a);
    if (!valid) continue;
    dec_flags<MODE>(y, groups_finite, flags);
    Tout* out = reinterpret_cast<Tout*>(a.out) + out_index(a, lh, t, 64 * half);
    if constexpr (sizeof(Tout) == 2) {
      uint4* o = reinterpret_cast<uint4*>(out);
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = pack_bf16x8(y + 8 * k);
    } else {
      float4* o = reinterpret_cast<float4*>(out);
#pragma unroll
      for (int k = 0; k < 16; ++k) o[k] = make_float4(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3]);
    }
  }
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// Staged decode (uniform width, contiguous bf16 output): per 64-row tile the
// packed rows (1024*W B), scales and zeros (each 64*(128/G)*2 B) are
// contiguous, so three 1-D bulk copies (cp.async.bulk, mbarrier completion)
// fill an NS-deep ring; the tile's 16 KB of bf16 rows is written to shared
// memory in the 128B-swizzled TMA layout (conflict-free 16 B stores) and
// leaves as one tensor store (double-buffered, bulk_group).  The partial last
// tile reads its inputs directly; the tensor store clips rows past the end.
// input ring depth: 3 stages, 2 for 8-bit rows (their 8 KB stages would
// otherwise hold the kernel at 3 CTAs/SM; with 2 it fits 4)
template <int W>
__host__ __device__ constexpr int dec_stages() {
  return W >= 8 ? 2 : 3;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(smem_u32(src))
               : "memory");
}
// paged cache view (64 ch, half, head, token row, layer): one box = bt tokens
// of one head
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int h, int r, int l) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(map),
               "r"(0), "r"(0), "r"(h), "r"(r), "r"(l), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// stage: packed rows, scales, zeros [, affine: the head's fp16 mu and a (256 B each)]
template <int MODE, int W, int G>
__host__ __device__ constexpr int dec_stage_bytes() {
  return 1024 * W + 2 * (64 * (128 / G) * 2) + (MODE == M_AFFINE ? 512 : 0);
}
template <int MODE, int W, int G>
__host__ __device__ constexpr int dec_smem_bytes() {
  return 2 * kTileBytes + dec_stages<W>() * dec_stage_bytes<MODE, W, G>() + 1024 + 64 + (MODE == M_AFFINE ? 6 * 128 * 4 : 0);
}

template <int MODE, int G, int W, bool PAGED>
__global__ void __launch_bounds__(kThreads, 4) k_dec128r(const __grid_constant__ CUtensorMap omap, const DecArgs a) {
  if (payload_rejected(a)) return;
  constexpr int NS = dec_stages<W>();
  constexpr int PK = 1024 * W, SB = 64 * (128 / G) * 2, STAGE = dec_stage_bytes<MODE, W, G>();
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned (128B swizzle atoms), indexed off smem_raw so the compiler keeps the
  // shared address space (LDS / STS rather than generic loads)
  uint8_t* obuf = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ibuf = obuf + 2 * kTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ibuf + NS * STAGE);
  // [2][128] RN(1/a), [2][128] mu, double-buffered by tile parity
  float* aff_tab = reinterpret_cast<float*>(ibuf + NS * STAGE + 64);
  const Geo& g = a.g;
  const int64_t nrows = g.LH * g.T;
  const int64_t ntiles = (nrows + kRows - 1) / kRows, nfull = nrows / kRows;
  const int tid = threadIdx.x, half = tid & 1, lr = tid >> 1;
  const uint32_t sw = (uint32_t)(tid & 7);
  const __half* scales = reinterpret_cast<const __half*>(a.meta);
  const __half* zeros = scales + g.ngroups;
  constexpr bool had = MODE == M_HADAMARD;
  const int cb0 = had ? 32 * half : 64 * half;
  const int cb1 = had ? 64 + 32 * half : 64 * half + 32;
  // affine: with whole-head tiles the head's mu / a ride along in the stage
  const bool tabs = MODE == M_AFFINE && g.T % kRows == 0;
  const uint8_t* aff_g = a.meta + g.meta_affine_off;
  auto issue = [&](int s, int64_t tile) {
    uint8_t* d = ibuf + s * STAGE;
    mbar_expect_tx(&full[s], (uint32_t)(PK + 2 * SB + (tabs ? 512 : 0)));
    bulk_g2s(d, a.packed + tile * PK, PK, &full[s]);
    bulk_g2s(d + PK, scales + tile * (SB / 2), SB, &full[s]);
    bulk_g2s(d + PK + SB, zeros + tile * (SB / 2), SB, &full[s]);
    if (tabs) {
      const int64_t lh = tile * kRows / g.T;
      bulk_g2s(d + PK + 2 * SB, aff_g + lh * 256, 256, &full[s]);
      bulk_g2s(d + PK + 2 * SB + 256, aff_g + (g.LH + lh) * 256, 256, &full[s]);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < nfull) issue(s, tile);
    }
  }
  uint32_t flags = 0;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % NS;
    const int64_t row0 = tile * kRows + lr;
    const bool valid = row0 < nrows;
    const int64_t row = valid ? row0 : nrows - 1;
    const int64_t lh = row / g.T;
    __align__(8) float y[64];
    float sc[2], zr[2];
    if (tile < nfull) {
      mbar_wait(&full[s], (uint32_t)((it / NS) & 1));
      const uint8_t* st = ibuf + s * STAGE;
      unpack32<W, true>(st + lr * 16 * W + cb0 * W / 8, y);
      unpack32<W, true>(st + lr * 16 * W + cb1 * W / 8, y + 32);
      const __half* ss = reinterpret_cast<const __half*>(st + PK) + lr * (128 / G);
      const __half* zz = reinterpret_cast<const __half*>(st + PK + SB) + lr * (128 / G);
      sc[0] = __half2float(ss[cb0 / G]);
      sc[1] = __half2float(ss[cb1 / G]);
      zr[0] = __half2float(zz[cb0 / G]);
      zr[1] = __half2float(zz[cb1 / G]);
    } else {  // the partial last tile
      const uint8_t* src = a.packed + row * 16 * W;
      unpack32<W, true>(src + cb0 * W / 8, y);
      unpack32<W, true>(src + cb1 * W / 8, y + 32);
      const int64_t gi0 = row * (128 / G) + cb0 / G, gi1 = row * (128 / G) + cb1 / G;
      sc[0] = __half2float(scales[gi0]);
      sc[1] = __half2float(scales[gi1]);
      zr[0] = __half2float(zeros[gi0]);
      zr[1] = __half2float(zeros[gi1]);
    }
    // output: each warp stores its own 16 rows (one TMA box, or one per page
    // run of the paged cache), so only the input ring needs a CTA barrier;
    // paged: the warp's page ids are fetched now, long before its store
    const int warp = tid >> 5, lane = tid & 31;
    int32_t page_id = 0;
    const int bt = a.page_tokens < 16 ? (int)a.page_tokens : 16;
    if (PAGED && lane * bt < 16) {
      const int64_t t0 = tile * kRows - (tile * kRows / g.T) * g.T + 16 * warp;
      page_id = a.block_table[(t0 + (int64_t)lane * bt) / a.page_tokens];
    }
    float* arc = aff_tab + (it & 1) * 384;
    float* amu = arc + 128;
    float* aav = arc + 256;
    if (tabs) {  // the tile's per-channel tables from the stage (every tile of the ring is full)
      const __half* mu = reinterpret_cast<const __half*>(ibuf + s * STAGE + PK + 2 * SB);
      const float av = __half2float(mu[128 + tid]);
      arc[tid] = __frcp_rn(av);
      aav[tid] = av;
      amu[tid] = __half2float(mu[tid]);
    }
    // contiguous output: one tensor store per tile from obuf[it & 1], whose
    // previous store (two tiles ago) must have been read out
    if (!PAGED && tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();  // stage s consumed by every thread; affine tables set; obuf[it & 1] free
    if (tid == 0) {
      const int64_t next = tile + (int64_t)NS * gridDim.x;
      if (next < nfull) {
        fence_proxy_async();
        issue(s, next);
      }
    }
    const bool groups_finite =
        dec_core<MODE, G>(y, sc, zr, half, lh, a, tabs ? arc : nullptr, tabs ? amu : nullptr, tabs ? aav : nullptr);
    if (valid) dec_flags<MODE>(y, groups_finite, flags);
    // paged: this warp's buffer of two tiles ago must have been read out
    if (PAGED && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (PAGED) __syncwarp();
    uint8_t* wb = obuf + (it & 1) * kTileBytes + warp * 4096;
    uint8_t* ob = wb + lane * 128;
#pragma unroll
    for (int k = 0; k < 8; ++k) *reinterpret_cast<uint4*>(ob + (((uint32_t)k ^ sw) << 4)) = pack_bf16x8(y + 8 * k);
    fence_proxy_async();
    if (!PAGED) {
      __syncthreads();
      if (tid == 0) {
        tma_store_2d(&omap, obuf + (it & 1) * kTileBytes, 0, (int)(tile * kThreads));
        bulk_commit();
      }
    } else {
      __syncwarp();
      const int64_t r0 = tile * kRows, lh0 = r0 / g.T, t0 = r0 - lh0 * g.T + 16 * warp;
      const int l = (int)(lh0 / g.H), h = (int)(lh0 - (int64_t)l * g.H);
      for (int j = 0; j < 16; j += bt) {
        const int64_t pg = __shfl_sync(0xffffffffu, page_id, j / bt);
        const int64_t row = pg * a.page_tokens + (t0 + j) % a.page_tokens;
        if (lane == 0) tma_store_5d(&omap, wb + j * 256, h, (int)row, l);
      }
      if (lane == 0) bulk_commit();
    }
  }
  if ((tid & 31) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// -------------------------------------------------------- host: tensor map
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_input_map(CUtensorMap* map, const void* kv, int64_t nrows, int box_rows = kThreads) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  // the (rows, 128) bf16 tensor viewed as (2*rows, 64): one 128 B half-row per box row
  cuuint64_t dims[2] = {64, (cuuint64_t)(2 * nrows)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(kv), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// the (rows, 128) fp32 tensor viewed as (4*rows, 32): one 128 B quarter row per box row
bool make_input_map_f32(CUtensorMap* map, const void* kv, int64_t nrows) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {32, (cuuint64_t)(4 * nrows)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, (cuuint32_t)(4 * kRows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(kv), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int MODE, int G, int W, bool F32>
cudaError_t launch_enc(const CUtensorMap& map, const EncArgs& a, int sm_count, cudaStream_t s) {
  constexpr int smem = enc_smem_bytes<F32>();
  auto k = k_enc128<MODE, G, W, F32, false>;
  const bool cert = MODE == M_HADAMARD && a.fix1_bits != nullptr;
  if constexpr (MODE == M_HADAMARD) {
    if (cert) {
      if constexpr (F32) {
        k = k_enc128<MODE, G, W, true, false, 1>;
        set_max_dyn_smem<k_enc128<MODE, G, W, true, false, 1>>(smem);
      } else if (a.paged) {
        k = k_enc128<MODE, G, W, false, true, 1>;
        set_max_dyn_smem<k_enc128<MODE, G, W, false, true, 1>>(smem);
      } else {
        k = k_enc128<MODE, G, W, false, false, 1>;
        set_max_dyn_smem<k_enc128<MODE, G, W, false, false, 1>>(smem);
      }
    }
  }
  if (!cert) {
    if constexpr (!F32) {
      if (a.paged) {
        k = k_enc128<MODE, G, W, false, true>;
        set_max_dyn_smem<k_enc128<MODE, G, W, false, true>>(smem);
      } else {
        set_max_dyn_smem<k_enc128<MODE, G, W, false, false>>(smem);
      }
    } else {
      set_max_dyn_smem<k_enc128<MODE, G, W, F32, false>>(smem);
    }
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = (a.g.LH * a.g.T + kRows - 1) / kRows;
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > ntiles) grid = ntiles;
  k<<<(unsigned)grid, kThreads, smem, s>>>(map, a);
  return cudaGetLastError();
}

template <int MODE, int G, bool F32>
cudaError_t launch_enc_w(const CUtensorMap& map, const EncArgs& a, int sm_count, cudaStream_t s) {
  const int w = a.g.quant == Q_UNIFORM ? a.g.bits : 0;
  switch (w) {
    case 2: return launch_enc<MODE, G, 2, F32>(map, a, sm_count, s);
    case 4: return launch_enc<MODE, G, 4, F32>(map, a, sm_count, s);
    case 8: return launch_enc<MODE, G, 8, F32>(map, a, sm_count, s);
    default: return launch_enc<MODE, G, 0, F32>(map, a, sm_count, s);
  }
}

template <int MODE, bool F32>
cudaError_t launch_enc_g(const CUtensorMap& map, const EncArgs& a, int sm_count, cudaStream_t s) {
  switch (a.g.group) {
    case 32: return launch_enc_w<MODE, 32, F32>(map, a, sm_count, s);
    case 64: return launch_enc_w<MODE, 64, F32>(map, a, sm_count, s);
    default: return launch_enc_w<MODE, 128, F32>(map, a, sm_count, s);
  }
}

template <bool F32>
cudaError_t launch_enc_t(const CUtensorMap& map, const EncArgs& a, int sm_count, cudaStream_t s) {
  switch (a.g.transform) {
    case T_IDENTITY: return launch_enc_g<M_IDENTITY, F32>(map, a, sm_count, s);
    case T_DELTA: return launch_enc_g<M_DELTA, F32>(map, a, sm_count, s);
    case T_HADAMARD: return launch_enc_g<M_HADAMARD, F32>(map, a, sm_count, s);
    default: return launch_enc_g<M_AFFINE, F32>(map, a, sm_count, s);
  }
}

// the staged kernel needs a contiguous bf16 output and 16-byte aligned tile
// bases for the bulk copies (packed rows, scales, zeros)
// paged cache [pages, page_tokens, H, 128] per layer (layer_stride elements)
// as a 5-D view (64 channels, half, head, token row, layer); the box is bt
// tokens of one head, the same 128B-swizzled smem rows as the contiguous map
bool make_paged_map(CUtensorMap* map, void* base, const Geo& g, int64_t layer_stride, int bt) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  const int64_t row_elems = g.H * 128;
  const int64_t rows = layer_stride / row_elems;  // token rows per layer in the pool
  cuuint64_t dims[5] = {64, 2, (cuuint64_t)g.H, (cuuint64_t)rows, (cuuint64_t)g.L};
  cuuint64_t strides[4] = {128, 256, (cuuint64_t)row_elems * 2, (cuuint64_t)layer_stride * 2};
  cuuint32_t box[5] = {64, 2, 1, (cuuint32_t)bt, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// paged encode input through the 5D map: whole 64-token tiles of one head,
// page runs that tile 64 tokens (4..64, or multiples of 64), a per-layer pool
// extent with 16-byte aligned strides
bool paged_input_ok(const EncArgs& a) {
  const int64_t pt = a.page_tokens, row_elems = a.g.H * 128;
  if (a.g.T % kRows != 0 || pt < 4 || (pt < kRows ? kRows % pt : pt % kRows) != 0) return false;
  if ((reinterpret_cast<uintptr_t>(a.kv) & 15u) != 0) return false;
  if (a.layer_stride <= 0 || a.layer_stride % row_elems != 0 || (a.layer_stride * 2) % 16 != 0) return false;
  return a.layer_stride / row_elems < (1ll << 31);
}

template <typename Tout, int W>
bool dec_staged_ok(const DecArgs& a) {
  if (sizeof(Tout) != 2 || W == 0) return false;
  const int64_t nrows = a.g.LH * a.g.T;
  if (2 * nrows >= (1ll << 31)) return false;
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!(al(a.packed) && al(a.meta) && al(a.out) && (a.g.ngroups % 8) == 0)) return false;
  if (a.paged) {
    // whole 64-token tiles of one head, page runs of >= 4 tokens (1 KB-aligned
    // smem sub-boxes), a per-layer pool extent
    const int64_t pt = a.page_tokens, row_elems = a.g.H * 128;
    if (a.g.T % kRows != 0 || pt < 4 || (pt < 16 ? 16 % pt : pt % 16) != 0) return false;
    if (a.layer_stride <= 0 || a.layer_stride % row_elems != 0 || (a.layer_stride * 2) % 16 != 0) return false;
    if (a.layer_stride / row_elems >= (1ll << 31)) return false;
  }
  return true;
}

template <int MODE, typename Tout, int G, int W>
cudaError_t launch_dec_gw(const DecArgs& a, int sm_count, cudaStream_t s) {
  if constexpr (sizeof(Tout) == 2 && W != 0) {
    CUtensorMap omap;
    const bool mapped = dec_staged_ok<Tout, W>(a) &&
                        (a.paged ? make_paged_map(&omap, a.out, a.g, a.layer_stride, (int)std::min<int64_t>(a.page_tokens, 16))
                                 : make_input_map(&omap, a.out, a.g.LH * a.g.T));
    if (mapped) {
      auto k = a.paged ? k_dec128r<MODE, G, W, true> : k_dec128r<MODE, G, W, false>;
      constexpr int smem = dec_smem_bytes<MODE, W, G>();
      if (a.paged) {
        set_max_dyn_smem<k_dec128r<MODE, G, W, true>>(smem);
      } else {
        set_max_dyn_smem<k_dec128r<MODE, G, W, false>>(smem);
      }
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem);
      if (per_sm < 1) per_sm = 1;
      const int64_t need = (a.g.LH * a.g.T + kRows - 1) / kRows;
      int64_t grid = (int64_t)sm_count * per_sm;
      if (grid > need) grid = need;
      k<<<(unsigned)grid, kThreads, smem, s>>>(omap, a);
      return cudaGetLastError();
    }
  }
  auto k = k_dec128<MODE, Tout, G, W>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.g.LH * a.g.T + kRows - 1) / kRows;
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > need) grid = need;
  k<<<(unsigned)grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

template <int MODE, typename Tout, int G>
cudaError_t launch_dec_g(const DecArgs& a, int sm_count, cudaStream_t s) {
  const int w = a.g.quant == Q_UNIFORM ? a.g.bits : 0;
  switch (w) {
    case 2: return launch_dec_gw<MODE, Tout, G, 2>(a, sm_count, s);
    case 4: return launch_dec_gw<MODE, Tout, G, 4>(a, sm_count, s);
    case 8: return launch_dec_gw<MODE, Tout, G, 8>(a, sm_count, s);
    default: return launch_dec_gw<MODE, Tout, G, 0>(a, sm_count, s);
  }
}

template <int MODE, typename Tout>
cudaError_t launch_dec(const DecArgs& a, int sm_count, cudaStream_t s) {
  switch (a.g.group) {
    case 32: return launch_dec_g<MODE, Tout, 32>(a, sm_count, s);
    case 64: return launch_dec_g<MODE, Tout, 64>(a, sm_count, s);
    default: return launch_dec_g<MODE, Tout, 128>(a, sm_count, s);
  }
}

}  // namespace

bool fast128_applicable(const Geo& g) {
  if (g.C != 128 || g.uchan) return false;
  if (!(g.group == 32 || g.group == 64 || g.group == 128)) return false;
  if (g.transform == T_AFFINE && (g.meta_affine_off % 16) != 0) return false;
  return true;
}

template <int G, int W>
cudaError_t launch_had64_list_gw(const EncArgs& a, int sm_count, cudaStream_t s) {
  auto k = a.g.in_dtype == KVC_DTYPE_F32 ? k_had64_list<G, W, true> : k_had64_list<G, W, false>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  k<<<(unsigned)(sm_count * per_sm), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

template <int G>
cudaError_t launch_had64_list_g(const EncArgs& a, int sm_count, cudaStream_t s) {
  switch (a.g.quant == Q_UNIFORM ? a.g.bits : 0) {
    case 2: return launch_had64_list_gw<G, 2>(a, sm_count, s);
    case 4: return launch_had64_list_gw<G, 4>(a, sm_count, s);
    case 8: return launch_had64_list_gw<G, 8>(a, sm_count, s);
    default: return launch_had64_list_gw<G, 0>(a, sm_count, s);
  }
}

// the float64 pass over the rows the certified encoder listed
cudaError_t launch_had64_list(const EncArgs& a, int sm_count, cudaStream_t s) {
  ProfScope ps("encode_had64_list", s);
  switch (a.g.group) {
    case 32: return launch_had64_list_g<32>(a, sm_count, s);
    case 64: return launch_had64_list_g<64>(a, sm_count, s);
    default: return launch_had64_list_g<128>(a, sm_count, s);
  }
}

cudaError_t launch_encode_fast128(const EncArgs& a, int sm_count, cudaStream_t s) {
  const bool f32 = a.g.in_dtype == KVC_DTYPE_F32;
  const int64_t nrows = a.g.LH * a.g.T;
  if ((f32 ? 4 : 2) * nrows >= (1ll << 31)) return launch_encode_generic(a, s);
  CUtensorMap map;
  if (a.paged) {
    if (f32 || !paged_input_ok(a) || !make_paged_map(&map, const_cast<void*>(a.kv), a.g, a.layer_stride,
                                                     (int)std::min<int64_t>(a.page_tokens, kRows)))
      return launch_encode_generic(a, s);
  } else if (!(f32 ? make_input_map_f32(&map, a.kv, nrows)
                   : make_input_map(&map, a.kv, nrows,
                                    (a.g.transform == T_HADAMARD && a.fix1_bits) ? 32 : kThreads))) {
    return launch_encode_generic(a, s);
  }
  cudaError_t e;
  {
    ProfScope ps("encode_fast128", s);
    e = f32 ? launch_enc_t<true>(map, a, sm_count, s) : launch_enc_t<false>(map, a, sm_count, s);
  }
  if (e == cudaSuccess && a.fix1_bits && a.g.transform == T_HADAMARD) e = launch_had64_list(a, sm_count, s);
  return e;
}

cudaError_t launch_decode_fast128(const DecArgs& a, int sm_count, cudaStream_t s) {
  if (a.g.transform == T_DELTA) return launch_decode_generic(a, s);
  ProfScope ps("decode_fast128", s);
  const bool bf = a.g.out_dtype == KVC_DTYPE_BF16;
  switch (a.g.transform) {
    case T_IDENTITY: return bf ? launch_dec<M_IDENTITY, __nv_bfloat16>(a, sm_count, s) : launch_dec<M_IDENTITY, float>(a, sm_count, s);
    case T_HADAMARD: return bf ? launch_dec<M_HADAMARD, __nv_bfloat16>(a, sm_count, s) : launch_dec<M_HADAMARD, float>(a, sm_count, s);
    default: return bf ? launch_dec<M_AFFINE, __nv_bfloat16>(a, sm_count, s) : launch_dec<M_AFFINE, float>(a, sm_count, s);
  }
}

}  // namespace kvc
