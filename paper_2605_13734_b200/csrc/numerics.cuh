// Exact-arithmetic device helpers.  Each reproduces one numpy expression of
// the reference bit-for-bit while avoiding the slow B200 pipes we measured
// (tools/ubench/pipes.cu: F2F f32<->f64 8-16/clk/SM, FRND 16, __fdiv_rn 3,
// __ddiv_rn 1.2 vs 64 DADD / 128 FFMA per clk per SM).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "kvc_internal.h"

namespace kvc {

constexpr float kMagicRound = 12582912.0f;  // 1.5 * 2^23: x + M rounds x to an integer, half-to-even
constexpr uint32_t kMagicBits = 0x4B400000u;

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

template <typename T>
__device__ __forceinline__ float load_f32(const T* p, int64_t i);
template <>
__device__ __forceinline__ float load_f32<float>(const float* p, int64_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ float load_f32<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return bf16_to_f32(__ldg(reinterpret_cast<const unsigned short*>(p) + i));
}

template <typename T>
__device__ __forceinline__ void store_f32(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void store_f32<float>(float* p, int64_t i, float v) { p[i] = v; }
template <>
__device__ __forceinline__ void store_f32<__nv_bfloat16>(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

// fp16 affine parameters sit right after the class bits in the metadata, so
// their byte offset can be odd: the generic kernels move them a byte at a time
__device__ __forceinline__ float ld_meta_half(const uint8_t* base, int64_t i) {
  const uint8_t* q = base + 2 * i;
  return __half2float(__ushort_as_half((unsigned short)(q[0] | (q[1] << 8))));
}
__device__ __forceinline__ void st_meta_half(uint8_t* base, int64_t i, float v) {
  // the f16 bits are widened to 32 bits inside PTX: ptxas (12.9) turns a byte
  // store of a 16-bit f16 register into a value conversion (F2I.U8.F16)
  unsigned w;
  asm("{\n\t.reg .b16 h;\n\tcvt.rn.f16.f32 h, %1;\n\tcvt.u32.u16 %0, h;\n\t}" : "=r"(w) : "f"(v));
  base[2 * i] = (uint8_t)(w & 0xffu);
  base[2 * i + 1] = (uint8_t)(w >> 8);
}

// ---------------------------------------------------------------------------
// Hadamard (transforms.py:33-47, :62): fp64 butterfly, / RN64(sqrt n), -> f32.
//
// An fp32 bit pattern reinterpreted as the high/low words of a double is the
// same value times 2^-896 for every finite input (zero, subnormal, normal):
// the 8-bit exponent field lands in the 11-bit field unbiased by 896.  The
// butterfly then runs on exactly scaled values (no rounding differs: tiny
// sums are exact multiples of 2^-1045, representable even as fp64
// subnormals), so the reference's fp64 results are reproduced without the
// 16/clk/SM F2F.F64.F32 conversion.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double f32bits_scaled_f64(uint32_t f) {
  return __hiloint2double((int)(((int)f >> 3) & (int)0x8FFFFFFF), (int)(f << 29));
}

// y = RN32(RN64(S / c)) where Sp = S * 2^-896 exactly, hk = 2^896 * RN64(1/c),
// hc = c.  Fast path: RN64(S * RN64(1/c)) rounded to f32 with integer ops;
// exact __ddiv_rn fallback when that product lies within 4 ulp64 of an f32
// rounding boundary or outside the normal f32 range.
// Exact fallback (cold): signed zero, f32 subnormal / overflow range, or a
// product within 4 ulp64 of an f32 rounding boundary.
static __device__ __noinline__ float hadamard_slow(double Sp, double hc, uint32_t* flags) {
  uint32_t H = (uint32_t)__double2hiint(Sp), Lw = (uint32_t)__double2loint(Sp);
  if (((H & 0x7FFFFFFFu) | Lw) == 0u) return __uint_as_float(H & 0x80000000u);  // signed zero
  float y = __double2float_rn(__ddiv_rn(Sp * 0x1p896, hc));
  if (!isfinite(y)) *flags |= KVC_FLAG_NONFINITE_TRANSFORM;
  return y;
}

// Branch-free fast path: q = RN64(S * RN64(1/c)), rounded to f32 by the
// hardware conversion (one F2F.F32.F64; its pipe has room in this issue-bound
// kernel).  q can differ from the reference's RN64(S / c) by one ulp64, which
// changes the f32 result only next to an f32 rounding boundary: `slow` is set
// when q lies within 4 ulp64 of a midpoint or outside the normal f32 range
// [2^-126, 2^128) (where the boundaries sit elsewhere), and the caller then
// takes hadamard_slow.
__device__ __forceinline__ float hadamard_fast(double Sp, double hk, bool& slow) {
  const double q = Sp * hk;
  const uint32_t H = (uint32_t)__double2hiint(q), Lw = (uint32_t)__double2loint(q);
  slow = ((H & 0x7FFFFFFFu) - 0x38100000u >= 0x0FE00000u) | (((Lw & 0x1FFFFFFFu) - 0x0FFFFFFCu) <= 8u);
  return __double2float_rn(q);
}

__device__ __forceinline__ float hadamard_out(double Sp, double hk, double hc, uint32_t& flags) {
  bool slow;
  float y = hadamard_fast(Sp, hk, slow);
  return slow ? hadamard_slow(Sp, hc, &flags) : y;
}

// ---------------------------------------------------------------------------
// Group scale (quantize.py:146): float16(float64(d) / levels), d = fp32 max-min.
// d/levels never rounds onto an fp16 midpoint through fp64 unless it is one
// exactly, so this equals RN16(d/levels); computed in fp32 and checked for
// proximity to an fp16 boundary (relative 2^-20 vs an error of 2^-23).
// ---------------------------------------------------------------------------
static __device__ __noinline__ unsigned short scale16_slow(float d, float levels) {
  return __half_as_ushort(__double2half(__ddiv_rn((double)d, (double)levels)));
}

__device__ __forceinline__ __half scale16_exact(float d, float levels, float rl) {
  float q = __fmul_rn(d, rl);
  __half a = __float2half_rn(__fmul_rn(q, 1.00000095367431640625f));
  __half b = __float2half_rn(__fmul_rn(q, 0.99999904632568359375f));
  if (__half_as_ushort(a) == __half_as_ushort(b)) return a;
  return __ushort_as_half(scale16_slow(d, levels));
}

// Per-group quantizer state (quantize.py:146-154).
struct GroupQ {
  float s, z, r, lv;
  int mode;  // 0 fast, 1 all-zero symbols (scale 0), 2 exact slow path (inf scale/zero)
};

__device__ __forceinline__ GroupQ group_setup(float mn, float mx, int w, float rl, __half& s16, __half& z16,
                                              uint32_t& flags) {
  GroupQ q;
  q.lv = (float)((1 << w) - 1);
  float d = __fsub_rn(mx, mn);
  s16 = scale16_exact(d, q.lv, rl);
  z16 = __float2half_rn(mn);
  q.s = __half2float(s16);
  q.z = __half2float(z16);
  if (!(q.s > 0.0f)) {
    q.mode = 1;
    q.r = 0.0f;
  } else if (isinf(q.s) || isinf(q.z)) {
    q.mode = 2;
    q.r = 0.0f;
    flags |= KVC_FLAG_FP16_RANGE;
  } else {
    q.mode = 0;
    q.r = __frcp_rn(q.s);
  }
  if (isinf(q.z)) flags |= KVC_FLAG_FP16_RANGE;
  return q;
}

// rint(fp32((v - z) / s)) clipped to [0, levels] (quantize.py:152-154).
// Reciprocal + two FMAs reproduce the IEEE quotient's clipped rint
// (exhaustively checked over all fp16 scales with |v - z| <= 2^24, which
// holds whenever scale and zero are finite: tools/numerics/markstein_check.c);
// rint is the 1.5*2^23 magic add, whose low byte is the symbol.
__device__ __forceinline__ float quant_magic(float v, const GroupQ& q) {
  float d = __fsub_rn(v, q.z);
  float q0 = __fmul_rn(d, q.r);
  float e = __fmaf_rn(-q0, q.s, d);
  float q1 = __fmaf_rn(e, q.r, q0);
  float c = fminf(fmaxf(q1, 0.0f), q.lv);
  return __fadd_rn(c, kMagicRound);
}

__device__ __forceinline__ uint32_t quant_fast(float v, const GroupQ& q) {
  return __float_as_uint(quant_magic(v, q)) - kMagicBits;
}

// exact slow path (cold): infinite fp16 scale or zero
static __device__ __noinline__ uint32_t quant_slow(float v, float z, float s, float lv) {
  float r = rintf(__fdiv_rn(__fsub_rn(v, z), s));
  r = fminf(fmaxf(r, 0.0f), lv);  // NaN -> 0 like numpy's uint8 cast on x86
  return (uint32_t)r;
}

__device__ __forceinline__ uint32_t quant_one(float v, const GroupQ& q) {
  if (q.mode == 0) return quant_fast(v, q);
  if (q.mode == 1) return 0u;
  return quant_slow(v, q.z, q.s, q.lv);
}

// y / a correctly rounded (the oracle's affine inverse divides)
// from r = RN(1/a): q0 = RN(y r), the exact residual y - a q0 by one FMA, and
// one correction step RN(q0 + r (y - a q0)) (Markstein: r correctly rounded
// and q0 within an ulp give the correctly rounded quotient; a is an fp16
// value, so no intermediate over/underflows for finite decoded y).
__device__ __forceinline__ float div_by_rcp(float y, float a, float r) {
  const float q0 = __fmul_rn(y, r);
  return __fmaf_rn(__fmaf_rn(-q0, a, y), r, q0);
}

// dequantize (quantize.py:178): zero + symbol*scale, unfused.
__device__ __forceinline__ float dequant(uint32_t sym, float s, float z) {
  return __fadd_rn(z, __fmul_rn(__uint_as_float(0x4B000000u | sym) - 8388608.0f, s));
}

// read a w-bit MSB-first symbol starting at absolute bit p
__device__ __forceinline__ uint32_t read_sym(const uint8_t* buf, int64_t p, int w) {
  int64_t byte = p >> 3;
  int sh = (int)(p & 7);
  uint32_t v = (uint32_t)buf[byte] << 8;
  if (sh + w > 8) v |= buf[byte + 1];
  return (v >> (16 - sh - w)) & ((1u << w) - 1u);
}

}  // namespace kvc
