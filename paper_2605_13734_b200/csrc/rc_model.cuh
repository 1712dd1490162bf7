// Small-alphabet (A = 2^w <= 16) adaptive frequency model of codecs.py:188-242
// in registers, shared by the range coder kernels (rc_small.cu) and the
// fused quantize + range-code kernels (fused_rc.cu).
#pragma once
#include <stdint.h>

#include "rc_coder.cuh"

namespace kvc {

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
  // Variants for the fused kernels (fused_rc.cu): the total is the warp-
  // uniform A + 32 i (no halving inside a block), passed in rather than kept
  // per lane, and the symbol arrives top-aligned in t (symbol = t >> 28, the
  // bits below are ignored), so s >= k is one compare against k << 28.
  __device__ __forceinline__ void lookup_top(uint32_t t, uint32_t tot, uint32_t& lo, uint32_t& hi) const {
    lo = 0;
    hi = C[1];
#pragma unroll
    for (int k = 1; k < A; ++k) {
      const bool ge = t >= ((uint32_t)k << 28);
      lo = ge ? C[k] : lo;
      hi = ge ? (k + 1 < A ? C[k + 1] : tot) : hi;
    }
  }
  __device__ __forceinline__ void add_top(uint32_t t) {
#pragma unroll
    for (int k = 1; k < A; ++k) C[k] += (t < ((uint32_t)k << 28)) ? 32u : 0u;
  }
  __device__ __forceinline__ void add_only(uint32_t s) {
#pragma unroll
    for (int k = 1; k < A; ++k) C[k] += (s < (uint32_t)k) ? 32u : 0u;
  }
  // Decoder search for A = 8, 16 without the division: binary search over
  // the cumulative counts, s = largest with x >= unit * C[s] (<=> floor(x /
  // unit) >= C[s]; the reference's clamp to total - 1 never changes s since
  // C[A-1] <= total - 1).  Level `bit` compares against C[s + bit], chosen
  // among the A / (2 bit) candidates by a select tree on the bits decided so
  // far; plo / phi are the last accepted / rejected unit * C (unit * tot if
  // none rejected).
  __device__ __forceinline__ uint32_t bsearch(uint32_t x, uint32_t unit, uint32_t tot, uint32_t& plo,
                                              uint32_t& phi) const {
    uint32_t s = 0;
    plo = 0;
    phi = unit * tot;
#pragma unroll
    for (int L = W - 1; L >= 0; --L) {
      const uint32_t bit = 1u << L;
      constexpr int kMax = A / 2;
      uint32_t cand[kMax];
      const int n = A / (2 * (int)bit);  // candidates C[(2i + 1) bit], i = s / (2 bit)
#pragma unroll
      for (int i = 0; i < kMax; ++i)
        if (i < n) cand[i] = C[(2 * i + 1) * bit];
      // select tree: fold pairs by the decided bits, lowest decided bit first
#pragma unroll
      for (int lev = 0; (1 << lev) < n; ++lev) {
        const bool hi = (s >> (L + 1 + lev)) & 1u;
#pragma unroll
        for (int i = 0; i < kMax / 2; ++i)
          if (2 * i + 1 < (n >> lev)) cand[i] = hi ? cand[2 * i + 1] : cand[2 * i];
      }
      const uint32_t v = unit * cand[0];
      const bool ok = x >= v;
      s += ok ? bit : 0u;
      plo = ok ? v : plo;
      phi = ok ? phi : v;
    }
    return s;
  }
  __device__ __forceinline__ uint32_t find_t(uint32_t x, uint32_t unit, uint32_t tot, uint32_t& plo,
                                             uint32_t& phi) const {
    if constexpr (A <= 4) {
      uint32_t s = 0;
      plo = 0;
      phi = unit * C[1];
#pragma unroll
      for (int k = 1; k < A; ++k) {
        const uint32_t pk = unit * C[k];
        const uint32_t pn = unit * (k + 1 < A ? C[k + 1] : tot);
        const bool ge = x >= pk;
        s += ge ? 1u : 0u;
        plo = ge ? pk : plo;
        phi = ge ? pn : phi;
      }
      return s;
    } else {
      return bsearch(x, unit, tot, plo, phi);
    }
  }
  // Encoder step for the fused kernels: (lo, hi) = (C[s], C[s+1]) and then
  // f[s] += 32, sharing the three predicates s >= k (A = 4: one predicated
  // instruction per select / add, written in PTX because the compiler
  // otherwise recomputes the compares and splits each add into two).
  __device__ __forceinline__ void step_top(uint32_t t, uint32_t tot, uint32_t& lo, uint32_t& hi) {
    if constexpr (A == 4) {
      asm("{\n\t.reg .pred p1, p2, p3;\n\t"
          "setp.ge.u32 p1, %5, 0x10000000;\n\tsetp.ge.u32 p2, %5, 0x20000000;\n\tsetp.ge.u32 p3, %5, 0x30000000;\n\t"
          "selp.u32 %0, %2, 0, p1;\n\t@p2 mov.u32 %0, %3;\n\t@p3 mov.u32 %0, %4;\n\t"
          "selp.u32 %1, %3, %2, p1;\n\t@p2 mov.u32 %1, %4;\n\t@p3 mov.u32 %1, %6;\n\t"
          "@!p1 add.u32 %2, %2, 32;\n\t@!p2 add.u32 %3, %3, 32;\n\t@!p3 add.u32 %4, %4, 32;\n\t}"
          : "=&r"(lo), "=&r"(hi), "+r"(C[1]), "+r"(C[2]), "+r"(C[3])
          : "r"(t), "r"(tot));
    } else if constexpr (A == 2) {
      asm("{\n\t.reg .pred p1;\n\tsetp.ge.u32 p1, %3, 0x10000000;\n\t"
          "selp.u32 %0, %2, 0, p1;\n\tselp.u32 %1, %4, %2, p1;\n\t@!p1 add.u32 %2, %2, 32;\n\t}"
          : "=&r"(lo), "=&r"(hi), "+r"(C[1])
          : "r"(t), "r"(tot));
    } else {
      lookup_top(t, tot, lo, hi);
      add_top(t);
    }
  }
  // Decoder step for the fused kernels (A <= 4): finds the symbol from
  // x = code - low, returns unit*C[s], unit*C[s+1] and the dequantized value
  // val[s] (precomputed per group), then f[s] += 32.
  __device__ __forceinline__ float dstep(uint32_t x, uint32_t unit, uint32_t tot, const float* val, uint32_t& plo,
                                         uint32_t& phi) {
    static_assert(A <= 4, "dstep: small alphabets");
    float v;
    if constexpr (A == 4) {
      const uint32_t pk1 = unit * C[1], pk2 = unit * C[2], pk3 = unit * C[3], pt = unit * tot;
      asm("{\n\t.reg .pred p1, p2, p3;\n\t"
          "setp.ge.u32 p1, %6, %7;\n\tsetp.ge.u32 p2, %6, %8;\n\tsetp.ge.u32 p3, %6, %9;\n\t"
          "selp.u32 %0, %7, 0, p1;\n\t@p2 mov.u32 %0, %8;\n\t@p3 mov.u32 %0, %9;\n\t"
          "selp.u32 %1, %8, %7, p1;\n\t@p2 mov.u32 %1, %9;\n\t@p3 mov.u32 %1, %10;\n\t"
          "selp.f32 %2, %12, %11, p1;\n\t@p2 mov.f32 %2, %13;\n\t@p3 mov.f32 %2, %14;\n\t"
          "@!p1 add.u32 %3, %3, 32;\n\t@!p2 add.u32 %4, %4, 32;\n\t@!p3 add.u32 %5, %5, 32;\n\t}"
          : "=&r"(plo), "=&r"(phi), "=&f"(v), "+r"(C[1]), "+r"(C[2]), "+r"(C[3])
          : "r"(x), "r"(pk1), "r"(pk2), "r"(pk3), "r"(pt), "f"(val[0]), "f"(val[1]), "f"(val[2]), "f"(val[3]));
    } else {
      const uint32_t pk1 = unit * C[1], pt = unit * tot;
      asm("{\n\t.reg .pred p1;\n\tsetp.ge.u32 p1, %4, %5;\n\t"
          "selp.u32 %0, %5, 0, p1;\n\tselp.u32 %1, %6, %5, p1;\n\tselp.f32 %2, %8, %7, p1;\n\t"
          "@!p1 add.u32 %3, %3, 32;\n\t}"
          : "=&r"(plo), "=&r"(phi), "=&f"(v), "+r"(C[1])
          : "r"(x), "r"(pk1), "r"(pt), "f"(val[0]), "f"(val[1]));
    }
    return v;
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
      return bsearch(x, unit, total, plo, phi);
    }
  }
};

template <int W>
__device__ __forceinline__ uint32_t dec_symbol_small(RcDec& d, SModel<W>& m, uint32_t unit) {
  // code < low only in a malformed stream; x = 0 then yields symbol 0 with
  // the same bounds the reference's search gives for a negative target
  const uint32_t x = d.offset();
  uint32_t plo, phi;
  const uint32_t s = m.find(x, unit, plo, phi);
  d.advance(plo, phi);
  m.add(s);
  return s;
}

}  // namespace kvc
