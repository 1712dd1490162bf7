// Range coder state machines shared by the small- and large-alphabet coders
// (codecs.py:245-307: 32-bit carry-less coder, TOP = 2^24, BOTTOM = 2^16).
//
// The reference renormalizes one byte per loop iteration.  On a GPU that
// loop diverges across the lanes of a warp (each lane codes its own block),
// so the common case is done in closed form: after `low += unit*cum; range =
// unit*freq` the bytes the loop would shift out while the top bytes of low
// and low + range agree are exactly the leading equal bytes,
//   k = carry ? 0 : clz(low ^ (low + range)) / 8      (0..3),
// because shifting a carry-free pair keeps it carry-free.  Those k bytes move
// in one step; only the rare underflow case (top bytes differ but range <
// BOTTOM, codecs.py:258-259) falls back to the reference's byte loop.
#pragma once
#include <stdint.h>

namespace kvc {

constexpr uint32_t kRcTop = 1u << 24;
constexpr uint32_t kRcBot = 1u << 16;

__device__ __forceinline__ uint32_t rc_clz(uint32_t x) {  // x != 0
  uint32_t r;
  asm("bfind.shiftamt.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// 8 * (number of settled leading bytes): 0, 8, 16 or 24 (branch-free: the
// compiler would otherwise branch around the bit scan)
__device__ __forceinline__ uint32_t rc_settled_shift(uint32_t low, uint32_t range) {
  uint32_t sh;
  asm("{\n\t.reg .u32 t, x, c;\n\t.reg .pred p;\n\t"
      "add.u32 t, %1, %2;\n\txor.b32 x, %1, t;\n\tbfind.shiftamt.u32 c, x;\n\tand.b32 c, c, 24;\n\t"
      "setp.lt.u32 p, t, %1;\n\tselp.u32 %0, 0, c, p;\n\t}"
      : "=r"(sh)
      : "r"(low), "r"(range));
  return sh;
}

// Encoder: output bytes accumulate in a 64-bit window (newest byte lowest)
// and are stored one big-endian word at a time.
struct RcEnc {
  uint32_t low, range;
  uint32_t whi, wlo;
  uint32_t nb;    // bits emitted
  uint32_t* out;

  __device__ __forceinline__ void init(uint32_t* o) {
    low = 0;
    range = 0xFFFFFFFFu;
    whi = wlo = 0;
    nb = 0;
    out = o;
  }
  // shift the top sh/8 <= 3 bytes of low out (codecs.py:261-263, once per byte)
  __device__ __forceinline__ void put_sh(uint32_t sh) {
    const uint32_t bytes = __funnelshift_l(low, 0u, sh);  // low >> (32 - sh), 0 for sh = 0
    whi = __funnelshift_l(wlo, whi, sh);
    wlo = (wlo << sh) | bytes;
    const uint32_t o = nb;
    nb += sh;
    if ((nb ^ o) >= 32u) out[(nb >> 5) - 1] = __byte_perm(__funnelshift_r(wlo, whi, nb), 0, 0x0123);
    low <<= sh;
    range <<= sh;
  }
  __device__ __forceinline__ void put(uint32_t k) { put_sh(8u * k); }
  // put_sh with the shifts done as multiplies by p = 2^sh: on the FMA pipe,
  // off the saturated ALU pipe (low * p yields the shifted low and the
  // outgoing bytes in one IMAD.WIDE)
  __device__ __forceinline__ void put_mul(uint32_t sh) {
    uint32_t p;
    asm("shl.b32 %0, 1, %1;" : "=r"(p) : "r"(sh));  // opaque: keep the multiplies
    const uint64_t lw = (uint64_t)low * p;
    whi = __funnelshift_l(wlo, whi, sh);
    wlo = wlo * p + (uint32_t)(lw >> 32);
    low = (uint32_t)lw;
    range *= p;
    const uint32_t o = nb;
    nb += sh;
    if ((nb ^ o) >= 32u) out[(nb >> 5) - 1] = __byte_perm(__funnelshift_r(wlo, whi, nb), 0, 0x0123);
  }
  __device__ __forceinline__ void underflow() {  // the reference's loop, from a settled state
    for (;;) {
      const uint32_t t = low + range;
      if (t < low || (low ^ t) >= kRcTop) {
        if (range >= kRcBot) break;
        range = (0u - low) & (kRcBot - 1u);
      }
      put(1);
    }
  }
  __device__ __forceinline__ void encode(uint32_t unit, uint32_t cum, uint32_t freq) {
    low += unit * cum;
    range = unit * freq;
    put_sh(rc_settled_shift(low, range));
    if (range < kRcBot) underflow();
  }
  // Same, for lanes known to be converged (`mask`): the rare underflow loop
  // runs warp-uniformly, each lane stepping the reference loop predicated on
  // its own state, so the common path carries no divergent branch.
  __device__ __forceinline__ void encode_warp(uint32_t unit, uint32_t cum, uint32_t freq, unsigned mask) {
    low += unit * cum;
    range = unit * freq;
    put_mul(rc_settled_shift(low, range));
    if (__any_sync(mask, range < kRcBot)) {
      for (;;) {
        const uint32_t t = low + range;
        const bool differ = t < low || (low ^ t) >= kRcTop;
        const bool fix = differ && range < kRcBot;
        const bool emit = !differ || fix;
        if (!__any_sync(mask, emit)) break;
        if (fix) range = (0u - low) & (kRcBot - 1u);
        put_sh(emit ? 8u : 0u);
      }
    }
  }
  // finish (codecs.py:266-270): four bytes of low, then the partial word;
  // returns the byte count
  __device__ __forceinline__ uint32_t finish() {
    put(3);
    put(1);
    const uint32_t r = nb & 31u;
    if (r) out[nb >> 5] = __byte_perm(wlo << (32u - r), 0, 0x0123);
    return nb >> 3;
  }
};

// Decoder: input bytes come from a 64-bit window (next byte at the top of
// hi) refilled one aligned word at a time; reads are clamped to the block's
// last word and an overrun shows up as pulled > available.
struct RcDec {
  uint32_t low, range, code;
  uint32_t hi, lo;
  uint32_t avail;  // bytes in the window; >= 4 between symbols
  uint32_t wi, wlast, skip;
  uint32_t nxt;  // word wi, loaded one refill ahead so its latency is hidden
  const uint32_t* words;

  __device__ __forceinline__ uint32_t load() {
    const uint32_t w = __byte_perm(nxt, 0, 0x0123);
    ++wi;
    nxt = __ldg(words + min(wi, wlast));
    return w;
  }
  __device__ __forceinline__ void refill() {
    if (avail < 4u) {  // avail in 1..3 here
      const uint32_t w = load();
      hi |= w >> (8u * avail);
      lo = w << (32u - 8u * avail);
      avail += 4u;
    }
  }
  // block = [BE32 length][range-coded bytes]; bytes [o0, o1) of the payload
  __device__ __forceinline__ void init(const uint8_t* blk, const uint8_t* blk_end) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(blk + 4) & ~(uintptr_t)3;
    const uintptr_t last = reinterpret_cast<uintptr_t>(blk_end - 1) & ~(uintptr_t)3;
    words = reinterpret_cast<const uint32_t*>(base);
    wlast = (uint32_t)((last - base) >> 2);
    skip = (uint32_t)(reinterpret_cast<uintptr_t>(blk + 4) - base);  // 0..3
    wi = 0;
    nxt = __ldg(words);
    hi = load() << (8u * skip);
    const uint32_t w1 = load();
    if (skip == 0) {
      lo = w1;
      avail = 8u;
    } else {
      hi |= w1 >> (32u - 8u * skip);
      lo = w1 << (8u * skip);
      avail = 8u - skip;
    }
    // the first four bytes prime `code` (codecs.py:280-281)
    code = hi;
    hi = lo;
    lo = 0;
    avail -= 4u;  // 1..4
    refill();
    low = 0;
    range = 0xFFFFFFFFu;
  }
  // pull sh/8 <= 3 bytes into code (codecs.py:303-305, once per byte)
  __device__ __forceinline__ void take_sh(uint32_t sh) {
    code = (code << sh) | __funnelshift_l(hi, 0u, sh);
    hi = __funnelshift_l(lo, hi, sh);
    lo <<= sh;
    avail -= sh >> 3;
    low <<= sh;
    range <<= sh;
    refill();
  }
  __device__ __forceinline__ void take(uint32_t k) { take_sh(8u * k); }
  // take_sh with the shifts as multiplies by p = 2^sh (FMA pipe; see
  // RcEnc::put_mul): hi * p yields the shifted window word and the bytes
  // entering `code` in one IMAD.WIDE
  __device__ __forceinline__ void take_mul(uint32_t sh) {
    uint32_t p;
    asm("shl.b32 %0, 1, %1;" : "=r"(p) : "r"(sh));
    const uint64_t hw = (uint64_t)hi * p, lw = (uint64_t)lo * p;
    code = code * p + (uint32_t)(hw >> 32);
    hi = (uint32_t)hw + (uint32_t)(lw >> 32);
    lo = (uint32_t)lw;
    avail -= sh >> 3;
    low *= p;
    range *= p;
    refill();
  }
  // stream bytes consumed after the 4 priming bytes
  __device__ __forceinline__ uint32_t pulled() const { return 4u * wi - skip - 4u - avail; }
  __device__ __forceinline__ void underflow() {
    for (;;) {
      const uint32_t t = low + range;
      if (t < low || (low ^ t) >= kRcTop) {
        if (range >= kRcBot) break;
        range = (0u - low) & (kRcBot - 1u);
      }
      take(1);
    }
  }
  // code - low (codecs.py:290-292); a malformed stream with code < low reads 0
  __device__ __forceinline__ uint32_t offset() const { return code >= low ? code - low : 0u; }
  __device__ __forceinline__ void advance(uint32_t plo, uint32_t phi) {  // plo = unit*cum, phi = unit*(cum+freq)
    low += plo;
    range = phi - plo;
    take_sh(rc_settled_shift(low, range));
    if (range < kRcBot) underflow();
  }
  // converged-lane variant (see RcEnc::encode_warp)
  __device__ __forceinline__ void advance_warp(uint32_t plo, uint32_t phi, unsigned mask) {
    low += plo;
    range = phi - plo;
    take_mul(rc_settled_shift(low, range));
    if (__any_sync(mask, range < kRcBot)) {
      for (;;) {
        const uint32_t t = low + range;
        const bool differ = t < low || (low ^ t) >= kRcTop;
        const bool fix = differ && range < kRcBot;
        const bool pull = !differ || fix;
        if (!__any_sync(mask, pull)) break;
        if (fix) range = (0u - low) & (kRcBot - 1u);
        take_sh(pull ? 8u : 0u);
      }
    }
  }
};

}  // namespace kvc
