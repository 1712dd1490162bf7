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
//
// The carry test is implicit.  Every reachable state has low + range <= 2^32
// (true initially; an encode step stays inside the interval; a settled shift
// leaves low + range < 2^32; the underflow fix rounds low + range up to a
// multiple of 2^16).  So a carry means low + range == 2^32 exactly, i.e. t = 0
// and x = low ^ t = low; that state is only entered through the underflow
// loop, which leaves range < 2^24, so low > 2^32 - 2^24 has a set top bit and
// clz(x) = 0: no bytes settle, as the reference decides.  (x = 0 would need
// range = 0, which the underflow fix cannot produce: it only runs when the
// interval crosses a multiple of 2^24, so low is not a multiple of 2^16.)
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
// compiler would otherwise branch around the bit scan; no carry select, see
// above)
__device__ __forceinline__ uint32_t rc_settled_shift(uint32_t low, uint32_t range) {
  uint32_t sh;
  asm("{\n\t.reg .u32 t, x, c;\n\t"
      "add.u32 t, %1, %2;\n\txor.b32 x, %1, t;\n\tbfind.shiftamt.u32 c, x;\n\tand.b32 %0, c, 24;\n\t}"
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
    asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(p) : "r"(sh));  // 2^sh in one instruction; opaque: keep the multiplies
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

// Decoder.  `code` is always the four stream bytes after the ones consumed
// (codecs.py:280-281, 303-305 shift one byte in per step), so it is not kept:
// it is read out of two cached big-endian stream words w0:w1 at bit offset
// pos (one funnel shift), and consuming bytes only advances pos.  When pos
// passes a word boundary the words rotate and the next word (prefetched one
// rotation ahead) comes in.  Reads are clamped to the block's last word; an
// overrun shows up as pulled() > available.
struct RcDec {
  uint32_t low, range;
  uint32_t w0, w1;  // stream words wi-2, wi-1 (big-endian values)
  uint32_t nxt;     // raw word wi, loaded one rotation ahead
  uint32_t pos;     // bit offset of code's first byte in w0: 0..31 between steps
  uint32_t wi, wlast, skip;
  const uint32_t* words;

  __device__ __forceinline__ uint32_t code() const { return __funnelshift_l(w1, w0, pos); }
  __device__ __forceinline__ void rotate() {  // at most one per step: pos < 32 + 24
    if (pos >= 32u) {
      w0 = w1;
      w1 = __byte_perm(nxt, 0, 0x0123);
      ++wi;
      nxt = __ldg(words + min(wi, wlast));
      pos -= 32u;
    }
  }
  // block = [BE32 length][range-coded bytes]; bytes [o0, o1) of the payload
  __device__ __forceinline__ void init(const uint8_t* blk, const uint8_t* blk_end) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(blk + 4) & ~(uintptr_t)3;
    const uintptr_t last = reinterpret_cast<uintptr_t>(blk_end - 1) & ~(uintptr_t)3;
    words = reinterpret_cast<const uint32_t*>(base);
    wlast = (uint32_t)((last - base) >> 2);
    skip = (uint32_t)(reinterpret_cast<uintptr_t>(blk + 4) - base);  // 0..3
    w0 = __byte_perm(__ldg(words), 0, 0x0123);
    w1 = __byte_perm(__ldg(words + min(1u, wlast)), 0, 0x0123);
    nxt = __ldg(words + min(2u, wlast));
    wi = 2;
    pos = 8u * skip;  // the first four bytes prime code
    low = 0;
    range = 0xFFFFFFFFu;
  }
  // consume sh/8 <= 3 bytes (codecs.py:303-305, once per byte)
  __device__ __forceinline__ void take_sh(uint32_t sh) {
    pos += sh;
    rotate();
    low <<= sh;
    range <<= sh;
  }
  __device__ __forceinline__ void take(uint32_t k) { take_sh(8u * k); }
  // take_sh with the low / range shifts as multiplies by p = 2^sh (FMA pipe)
  __device__ __forceinline__ void take_mul(uint32_t sh) {
    uint32_t p;
    asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(p) : "r"(sh));  // 2^sh
    low *= p;
    range *= p;
    pos += sh;
    rotate();
  }
  // stream bytes consumed after the 4 priming bytes
  __device__ __forceinline__ uint32_t pulled() const { return 4u * (wi - 2u) + (pos >> 3) - skip; }
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
  __device__ __forceinline__ uint32_t offset() const {
    const uint32_t c = code();
    return c >= low ? c - low : 0u;
  }
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
