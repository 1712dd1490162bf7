// Width-stream position of a quant row (codecs.py:339-345 layout).
#pragma once
#include "kvc_internal.h"

namespace kvc {

// (width, absolute bit) of per-token quant row (lh, t): streams by descending
// width, heads (or rows) in scan order within a stream, each stream padded to
// a byte.  Head-mixed strategies use the per-head table from k_setup.
__device__ __forceinline__ void token_row_pos(const Geo& g, const HeadEntry* heads, int64_t lh, int64_t t, int& w,
                                              int64_t& bit) {
  if (g.quant == Q_UNIFORM) {
    w = g.bits;
    bit = (lh * g.T + t) * g.C * w;
  } else if (g.quant == Q_MIXTOK) {
    const int64_t k = g.k_tok, tl = g.T - k;
    if (t >= tl) {
      w = g.hi;
      bit = (lh * k + (t - tl)) * g.C * w;
    } else {
      w = g.lo;
      const int64_t lo_start = ((g.LH * k * g.C * g.hi + 7) / 8) * 8;
      bit = lo_start + (lh * tl + t) * g.C * w;
    }
  } else {
    HeadEntry e = heads[lh];
    w = e.w;
    bit = e.bit + t * g.C * w;
  }
}

}  // namespace kvc
