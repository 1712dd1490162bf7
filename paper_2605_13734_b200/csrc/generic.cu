// Shape-generic codec kernels: every strategy on every valid shape.
//
// These are the correctness backbone (any L,H,T,C; any group; C not a
// multiple of 8; per-channel groups; every transform).  The head_dim-128
// per-token hot path has its own fused kernels (fast128.cu); both produce the
// same bytes.  Layout of the work: one CTA per tile of TT tokens x C channels
// of one (layer, head); the tile is staged in shared memory as fp32.
#include <cuda_bf16.h>

#include "kernels.h"
#include "numerics.cuh"
#include "profile.h"
#include "rowpos.cuh"

namespace kvc {

// ------------------------------------------------------------------ setup
// Derive the width-stream table and per-head entries from the class map
// stored in the metadata (codecs.py:339-345 stream order; quantize.py:115-123).
__global__ void k_setup(Geo g, const uint8_t* meta, StreamTab* st, HeadEntry* heads) {
  __shared__ int64_t s_nhi;
  const bool head_mixed = (g.quant == Q_MIXED || g.quant == Q_MIXLAYER);
  const uint8_t* cmap = head_mixed ? meta + g.meta_class_off : nullptr;
  if (threadIdx.x == 0) {
    int64_t nhi = 0;
    if (head_mixed)
      for (int64_t i = 0; i < g.LH; ++i) nhi += (cmap[i >> 3] >> (7 - (i & 7))) & 1;
    s_nhi = nhi;
  }
  __syncthreads();
  const int64_t per_head = g.T * g.C;
  if (threadIdx.x == 0) {
    StreamTab t;
    int64_t cnt[2];
    int w[2];
    int n = 0;
    if (g.quant == Q_UNIFORM || g.quant == Q_UCHAN) {
      w[0] = g.bits; cnt[0] = g.E; n = 1;
    } else {
      int64_t hi_cnt = head_mixed ? s_nhi * per_head : g.LH * g.k_tok * g.C;
      int64_t lo_cnt = g.E - hi_cnt;
      if (hi_cnt > 0) { w[n] = g.hi; cnt[n] = hi_cnt; ++n; }
      if (lo_cnt > 0) { w[n] = g.lo; cnt[n] = lo_cnt; ++n; }
    }
    t.n = n;
    int64_t off = 0, blk = 0;
    for (int i = 0; i < kMaxStreams; ++i) {
      if (i < n) {
        t.w[i] = w[i]; t.count[i] = cnt[i]; t.byte_off[i] = off; t.first_block[i] = blk;
        off += (cnt[i] * w[i] + 7) / 8;
        blk += (g.codec == C_NONE) ? 0 : (cnt[i] + g.block - 1) / g.block;
      } else {
        t.w[i] = 0; t.count[i] = 0; t.byte_off[i] = off; t.first_block[i] = blk;
      }
    }
    if (g.rle_whole) {  // one rle block over all streams (the reference's whole-tensor format)
      for (int i = 0; i < kMaxStreams; ++i) t.first_block[i] = 0;
      blk = off > 0 ? 1 : 0;
    }
    t.nblocks = blk;
    t.packed_bytes = off;
    *st = t;
  }
  if (head_mixed) {
    // per-head bit offsets: rank among heads of the same class (warp 0 scans)
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int64_t hi_before = 0, lo_before = 0;
      const int64_t lo_start = ((s_nhi * per_head * g.hi + 7) / 8) * 8;
      for (int64_t base = 0; base < g.LH; base += 32) {
        int64_t i = base + lane;
        int is_hi = (i < g.LH) ? ((cmap[i >> 3] >> (7 - (i & 7))) & 1) : 0;
        int valid = i < g.LH;
        unsigned bal = __ballot_sync(0xffffffffu, is_hi && valid);
        unsigned val = __ballot_sync(0xffffffffu, valid);
        unsigned below = (1u << lane) - 1u;
        int64_t r_hi = hi_before + __popc(bal & below);
        int64_t r_lo = lo_before + __popc(val & ~bal & below);
        if (valid) {
          HeadEntry e;
          e.w = is_hi ? g.hi : g.lo;
          e.bit = is_hi ? r_hi * per_head * g.hi : lo_start + r_lo * per_head * g.lo;
          e.pad = 0;
          heads[i] = e;
        }
        hi_before += __popc(bal);
        lo_before += __popc(val & ~bal);
      }
    }
  }
}

// class map bits (passed by value) -> metadata
__global__ void k_write_classmap(ClassBits cb, uint8_t* dst, int nbytes) {
  for (int i = threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = cb.b[i];
}

// ------------------------------------------------------- affine calibration
// mu = f16(0.5*(max+min)), a = f16(min(2/(max-min), 65504)) over the first
// min(T,128) tokens of each (layer, head, channel).  DESIGN.md §3 (extension).
template <typename Tin>
__global__ void k_affine_calibrate(const EncArgs a) {
  const Geo& g = a.g;
  const Tin* kv = reinterpret_cast<const Tin*>(a.kv);
  uint8_t* meta = a.meta;
  const int64_t lh = blockIdx.x;
  const int64_t nt = g.T < kAffinePrefix ? g.T : kAffinePrefix;
  uint8_t* aff = meta + g.meta_affine_off;  // mu16[LH*C] || a16[LH*C]
  for (int64_t c = threadIdx.x; c < g.C; c += blockDim.x) {
    float mx = -INFINITY, mn = INFINITY;
    for (int64_t t = 0; t < nt; ++t) {
      float v = load_f32(kv, out_index(a, lh, t, c));
      mx = fmaxf(mx, v);
      mn = fminf(mn, v);
    }
    float m = __fmul_rn(0.5f, __fadd_rn(mx, mn));
    float r = __fsub_rn(mx, mn);
    float s = r > 0.0f ? __fdiv_rn(2.0f, r) : 1.0f;
    s = fminf(s, 65504.0f);
    st_meta_half(aff, lh * g.C + c, m);
    st_meta_half(aff, g.LH * g.C + lh * g.C + c, s);
  }
}

__device__ __forceinline__ int64_t meta_group_index(const Geo& g, int64_t lh, int64_t t, int64_t c) {
  // scale/zero index of element (lh, t, c)
  if (g.uchan) return (lh * g.C + c) * g.G + t / g.group;
  return (lh * g.T + t) * g.G + c / g.group;
}

// write `n` symbols of width w starting at absolute bit `bit`; byte-producer
// when aligned, atomicOr (payload pre-zeroed) otherwise.
__device__ void pack_segment(uint8_t* out, int64_t bit, const uint8_t* s, int64_t stride, int64_t n, int w,
                             int tid, int nthr) {
  const int64_t nbits = n * w;
  if ((bit & 7) == 0 && (nbits & 7) == 0) {
    uint8_t* o = out + (bit >> 3);
    for (int64_t jb = tid; jb < (nbits >> 3); jb += nthr) {
      uint32_t v = 0;
      for (int k = 0; k < 8; ++k) {
        int64_t p = jb * 8 + k;
        int64_t i = p / w;
        int sb = w - 1 - (int)(p - i * w);
        v |= ((uint32_t)(s[i * stride] >> sb) & 1u) << (7 - k);
      }
      o[jb] = (uint8_t)v;
    }
  } else {
    unsigned int* words = reinterpret_cast<unsigned int*>(out);
    for (int64_t i = tid; i < n; i += nthr) {
      uint32_t sym = s[i * stride];
      for (int k = 0; k < w; ++k) {
        if (!((sym >> (w - 1 - k)) & 1u)) continue;
        int64_t p = bit + i * w + k;
        int64_t byte = p >> 3;
        int sh = (int)((byte & 3) * 8 + (7 - (p & 7)));
        atomicOr(words + (byte >> 2), 1u << sh);
      }
    }
  }
}

// ------------------------------------------------------------ generic encode
// one tile of TT token rows (lh, t0 .. t0+nt-1), all of it in shared memory
template <typename Tin>
__device__ void encode_tile(const EncArgs& a, int TT, int64_t lh, int64_t t0, int nt, unsigned char* smem) {
  const Geo& g = a.g;
  const int64_t C = g.C, T = g.T;
  float* y = reinterpret_cast<float*>(smem);  // [TT][C]
  float* prev = y + (int64_t)TT * C;          // [C]
  uint8_t* sym = reinterpret_cast<uint8_t*>(prev + C);  // quant-ordered symbols
  double* fw = reinterpret_cast<double*>(smem + (((int64_t)TT * C * 5 + C * 4 + 15) & ~15ll));
  const Tin* kv = reinterpret_cast<const Tin*>(a.kv);
  const Tin* src = kv + (lh * T + t0) * C;
  uint32_t flags = 0;

  float nanacc = 0.0f;
  if (!a.paged) {
    for (int64_t i = threadIdx.x; i < (int64_t)nt * C; i += blockDim.x) {
      float v = load_f32(src, i);
      nanacc = __fmaf_rn(v, 0.0f, nanacc);
      y[i] = v;
    }
  } else {  // paged input: each token row from its page
    for (int64_t i = threadIdx.x; i < (int64_t)nt * C; i += blockDim.x) {
      const int64_t tr = i / C;
      float v = load_f32(kv, out_index(a, lh, t0 + tr, i - tr * C));
      nanacc = __fmaf_rn(v, 0.0f, nanacc);
      y[i] = v;
    }
  }
  if (nanacc != 0.0f) flags |= KVC_FLAG_NONFINITE_INPUT;
  if (g.transform == T_DELTA && t0 > 0)
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) prev[c] = load_f32(kv, out_index(a, lh, t0 - 1, c));
  __syncthreads();

  // ---- transform (transforms.py:50-64; affine: extension)
  if (g.transform == T_DELTA) {
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
      for (int t = nt - 1; t >= 1; --t) y[t * C + c] = __fsub_rn(y[t * C + c], y[(t - 1) * C + c]);
      if (t0 > 0) y[c] = __fsub_rn(y[c], prev[c]);
    }
  } else if (g.transform == T_HADAMARD) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* f = fw + warp * C;
    for (int t = warp; t < nt; t += nw) {
      for (int64_t c = lane; c < C; c += 32) f[c] = f32bits_scaled_f64(__float_as_uint(y[t * C + c]));
      __syncwarp();
      for (int64_t h = 1; h < C; h <<= 1) {
        for (int64_t p = lane; p < C / 2; p += 32) {
          int64_t j = p / h, i = p - j * h;
          int64_t ia = j * 2 * h + i, ib = ia + h;
          double u = f[ia], v = f[ib];
          f[ia] = u + v;
          f[ib] = u - v;
        }
        __syncwarp();
      }
      for (int64_t c = lane; c < C; c += 32) y[t * C + c] = hadamard_out(f[c], a.hk, a.hc, flags);
      __syncwarp();
    }
  } else if (g.transform == T_AFFINE) {
    const uint8_t* aff = a.meta + g.meta_affine_off;
    for (int64_t i = threadIdx.x; i < (int64_t)nt * C; i += blockDim.x) {
      int64_t c = i % C;
      float v = __fmul_rn(__fsub_rn(y[i], ld_meta_half(aff, lh * C + c)), ld_meta_half(aff, (g.LH + lh) * C + c));
      if (!isfinite(v)) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
      y[i] = v;
    }
  }
  __syncthreads();

  // ---- quantize (quantize.py:126-164)
  __half* scales = reinterpret_cast<__half*>(a.meta);
  __half* zeros = scales + g.ngroups;
  if (!g.uchan) {
    const int64_t ngr = (int64_t)nt * g.G;
    for (int64_t q = threadIdx.x; q < ngr; q += blockDim.x) {
      const int t = (int)(q / g.G);
      const int64_t j = q - (int64_t)t * g.G;
      int w;
      int64_t bitdummy;
      token_row_pos(g, a.heads, lh, t0 + t, w, bitdummy);
      const float* yy = y + t * C + j * g.group;
      float mn = yy[0], mx = yy[0];
      for (int i = 1; i < g.group; ++i) { mn = fminf(mn, yy[i]); mx = fmaxf(mx, yy[i]); }
      __half s16, z16;
      GroupQ gq = group_setup(mn, mx, w, a.rl[w], s16, z16, flags);
      const int64_t gi = (lh * T + t0 + t) * g.G + j;
      scales[gi] = s16;
      zeros[gi] = z16;
      uint8_t* so = sym + t * C + j * g.group;
      for (int i = 0; i < g.group; ++i) so[i] = (uint8_t)quant_one(yy[i], gq);
    }
  } else {
    const int64_t gt = nt / g.group;  // tiles are group aligned
    const int64_t ngr = C * gt;
    for (int64_t q = threadIdx.x; q < ngr; q += blockDim.x) {
      const int64_t c = q % C;
      const int64_t jt = q / C;
      const float* yy = y + jt * g.group * C + c;
      float mn = yy[0], mx = yy[0];
      for (int i = 1; i < g.group; ++i) { mn = fminf(mn, yy[i * C]); mx = fmaxf(mx, yy[i * C]); }
      __half s16, z16;
      GroupQ gq = group_setup(mn, mx, g.bits, a.rl[g.bits], s16, z16, flags);
      const int64_t gi = (lh * C + c) * g.G + t0 / g.group + jt;
      scales[gi] = s16;
      zeros[gi] = z16;
      uint8_t* so = sym + c * TT + jt * g.group;
      for (int i = 0; i < g.group; ++i) so[i] = (uint8_t)quant_one(yy[i * C], gq);
    }
  }
  __syncthreads();

  // ---- pack into the width streams (codecs.py:79-87, :339-345, :359)
  if (!g.uchan) {
    // one warp per token row
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int t = warp; t < nt; t += nw) {
      int w;
      int64_t bit;
      token_row_pos(g, a.heads, lh, t0 + t, w, bit);
      pack_segment(a.packed, bit, sym + t * C, 1, C, w, lane, 32);
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int64_t c = warp; c < C; c += nw) {
      const int64_t bit = ((lh * C + c) * T + t0) * g.bits;
      pack_segment(a.packed, bit, sym + c * TT, 1, nt, g.bits, lane, 32);
    }
  }
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

template <typename Tin>
__global__ void __launch_bounds__(256) k_encode_generic(EncArgs a, int TT) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t tiles = (a.g.T + TT - 1) / TT;
  const int64_t lh = blockIdx.x / tiles;
  const int64_t t0 = (blockIdx.x % tiles) * TT;
  encode_tile<Tin>(a, TT, lh, t0, (int)min((int64_t)TT, a.g.T - t0), smem);
}

// Exact re-encode of the token rows the fused Hadamard encode listed (rows
// whose fast rounding it could not prove exact, fast128.cu): each CTA takes
// list entries in turn and overwrites the row's bytes, scales and zeros.  The
// count is read on the device, so the launch never waits on the host.
template <typename Tin>
__global__ void __launch_bounds__(256) k_encode_fixup(EncArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t n = *a.fix_count;
  for (uint32_t e = blockIdx.x; e < n; e += gridDim.x) {
    const int64_t row = a.fix_rows[e];
    const int64_t lh = row / a.g.T;
    encode_tile<Tin>(a, 1, lh, row - lh * a.g.T, 1, smem);
    __syncthreads();
  }
}

// ------------------------------------------------------------ generic decode
template <typename Tout>
__global__ void __launch_bounds__(256) k_decode_generic(DecArgs a, int TT) {
  if (payload_rejected(a)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const Geo& g = a.g;
  const int64_t C = g.C, T = g.T;
  const int64_t tiles = (T + TT - 1) / TT;
  const int64_t lh = blockIdx.x / tiles;
  const int64_t t0 = (blockIdx.x % tiles) * TT;
  const int nt = (int)min((int64_t)TT, T - t0);
  float* y = reinterpret_cast<float*>(smem);
  double* fw = reinterpret_cast<double*>(smem + (((int64_t)TT * C * 4 + 15) & ~15ll));
  const __half* scales = reinterpret_cast<const __half*>(a.meta);
  const __half* zeros = scales + g.ngroups;
  uint32_t flags = 0;

  for (int64_t i = threadIdx.x; i < (int64_t)nt * C; i += blockDim.x) {
    const int t = (int)(i / C);
    const int64_t c = i - (int64_t)t * C;
    int w;
    int64_t bit;
    if (g.uchan) {
      w = g.bits;
      bit = ((lh * C + c) * T + t0 + t) * w;
    } else {
      token_row_pos(g, a.heads, lh, t0 + t, w, bit);
      bit += c * w;
    }
    uint32_t s = read_sym(a.packed, bit, w);
    int64_t gi = meta_group_index(g, lh, t0 + t, c);
    y[i] = dequant(s, __half2float(scales[gi]), __half2float(zeros[gi]));
  }
  __syncthreads();
  if (g.transform == T_HADAMARD) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* f = fw + warp * C;
    for (int t = warp; t < nt; t += nw) {
      for (int64_t c = lane; c < C; c += 32) f[c] = f32bits_scaled_f64(__float_as_uint(y[t * C + c]));
      __syncwarp();
      for (int64_t h = 1; h < C; h <<= 1) {
        for (int64_t p = lane; p < C / 2; p += 32) {
          int64_t j = p / h, i = p - j * h;
          int64_t ia = j * 2 * h + i, ib = ia + h;
          double u = f[ia], v = f[ib];
          f[ia] = u + v;
          f[ib] = u - v;
        }
        __syncwarp();
      }
      for (int64_t c = lane; c < C; c += 32) y[t * C + c] = hadamard_out(f[c], a.hk, a.hc, flags);
      __syncwarp();
    }
    __syncthreads();
  } else if (g.transform == T_AFFINE) {
    const uint8_t* aff = a.meta + g.meta_affine_off;
    for (int64_t i = threadIdx.x; i < (int64_t)nt * C; i += blockDim.x) {
      int64_t c = i % C;
      y[i] = __fadd_rn(__fdiv_rn(y[i], ld_meta_half(aff, (g.LH + lh) * C + c)), ld_meta_half(aff, lh * C + c));
    }
    __syncthreads();
  }
  Tout* out = reinterpret_cast<Tout*>(a.out);
  for (int64_t i = threadIdx.x; i < (int64_t)nt * C; i += blockDim.x) {
    const int t = (int)(i / C);
    const int64_t c = i - (int64_t)t * C;
    float v = y[i];
    if (!isfinite(v)) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
    store_f32(out, out_index(a, lh, t0 + t, c), v);
  }
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// delta decode: fp64 running sum along tokens per (head, channel) column,
// in token order exactly like np.cumsum(dtype=float64) (transforms.py:72).
template <typename Tout>
__global__ void __launch_bounds__(128) k_decode_delta(DecArgs a) {
  if (payload_rejected(a)) return;
  const Geo& g = a.g;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= g.LH * g.C) return;
  const int64_t lh = col / g.C, c = col - lh * g.C;
  const __half* scales = reinterpret_cast<const __half*>(a.meta);
  const __half* zeros = scales + g.ngroups;
  Tout* out = reinterpret_cast<Tout*>(a.out);
  double acc = 0.0;
  uint32_t flags = 0;
  for (int64_t t = 0; t < g.T; ++t) {
    int w;
    int64_t bit;
    if (g.uchan) {
      w = g.bits;
      bit = ((lh * g.C + c) * g.T + t) * w;
    } else {
      token_row_pos(g, a.heads, lh, t, w, bit);
      bit += c * w;
    }
    uint32_t s = read_sym(a.packed, bit, w);
    int64_t gi = meta_group_index(g, lh, t, c);
    acc += (double)dequant(s, __half2float(scales[gi]), __half2float(zeros[gi]));
    float v = __double2float_rn(acc);
    if (!isfinite(v)) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
    store_f32(out, out_index(a, lh, t, c), v);
  }
  if (flags) atomicOr(a.status, flags);
}

// ------------------------------------------------------------ host launchers
int generic_tile_tokens(const Geo& g) {
  int64_t tt;
  if (g.uchan) {
    tt = g.group;
    while (tt * 2 * g.C <= 8192 && (g.T % (tt * 2)) == 0) tt *= 2;
  } else {
    tt = 8192 / g.C;
    if (tt < 1) tt = 1;
    if (tt > g.T) tt = g.T;
    if (tt >= 8) tt &= ~7ll;
  }
  return (int)tt;
}

size_t generic_encode_smem(const Geo& g, int TT) {
  size_t base = (((size_t)TT * g.C * 5 + g.C * 4 + 15) & ~(size_t)15);
  if (g.transform == T_HADAMARD) base += 8 * g.C * 8;
  return base;
}

size_t generic_decode_smem(const Geo& g, int TT) {
  size_t base = (((size_t)TT * g.C * 4 + 15) & ~(size_t)15);
  if (g.transform == T_HADAMARD) base += 8 * g.C * 8;
  return base;
}

cudaError_t launch_encode_generic(const EncArgs& a, cudaStream_t s) {
  const Geo& g = a.g;
  int TT = generic_tile_tokens(g);
  size_t sm = generic_encode_smem(g, TT);
  int64_t tiles = g.LH * ((g.T + TT - 1) / TT);
  ProfScope ps("encode_generic", s);
  if (g.in_dtype == KVC_DTYPE_BF16) {
    cudaFuncSetAttribute(k_encode_generic<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_encode_generic<__nv_bfloat16><<<(unsigned)tiles, 256, sm, s>>>(a, TT);
  } else {
    cudaFuncSetAttribute(k_encode_generic<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_encode_generic<float><<<(unsigned)tiles, 256, sm, s>>>(a, TT);
  }
  return cudaGetLastError();
}

cudaError_t launch_encode_fixup(const EncArgs& a, cudaStream_t s) {
  const size_t sm = generic_encode_smem(a.g, 1);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  ProfScope ps("encode_fixup", s);
  if (a.g.in_dtype == KVC_DTYPE_BF16) {
    cudaFuncSetAttribute(k_encode_fixup<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_encode_fixup<__nv_bfloat16><<<(unsigned)(2 * sms), 256, sm, s>>>(a);
  } else {
    cudaFuncSetAttribute(k_encode_fixup<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_encode_fixup<float><<<(unsigned)(2 * sms), 256, sm, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_decode_generic(const DecArgs& a, cudaStream_t s) {
  const Geo& g = a.g;
  if (g.transform == T_DELTA) {
    int64_t cols = g.LH * g.C;
    unsigned blocks = (unsigned)((cols + 127) / 128);
    ProfScope ps("decode_delta", s);
    if (g.out_dtype == KVC_DTYPE_BF16)
      k_decode_delta<__nv_bfloat16><<<blocks, 128, 0, s>>>(a);
    else
      k_decode_delta<float><<<blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
  }
  int TT = generic_tile_tokens(g);
  size_t sm = generic_decode_smem(g, TT);
  int64_t tiles = g.LH * ((g.T + TT - 1) / TT);
  ProfScope ps("decode_generic", s);
  if (g.out_dtype == KVC_DTYPE_BF16) {
    cudaFuncSetAttribute(k_decode_generic<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_decode_generic<__nv_bfloat16><<<(unsigned)tiles, 256, sm, s>>>(a, TT);
  } else {
    cudaFuncSetAttribute(k_decode_generic<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_decode_generic<float><<<(unsigned)tiles, 256, sm, s>>>(a, TT);
  }
  return cudaGetLastError();
}

cudaError_t launch_setup(const Geo& g, const uint8_t* meta, StreamTab* st, HeadEntry* heads, cudaStream_t s) {
  ProfScope ps("setup", s);
  k_setup<<<1, 32, 0, s>>>(g, meta, st, heads);
  return cudaGetLastError();
}

cudaError_t launch_write_classmap(const ClassBits& cb, uint8_t* dst, int nbytes, cudaStream_t s) {
  ProfScope ps("classmap", s);
  k_write_classmap<<<1, 256, 0, s>>>(cb, dst, nbytes);
  return cudaGetLastError();
}

cudaError_t launch_affine_calibrate(const EncArgs& a, cudaStream_t s) {
  const Geo& g = a.g;
  unsigned thr = (unsigned)(g.C < 256 ? ((g.C + 31) / 32) * 32 : 256);
  ProfScope ps("affine_calibrate", s);
  if (g.in_dtype == KVC_DTYPE_BF16)
    k_affine_calibrate<__nv_bfloat16><<<(unsigned)g.LH, thr, 0, s>>>(a);
  else
    k_affine_calibrate<float><<<(unsigned)g.LH, thr, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace kvc
