// Delta-transform decode for head_dim 128 (t=delta, per-token groups).
//
// invert_transform for delta is np.cumsum(y, axis=tokens, dtype=float64)
// cast to float32 (transforms.py:72): a sequential float64 running sum per
// (layer, head, channel) column.  One CTA owns one (layer, head); thread c
// owns channel c and walks the tokens in order, so the additions happen in
// exactly the reference's order (bit-exact, no tolerance).  Token tiles of
// 32 rows (packed symbols + fp16 scales/zeros) are staged through shared
// memory with coalesced loads; the next tile is prefetched into registers
// before the current tile's sequential adds and committed after them, so
// memory latency overlaps the dependent add chain.  fp32 -> fp64 uses the
// exact 2^-896 bit reinterpretation (numerics.cuh), not the slow F2F pipe.
#include <cuda_bf16.h>

#include "kernels.h"
#include "numerics.cuh"
#include "profile.h"
#include "rowpos.cuh"

namespace kvc {
namespace {

constexpr int kDT = 32;         // tokens per tile
constexpr int kDThreads = 128;  // one thread per channel
constexpr int kWPR = 32;        // words per staged row (16 * w bytes <= 128 B)
constexpr int kSymPer = kDT * kWPR / kDThreads;  // staged words per thread (8)
constexpr int kGMax = 16;       // groups per row (group >= 8)
constexpr int kSzPer = kDT * kGMax / kDThreads;  // staged scale (and zero) halves per thread (4)

// chunks per head: ~24 CTAs per SM in total (the per-channel add chains are
// latency bound, so the GPU needs many of them in flight), >= 4 tiles each
__host__ __device__ inline void delta_chunking(const Geo& g, int& nchunks, int& chunk_tiles) {
  const int ntiles = (int)((g.T + kDT - 1) / kDT);
  int64_t want = (148 * 24 + g.LH - 1) / g.LH;
  if (want < 1) want = 1;
  if (want > 256) want = 256;
  chunk_tiles = (int)((ntiles + want - 1) / want);
  if (chunk_tiles < 4) chunk_tiles = 4;
  nchunks = (ntiles + chunk_tiles - 1) / chunk_tiles;
}

inline void delta_ws_layout(const Geo& g, void* ws, double*& sum, double*& carry, uint32_t*& bad, uint32_t*& nf,
                            int& nchunks, int& chunk_tiles) {
  delta_chunking(g, nchunks, chunk_tiles);
  const int64_t n = g.LH * (int64_t)nchunks * kDThreads;
  sum = reinterpret_cast<double*>(ws);
  carry = sum + n;
  bad = reinterpret_cast<uint32_t*>(carry + n);
  nf = bad + g.LH;
}

struct Prefetch {
  uint32_t wv[kSymPer];
  unsigned short sv[kSzPer], zv[kSzPer];
  uint32_t wid;  // row width, valid for threads < nt
};

// Decode tokens [tile0*kDT, tile1*kDT) of head lh starting from the running
// sum `acc` (scaled by 2^-896); PASS 0 = full sequential decode (outputs),
// PASS 1 = chunk sum only (no outputs), PASS 3 = outputs of one chunk.
// Returns the running sum after the range.
template <typename Tout, int PASS>
__device__ double delta_range(const DecArgs& a, int64_t lh, int tile0, int tile1, double acc, uint32_t& flags) {
  __shared__ __align__(16) uint32_t sym[2][kDT][kWPR];
  __shared__ unsigned short ssc[2][kDT][kGMax], szr[2][kDT][kGMax];
  __shared__ uint32_t rw[2][kDT];
  const Geo& g = a.g;
  const int tid = threadIdx.x;
  const int G = (int)g.G;
  const unsigned short* scales = reinterpret_cast<const unsigned short*>(a.meta);
  const unsigned short* zeros = scales + g.ngroups;
  Tout* out = reinterpret_cast<Tout*>(a.out);

  auto prefetch = [&](int tile, Prefetch& pf) {
    const int t0 = tile * kDT;
    const int nt = (int)min((int64_t)kDT, g.T - t0);
#pragma unroll
    for (int k = 0; k < kSymPer; ++k) {
      const int idx = tid + kDThreads * k, r = idx / kWPR, wo = idx % kWPR;
      pf.wv[k] = 0;
      if (r < nt) {
        int w;
        int64_t bit;
        token_row_pos(g, a.heads, lh, t0 + r, w, bit);
        if (wo < 4 * w) pf.wv[k] = __ldg(reinterpret_cast<const uint32_t*>(a.packed + (bit >> 3)) + wo);
      }
    }
#pragma unroll
    for (int k = 0; k < kSzPer; ++k) {
      const int idx = tid + kDThreads * k;
      const int r = idx / kGMax, j = idx % kGMax;
      pf.sv[k] = pf.zv[k] = 0;
      if (r < nt && j < G) {
        const int64_t gi = (lh * g.T + t0 + r) * G + j;
        pf.sv[k] = __ldg(scales + gi);
        pf.zv[k] = __ldg(zeros + gi);
      }
    }
    pf.wid = 0;
    if (tid < nt) {
      int w;
      int64_t bit;
      token_row_pos(g, a.heads, lh, t0 + tid, w, bit);
      pf.wid = (uint32_t)w;
    }
  };
  auto commit = [&](const Prefetch& pf, int buf) {
#pragma unroll
    for (int k = 0; k < kSymPer; ++k) {
      const int idx = tid + kDThreads * k;
      sym[buf][idx / kWPR][idx % kWPR] = pf.wv[k];
    }
#pragma unroll
    for (int k = 0; k < kSzPer; ++k) {
      const int idx = tid + kDThreads * k;
      ssc[buf][idx / kGMax][idx % kGMax] = pf.sv[k];
      szr[buf][idx / kGMax][idx % kGMax] = pf.zv[k];
    }
    if (tid < kDT) rw[buf][tid] = pf.wid;
  };

  Prefetch pf;
  prefetch(tile0, pf);
  commit(pf, 0);
  __syncthreads();
  const int c = tid, j = c / g.group;
  for (int tile = tile0; tile < tile1; ++tile) {
    const int buf = (tile - tile0) & 1;
    if (tile + 1 < tile1) prefetch(tile + 1, pf);  // loads in flight during the adds
    const int t0 = tile * kDT;
    const int nt = (int)min((int64_t)kDT, g.T - t0);
#pragma unroll 8
    for (int r = 0; r < nt; ++r) {
      const int w = (int)rw[buf][r];
      const int p = c * w, off = p & 31;
      const uint32_t word = __byte_perm(sym[buf][r][p >> 5], 0, 0x0123);
      uint32_t s;
      if (off + w <= 32) {
        s = (word >> (32 - off - w)) & ((1u << w) - 1u);
      } else {
        const uint32_t nxt = __byte_perm(sym[buf][r][(p >> 5) + 1], 0, 0x0123);
        s = ((word << (off + w - 32)) | (nxt >> (64 - off - w))) & ((1u << w) - 1u);
      }
      const float sc = __half2float(__ushort_as_half(ssc[buf][r][j]));
      const float ze = __half2float(__ushort_as_half(szr[buf][r][j]));
      acc += f32bits_scaled_f64(__float_as_uint(dequant(s, sc, ze)));
      if (PASS != 1) {
        const float v = __double2float_rn(acc * 0x1p896);
        if (!isfinite(v)) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
        store_f32(out, out_index(a, lh, t0 + r, c), v);
      }
    }
    __syncthreads();  // buffer buf^1 (tile-1) is free and buf fully read
    if (tile + 1 < tile1) commit(pf, buf ^ 1);
    __syncthreads();
  }
  return acc;
}

// Uniform width W in {1, 2, 4, 8} (symbols never straddle a 32-bit word):
// no shared-memory staging -- thread c loads the word holding its symbol and
// its group's scale / zero straight from global memory (L1 broadcasts them
// across the threads that share them), 8 tokens per step with every load of
// the step issued before the dependent adds.
template <typename Tout, int PASS, int W>
__device__ double delta_range_u(const DecArgs& a, int64_t lh, int t_begin, int t_end, double acc, uint32_t& flags) {
  const Geo& g = a.g;
  const int c = threadIdx.x;
  const int G = (int)g.G, j = c / g.group;
  constexpr int kWordsPerRow = 4 * W;  // 128 symbols * W bits
  const int wi = (c * W) >> 5, sh = 32 - ((c * W) & 31) - W;  // MSB-first within the big-endian word
  const int64_t r0 = lh * g.T + t_begin;
  // running pointers (fixed strides per token; immediate offsets inside a step)
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(a.packed) + r0 * kWordsPerRow + wi;
  const unsigned short* sp = reinterpret_cast<const unsigned short*>(a.meta) + r0 * G + j;
  const unsigned short* zp = sp + g.ngroups;
  Tout* op = reinterpret_cast<Tout*>(a.out) + r0 * 128 + c;  // contiguous output
  const bool paged = a.paged != 0;
  auto emit = [&](int t, float v) {
    if (!isfinite(v)) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
    if (paged)
      store_f32(reinterpret_cast<Tout*>(a.out), out_index(a, lh, t, c), v);
    else
      store_f32(op, (int64_t)(t - t_begin) * 128, v);
  };
  constexpr int kU = 8;
  int t = t_begin;
  for (; t + kU <= t_end; t += kU) {
    uint32_t wv[kU];
    unsigned short sv[kU], zv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      wv[u] = __ldg(wp + u * kWordsPerRow);
      sv[u] = __ldg(sp + u * G);
      zv[u] = __ldg(zp + u * G);
    }
    wp += kU * kWordsPerRow;
    sp += kU * G;
    zp += kU * G;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t sym = (__byte_perm(wv[u], 0, 0x0123) >> sh) & ((1u << W) - 1u);
      const float y = dequant(sym, __half2float(__ushort_as_half(sv[u])), __half2float(__ushort_as_half(zv[u])));
      acc += f32bits_scaled_f64(__float_as_uint(y));
      if (PASS != 1) emit(t + u, __double2float_rn(acc * 0x1p896));
    }
  }
  for (; t < t_end; ++t) {
    const uint32_t sym = (__byte_perm(__ldg(wp), 0, 0x0123) >> sh) & ((1u << W) - 1u);
    const float y = dequant(sym, __half2float(__ushort_as_half(__ldg(sp))), __half2float(__ushort_as_half(__ldg(zp))));
    wp += kWordsPerRow;
    sp += G;
    zp += G;
    acc += f32bits_scaled_f64(__float_as_uint(y));
    if (PASS != 1) emit(t, __double2float_rn(acc * 0x1p896));
  }
  return acc;
}

// Sequential decode of whole heads (one CTA per head, thread per channel):
// the additions happen in exactly the reference's order.  `only` (optional)
// restricts it to heads whose chunked decode failed verification.
template <typename Tout>
__global__ void __launch_bounds__(kDThreads) k_dec_delta128(const DecArgs a, const uint32_t* only) {
  if (payload_rejected(a)) return;
  const int64_t lh = blockIdx.x;
  if (only && !only[lh]) return;
  uint32_t flags = 0;
  const int ntiles = (int)((a.g.T + kDT - 1) / kDT);
  delta_range<Tout, 0>(a, lh, 0, ntiles, 0.0, flags);
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// ---------------------------------------------------------- chunked decode
// The running sum is sequential in the reference (np.cumsum, float64), but
// for real KV every partial sum is exactly representable, and then a chunk
// can start from the exact prefix of the chunks before it.  Three passes:
//   1. each (head, chunk) CTA sums its chunk from 0 (the reference's order);
//   2. one thread per (head, channel) turns the chunk sums into chunk-start
//      carries (sequential over chunks);
//   3. each (head, chunk) CTA decodes its chunk from its carry with the
//      reference's additions and checks that its final running sum equals
//      the next chunk's carry.
// Pass 3 reproduces the reference bit for bit whenever the chunk's start
// value is the reference's; chunk 0 starts from 0 and every later start is
// verified against the previous chunk's exact end (induction).  A head with
// any mismatch is redone sequentially (k_dec_delta128 restricted to it), and
// its pass-3 flags are discarded.
struct DeltaWs {
  double* sum;    // [LH][nchunks][128]
  double* carry;  // [LH][nchunks][128]
  uint32_t* bad;  // [LH]
  uint32_t* nf;   // [LH] non-finite output seen in pass 3
  int nchunks, chunk_tiles;
};

template <typename Tout, int PASS>
__global__ void __launch_bounds__(kDThreads) k_delta_chunk(const DecArgs a, DeltaWs w) {
  if (payload_rejected(a)) return;
  const int64_t lh = blockIdx.x / w.nchunks;
  const int ch = (int)(blockIdx.x % w.nchunks);
  const int ntiles = (int)((a.g.T + kDT - 1) / kDT);
  const int tile0 = ch * w.chunk_tiles;
  const int tile1 = min(ntiles, tile0 + w.chunk_tiles);
  const int64_t slot = (lh * w.nchunks + ch) * kDThreads + threadIdx.x;
  uint32_t flags = 0;
  if (tile0 >= tile1) {  // empty trailing chunk
    if (PASS == 1) w.sum[slot] = 0.0;
    return;
  }
  const double start = PASS == 1 ? 0.0 : w.carry[slot];
  const int t0 = tile0 * kDT, t1 = (int)min((int64_t)tile1 * kDT, a.g.T);
  double end;
  switch (a.g.quant == Q_UNIFORM ? a.g.bits : 0) {  // uniform widths without straddling symbols
    case 1: end = delta_range_u<Tout, PASS, 1>(a, lh, t0, t1, start, flags); break;
    case 2: end = delta_range_u<Tout, PASS, 2>(a, lh, t0, t1, start, flags); break;
    case 4: end = delta_range_u<Tout, PASS, 4>(a, lh, t0, t1, start, flags); break;
    case 8: end = delta_range_u<Tout, PASS, 8>(a, lh, t0, t1, start, flags); break;
    default: end = delta_range<Tout, PASS>(a, lh, tile0, tile1, start, flags); break;
  }
  if (PASS == 1) {
    w.sum[slot] = end;
  } else {
    bool bad = ch + 1 < w.nchunks &&
               __double_as_longlong(end) != __double_as_longlong(w.carry[slot + kDThreads]);
    bad = __syncthreads_or(bad);  // used as a predicate here
    if (threadIdx.x == 0 && bad) atomicOr(&w.bad[lh], 1u);
    const bool nf = __syncthreads_or(flags != 0);
    if (threadIdx.x == 0 && nf) atomicOr(&w.nf[lh], 1u);
  }
}

__global__ void k_delta_carry(DeltaWs w, int64_t LH) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (head, channel)
  if (i >= LH * kDThreads) return;
  const int64_t lh = i / kDThreads, c = i - lh * kDThreads;
  double run = 0.0;
  for (int ch = 0; ch < w.nchunks; ++ch) {
    const int64_t slot = (lh * w.nchunks + ch) * kDThreads + c;
    w.carry[slot] = run;
    run += w.sum[slot];
  }
  if (c == 0) w.bad[lh] = 0u, w.nf[lh] = 0u;
}

// flags of the heads that passed verification
__global__ void k_delta_flags(DeltaWs w, int64_t LH, uint32_t* status) {
  const int64_t lh = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lh < LH && !w.bad[lh] && w.nf[lh]) atomicOr(status, (uint32_t)KVC_FLAG_NONFINITE_TRANSFORM);
}

template <typename Tout>
cudaError_t launch_delta(const DecArgs& a, void* ws, cudaStream_t s) {
  const Geo& g = a.g;
  const int ntiles = (int)((g.T + kDT - 1) / kDT);
  if (!ws || ntiles < 16) {  // short sequences: one pass
    k_dec_delta128<Tout><<<(unsigned)g.LH, kDThreads, 0, s>>>(a, nullptr);
    return cudaGetLastError();
  }
  DeltaWs w;
  delta_ws_layout(g, ws, w.sum, w.carry, w.bad, w.nf, w.nchunks, w.chunk_tiles);
  const unsigned grid = (unsigned)(g.LH * w.nchunks);
  k_delta_chunk<Tout, 1><<<grid, kDThreads, 0, s>>>(a, w);
  k_delta_carry<<<(unsigned)((g.LH * kDThreads + 255) / 256), 256, 0, s>>>(w, g.LH);
  k_delta_chunk<Tout, 3><<<grid, kDThreads, 0, s>>>(a, w);
  k_dec_delta128<Tout><<<(unsigned)g.LH, kDThreads, 0, s>>>(a, w.bad);
  k_delta_flags<<<(unsigned)((g.LH + 255) / 256), 256, 0, s>>>(w, g.LH, a.status);
  return cudaGetLastError();
}

}  // namespace

bool delta128_applicable(const Geo& g) {
  return g.transform == T_DELTA && !g.uchan && g.C == 128 && g.group >= 8 && 128 % g.group == 0;
}

int64_t delta128_ws_bytes(const Geo& g) {
  int nchunks, chunk_tiles;
  delta_chunking(g, nchunks, chunk_tiles);
  return (int64_t)g.LH * nchunks * kDThreads * 16 + 8 * g.LH + 64;
}

cudaError_t launch_decode_delta128(const DecArgs& a, void* ws, cudaStream_t s) {
  ProfScope ps("decode_delta128", s);
  if (a.g.out_dtype == KVC_DTYPE_BF16) return launch_delta<__nv_bfloat16>(a, ws, s);
  return launch_delta<float>(a, ws, s);
}

}  // namespace kvc
