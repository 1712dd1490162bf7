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

struct Prefetch {
  uint32_t wv[kSymPer];
  unsigned short sv[kSzPer], zv[kSzPer];
  uint32_t wid;  // row width, valid for threads < nt
};

template <typename Tout>
__global__ void __launch_bounds__(kDThreads) k_dec_delta128(const DecArgs a) {
  __shared__ __align__(16) uint32_t sym[2][kDT][kWPR];
  __shared__ unsigned short ssc[2][kDT][kGMax], szr[2][kDT][kGMax];
  __shared__ uint32_t rw[2][kDT];
  const Geo& g = a.g;
  const int64_t lh = blockIdx.x;
  const int tid = threadIdx.x;
  const int G = (int)g.G;
  const unsigned short* scales = reinterpret_cast<const unsigned short*>(a.meta);
  const unsigned short* zeros = scales + g.ngroups;
  const int ntiles = (int)((g.T + kDT - 1) / kDT);
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

  double acc = 0.0;  // running sum * 2^-896 (exact scaling)
  uint32_t flags = 0;
  Prefetch pf;
  prefetch(0, pf);
  commit(pf, 0);
  __syncthreads();
  const int c = tid, j = c / g.group;
  for (int tile = 0; tile < ntiles; ++tile) {
    const int buf = tile & 1;
    if (tile + 1 < ntiles) prefetch(tile + 1, pf);  // loads in flight during the adds
    const int t0 = tile * kDT;
    const int nt = (int)min((int64_t)kDT, g.T - t0);
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
      const float v = __double2float_rn(acc * 0x1p896);
      if (!isfinite(v)) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
      store_f32(out, out_index(a, lh, t0 + r, c), v);
    }
    __syncthreads();  // buffer buf^1 (tile-1) is free and buf fully read
    if (tile + 1 < ntiles) commit(pf, buf ^ 1);
    __syncthreads();
  }
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

}  // namespace

bool delta128_applicable(const Geo& g) {
  return g.transform == T_DELTA && !g.uchan && g.C == 128 && g.group >= 8 && 128 % g.group == 0;
}

cudaError_t launch_decode_delta128(const DecArgs& a, cudaStream_t s) {
  ProfScope ps("decode_delta128", s);
  if (a.g.out_dtype == KVC_DTYPE_BF16)
    k_dec_delta128<__nv_bfloat16><<<(unsigned)a.g.LH, kDThreads, 0, s>>>(a);
  else
    k_dec_delta128<float><<<(unsigned)a.g.LH, kDThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace kvc
