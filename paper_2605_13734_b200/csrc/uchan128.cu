// Per-channel (KIVI-K, q=uchan) kernels for head_dim 128, groups of 32 tokens.
//
// Quant layout = the reference quantizer applied to the (L,H,C,T) transpose
// (DESIGN.md §3): symbols of channel c run along tokens, scales are
// (L,H,C,T/32).  A CTA owns a block of 128 tokens x 128 channels of one head
// (32 KB bf16) loaded by TMA into a 2-deep ring; warp k quantizes token group
// k (32 tokens) for all 128 channels (4 channels per lane), then the packed
// groups are regrouped through shared memory so every channel's 4 groups leave
// as one contiguous 16*w-byte run (full 32 B sectors at w = 2).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <mutex>

#include "kernels.h"
#include "numerics.cuh"
#include "profile.h"

namespace kvc {
namespace {

constexpr int kUT = 128;                        // tokens per block
constexpr int kUThreads = 128;                  // 4 warps
constexpr int kUStages = 2;
constexpr int kUTileBytes = kUT * 128 * 2;      // 32 KB
// ring + symbol staging [128 ch][4 groups][8 words] + scale/zero staging + align + barriers
constexpr int kUSmem = kUStages * kUTileBytes + 128 * 4 * 8 * 4 + 128 * 8 * 2 + 1024 + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// pack 32 symbols of width W (low byte of magic floats), MSB-first, into W words (LE bytes)
template <int W>
__device__ __forceinline__ void pack32_words(const float* q, uint32_t* wd) {
  uint32_t be[W];
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
#pragma unroll
  for (int k = 0; k < W; ++k) wd[k] = __byte_perm(be[k], 0, 0x0123);
}

template <int W>
__device__ __forceinline__ void unpack32_words(const uint32_t* wd, float* v) {
  uint32_t be[W];
#pragma unroll
  for (int k = 0; k < W; ++k) be[k] = __byte_perm(wd[k], 0, 0x0123);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int p = i * W, k = p >> 5, off = p & 31;
    uint32_t s;
    if (off + W <= 32) s = (be[k] >> (32 - off - W)) & ((1u << W) - 1u);
    else s = ((be[k] << (off + W - 32)) | (be[k + 1] >> (64 - off - W))) & ((1u << W) - 1u);
    v[i] = __uint_as_float(0x4B000000u | s) - 8388608.0f;
  }
}

// ------------------------------------------------------------------ encode
template <int W, bool AFFINE>
__global__ void __launch_bounds__(kUThreads, 3) k_enc_uchan128(const __grid_constant__ CUtensorMap tmap, const EncArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned (128B swizzle atoms), indexed off smem_raw so the compiler keeps the
  // shared address space (LDS / STS rather than generic loads)
  uint8_t* tiles = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint32_t* stage_sym = reinterpret_cast<uint32_t*>(tiles + kUStages * kUTileBytes);  // [128 ch][4 groups][W words]
  uint16_t* stage_sz = reinterpret_cast<uint16_t*>(stage_sym + 128 * 4 * 8);          // [128 ch][4][2] scale, zero
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_sz + 128 * 8);
  const Geo& g = a.g;
  const int64_t blocks_per_head = g.T / kUT;
  const int64_t nblocks = g.LH * blocks_per_head;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kUStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kUStages; ++s) {
      const int64_t b = blockIdx.x + (int64_t)s * gridDim.x;
      if (b < nblocks) {
        mbar_expect_tx(&full[s], kUTileBytes);
        tma_load_2d(tiles + s * kUTileBytes, &tmap, 0, (int)(b * kUT), &full[s]);
      }
    }
  }
  __half* scales = reinterpret_cast<__half*>(a.meta);
  __half* zeros = scales + g.ngroups;
  const float rl = a.rl[W];
  uint32_t flags = 0;
  float nanacc = 0.0f;
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const int s = it % kUStages;
    mbar_wait(&full[s], (uint32_t)((it / kUStages) & 1));
    const int64_t lh = b / blocks_per_head;
    const int64_t t0 = (b - lh * blocks_per_head) * kUT;
    const uint8_t* tb = tiles + s * kUTileBytes;
    // lane: channels 4*lane .. 4*lane+3, tokens 32*warp .. +31
    uint2 v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = *reinterpret_cast<const uint2*>(tb + (32 * warp + i) * 256 + lane * 8);
    __syncthreads();  // slot s consumed by every warp
    if (tid == 0) {
      const int64_t nb = b + (int64_t)kUStages * gridDim.x;
      if (nb < nblocks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s], kUTileBytes);
        tma_load_2d(tiles + s * kUTileBytes, &tmap, 0, (int)(nb * kUT), &full[s]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 4 * lane + j;
      float y[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t word = (j < 2) ? v[i].x : v[i].y;
        y[i] = __uint_as_float((j & 1) ? (word & 0xFFFF0000u) : (word << 16));
        nanacc = __fmaf_rn(y[i], 0.0f, nanacc);
      }
      if (AFFINE) {
        const __half* mu = reinterpret_cast<const __half*>(a.meta + g.meta_affine_off);
        const float m = __half2float(mu[lh * 128 + c]), sc = __half2float(mu[g.LH * 128 + lh * 128 + c]);
        float chk = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          y[i] = __fmul_rn(__fsub_rn(y[i], m), sc);
          chk = __fmaf_rn(y[i], 0.0f, chk);
        }
        if (chk != 0.0f) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
      }
      float mn = y[0], mx = y[0];
#pragma unroll
      for (int i = 1; i < 32; ++i) {
        mn = fminf(mn, y[i]);
        mx = fmaxf(mx, y[i]);
      }
      __half s16, z16;
      GroupQ q = group_setup(mn, mx, W, rl, s16, z16, flags);
      if (q.mode == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) y[i] = quant_magic(y[i], q);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) y[i] = __uint_as_float(kMagicBits + quant_one(y[i], q));
      }
      uint32_t wd[W];
      pack32_words<W>(y, wd);
#pragma unroll
      for (int k = 0; k < W; ++k) stage_sym[(c * 4 + warp) * W + k] = wd[k];
      stage_sz[(c * 4 + warp) * 2] = __half_as_ushort(s16);
      stage_sz[(c * 4 + warp) * 2 + 1] = __half_as_ushort(z16);
    }
    __syncthreads();
    {
      // thread = channel: 4 groups -> 16*W contiguous bytes, 4 scales, 4 zeros
      const int c = tid;
      uint8_t* dst = a.packed + (((lh * 128 + c) * g.T + t0) * W) / 8;
      const uint32_t* srcw = stage_sym + c * 4 * W;
      if constexpr ((4 * W) % 4 == 0) {
#pragma unroll
        for (int k = 0; k < W; ++k)
          reinterpret_cast<uint4*>(dst)[k] = make_uint4(srcw[4 * k], srcw[4 * k + 1], srcw[4 * k + 2], srcw[4 * k + 3]);
      }
      const int64_t gi = (lh * 128 + c) * g.G + t0 / 32;
      const uint16_t* sz = stage_sz + c * 8;
      *reinterpret_cast<uint2*>(scales + gi) =
          make_uint2((uint32_t)sz[0] | ((uint32_t)sz[2] << 16), (uint32_t)sz[4] | ((uint32_t)sz[6] << 16));
      *reinterpret_cast<uint2*>(zeros + gi) =
          make_uint2((uint32_t)sz[1] | ((uint32_t)sz[3] << 16), (uint32_t)sz[5] | ((uint32_t)sz[7] << 16));
    }
    // the staging buffers are rewritten only after the next block's first
    // __syncthreads, which every thread reaches after finishing these stores
  }
  if (nanacc != 0.0f) flags |= KVC_FLAG_NONFINITE_INPUT;
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

// ------------------------------------------------------------------ decode
template <int W, bool AFFINE, typename Tout>
__global__ void __launch_bounds__(kUThreads, 3) k_dec_uchan128(const DecArgs a) {
  if (payload_rejected(a)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* tile = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 15) & ~(uintptr_t)15);
  // [128 tokens][128 ch] Tout  (bf16: 32 KB, f32: 64 KB)
  uint32_t* stage_sym = reinterpret_cast<uint32_t*>(tile + kUT * 128 * sizeof(Tout));  // [128 ch][4][W]
  float* stage_sz = reinterpret_cast<float*>(stage_sym + 128 * 4 * 8);                 // [128 ch][4][2]
  const Geo& g = a.g;
  const int64_t blocks_per_head = g.T / kUT;
  const int64_t nblocks = g.LH * blocks_per_head;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const __half* scales = reinterpret_cast<const __half*>(a.meta);
  const __half* zeros = scales + g.ngroups;
  uint32_t flags = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const int64_t lh = b / blocks_per_head;
    const int64_t t0 = (b - lh * blocks_per_head) * kUT;
    {
      const int c = tid;
      const uint8_t* src = a.packed + (((lh * 128 + c) * g.T + t0) * W) / 8;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        uint4 w4 = __ldg(reinterpret_cast<const uint4*>(src) + k);
        reinterpret_cast<uint4*>(stage_sym + c * 4 * W)[k] = w4;
      }
      const int64_t gi = (lh * 128 + c) * g.G + t0 / 32;
      uint2 s2 = __ldg(reinterpret_cast<const uint2*>(scales + gi));
      uint2 z2 = __ldg(reinterpret_cast<const uint2*>(zeros + gi));
      const uint32_t sw[2] = {s2.x, s2.y}, zw[2] = {z2.x, z2.y};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint16_t sb = (uint16_t)(sw[k >> 1] >> (16 * (k & 1))), zb = (uint16_t)(zw[k >> 1] >> (16 * (k & 1)));
        stage_sz[(c * 4 + k) * 2] = __half2float(__ushort_as_half(sb));
        stage_sz[(c * 4 + k) * 2 + 1] = __half2float(__ushort_as_half(zb));
      }
    }
    __syncthreads();
    // warp k = token group k; lane = 4 channels
    float outv[4][32];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 4 * lane + j;
      uint32_t wd[W];
#pragma unroll
      for (int k = 0; k < W; ++k) wd[k] = stage_sym[(c * 4 + warp) * W + k];
      unpack32_words<W>(wd, outv[j]);
      const float s = stage_sz[(c * 4 + warp) * 2], z = stage_sz[(c * 4 + warp) * 2 + 1];
      float m = 0.0f, av = 1.0f, rs = 1.0f;
      if (AFFINE) {
        const __half* mu = reinterpret_cast<const __half*>(a.meta + g.meta_affine_off);
        m = __half2float(mu[lh * 128 + c]);
        av = __half2float(mu[g.LH * 128 + lh * 128 + c]);
        rs = __frcp_rn(av);
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float x = __fadd_rn(z, __fmul_rn(outv[j][i], s));
        if (AFFINE) x = __fadd_rn(div_by_rcp(x, av, rs), m);  // y / a correctly rounded
        outv[j][i] = x;
      }
    }
    float chk = 0.0f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int tok = 32 * warp + i;
      if constexpr (sizeof(Tout) == 2) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(outv[0][i], outv[1][i]);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(outv[2][i], outv[3][i]);
        *reinterpret_cast<uint2*>(tile + tok * 256 + lane * 8) =
            make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
      } else {
        *reinterpret_cast<float4*>(tile + tok * 512 + lane * 16) = make_float4(outv[0][i], outv[1][i], outv[2][i], outv[3][i]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) chk = __fmaf_rn(outv[j][i], 0.0f, chk);
    }
    if (chk != 0.0f) flags |= KVC_FLAG_NONFINITE_TRANSFORM;
    __syncthreads();
    // coalesced row stores (contiguous or paged): 16-byte chunks
    constexpr int kRowChunks = 128 * sizeof(Tout) / 16;
    for (int idx = tid; idx < kUT * kRowChunks; idx += kUThreads) {
      const int tok = idx / kRowChunks, ch = idx - tok * kRowChunks;
      Tout* out = reinterpret_cast<Tout*>(a.out) + out_index(a, lh, t0 + tok, 0);
      reinterpret_cast<uint4*>(out)[ch] = reinterpret_cast<const uint4*>(tile + tok * 128 * sizeof(Tout))[ch];
    }
    __syncthreads();
  }
  // OR of the flag bits (not __syncthreads_or, which returns a 0/1 predicate)
  flags = __reduce_or_sync(__activemask(), flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(a.status, flags);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

template <int W, bool AFF>
cudaError_t launch_enc_u(const CUtensorMap& map, const EncArgs& a, int sm_count, cudaStream_t s) {
  auto k = k_enc_uchan128<W, AFF>;
  set_max_dyn_smem<k_enc_uchan128<W, AFF>>(kUSmem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kUThreads, kUSmem);
  if (per_sm < 1) per_sm = 1;
  const int64_t nb = a.g.LH * (a.g.T / kUT);
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > nb) grid = nb;
  k<<<(unsigned)grid, kUThreads, kUSmem, s>>>(map, a);
  return cudaGetLastError();
}

template <int W, bool AFF, typename Tout>
cudaError_t launch_dec_u(const DecArgs& a, int sm_count, cudaStream_t s) {
  auto k = k_dec_uchan128<W, AFF, Tout>;
  const int smem = kUT * 128 * (int)sizeof(Tout) + 128 * 4 * 8 * 4 + 128 * 8 * 4 + 16;
  set_max_dyn_smem<k_dec_uchan128<W, AFF, Tout>>(smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kUThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t nb = a.g.LH * (a.g.T / kUT);
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > nb) grid = nb;
  k<<<(unsigned)grid, kUThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool AFF>
cudaError_t enc_w(const CUtensorMap& m, const EncArgs& a, int sm, cudaStream_t s) {
  switch (a.g.bits) {
    case 1: return launch_enc_u<1, AFF>(m, a, sm, s);
    case 2: return launch_enc_u<2, AFF>(m, a, sm, s);
    case 3: return launch_enc_u<3, AFF>(m, a, sm, s);
    case 4: return launch_enc_u<4, AFF>(m, a, sm, s);
    case 5: return launch_enc_u<5, AFF>(m, a, sm, s);
    case 6: return launch_enc_u<6, AFF>(m, a, sm, s);
    case 7: return launch_enc_u<7, AFF>(m, a, sm, s);
    default: return launch_enc_u<8, AFF>(m, a, sm, s);
  }
}

template <bool AFF, typename Tout>
cudaError_t dec_w(const DecArgs& a, int sm, cudaStream_t s) {
  switch (a.g.bits) {
    case 1: return launch_dec_u<1, AFF, Tout>(a, sm, s);
    case 2: return launch_dec_u<2, AFF, Tout>(a, sm, s);
    case 3: return launch_dec_u<3, AFF, Tout>(a, sm, s);
    case 4: return launch_dec_u<4, AFF, Tout>(a, sm, s);
    case 5: return launch_dec_u<5, AFF, Tout>(a, sm, s);
    case 6: return launch_dec_u<6, AFF, Tout>(a, sm, s);
    case 7: return launch_dec_u<7, AFF, Tout>(a, sm, s);
    default: return launch_dec_u<8, AFF, Tout>(a, sm, s);
  }
}

}  // namespace

bool uchan128_applicable(const Geo& g) {
  return g.uchan && g.C == 128 && g.group == 32 && g.T % kUT == 0 &&
         (g.transform == T_IDENTITY || (g.transform == T_AFFINE && g.meta_affine_off % 16 == 0)) &&
         (g.ngroups * 2) % 8 == 0;
}

cudaError_t launch_encode_uchan128(const EncArgs& a, int sm_count, cudaStream_t s) {
  if (a.g.in_dtype != KVC_DTYPE_BF16 || a.g.LH * a.g.T >= (1ll << 31) || a.paged) return launch_encode_generic(a, s);
  auto fn = encode_fn();
  if (!fn) return launch_encode_generic(a, s);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, (cuuint64_t)(a.g.LH * a.g.T)};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {128, (cuuint32_t)kUT};
  cuuint32_t estr[2] = {1, 1};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.kv), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return launch_encode_generic(a, s);
  ProfScope ps("encode_uchan", s);
  return a.g.transform == T_AFFINE ? enc_w<true>(map, a, sm_count, s) : enc_w<false>(map, a, sm_count, s);
}

cudaError_t launch_decode_uchan128(const DecArgs& a, int sm_count, cudaStream_t s) {
  ProfScope ps("decode_uchan", s);
  const bool aff = a.g.transform == T_AFFINE;
  if (a.g.out_dtype == KVC_DTYPE_BF16)
    return aff ? dec_w<true, __nv_bfloat16>(a, sm_count, s) : dec_w<false, __nv_bfloat16>(a, sm_count, s);
  return aff ? dec_w<true, float>(a, sm_count, s) : dec_w<false, float>(a, sm_count, s);
}

}  // namespace kvc
