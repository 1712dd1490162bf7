// Codec stage over packed width streams: dispatch of the block range coders
// (rc_small.cu: w <= 4, rc_large.cu: w >= 5), PackBits RLE, and the
// block-offset scan + gather.
//
// A width stream (codecs.py:339-345) is cut into blocks of g.block symbols;
// each block is coded independently with the reference's own algorithm so
// decoding is parallel (one thread per block):
//   entropy block = BE32(len) || range_encode(block, 1 << w)  (codecs.py:245-270, :310-317, :364-366)
//   rle block     = rle_encode(packed block bytes)             (codecs.py:112-152)
// Encode writes each block into a worst-case-sized scratch slot, then one
// kernel (k_scan_offsets: single-pass decoupled look-back) turns the sizes into
// block_offsets and k_gather packs the slots into the payload.
#include "kernels.h"
#include "profile.h"
#include "rc_tables.cuh"

namespace kvc {

namespace {

// ----------------------------------------------------------------- RLE
// 16-byte vector reader (byte loads when the range is not 16-byte aligned,
// e.g. tiny blocks of odd widths)
struct VecReader {
  const uint4* p;
  const uint8_t* bp;
  uint4 cur;
  int idx;  // next byte within cur (0..16)
  bool vec;
  __device__ __forceinline__ void init(const uint8_t* src) {
    p = reinterpret_cast<const uint4*>(src);
    bp = src;
    vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    idx = 16;
  }
  __device__ __forceinline__ uint32_t next() {
    if (!vec) return __ldg(bp++);
    if (idx == 16) {
      cur = __ldg(p++);
      idx = 0;
    }
    const uint32_t w = (idx < 8) ? ((idx < 4) ? cur.x : cur.y) : ((idx < 12) ? cur.z : cur.w);
    const uint32_t b = (w >> (8 * (idx & 3))) & 0xFFu;
    ++idx;
    return b;
  }
};

__device__ void rle_encode_block(const uint8_t* src, int n, uint8_t* slot, int64_t cap, uint64_t* size_out,
                                 uint32_t* status) {
  // greedy PackBits (codecs.py:112-152), single pass: runs >= 3 become
  // (128+len-3, byte) in chunks <= 130; all other bytes go into literal
  // chunks <= 128 whose control byte is back-filled when the chunk closes.
  // Output <= n + ceil(n/128) bytes, within the slot by construction.
  (void)cap;
  (void)status;
  VecReader rd;
  rd.init(src);
  // output bytes collect in a little-endian word and leave as 32-bit stores
  // (the slot is 16-byte aligned); a literal chunk's control byte is patched
  // in the word if it is still open, else by one byte store
  uint32_t* sw = reinterpret_cast<uint32_t*>(slot);
  uint32_t acc = 0;
  int pos = 0;         // output position
  int lit_ctrl = -1;   // position of the open literal chunk's control byte
  int lit_len = 0;
  auto put = [&](uint32_t b) {
    acc |= b << (8 * (pos & 3));
    if ((pos & 3) == 3) {
      sw[pos >> 2] = acc;
      acc = 0;
    }
    ++pos;
  };
  auto patch = [&](int at, uint32_t b) {
    if ((at >> 2) == (pos >> 2)) {
      acc |= b << (8 * (at & 3));
    } else {
      slot[at] = (uint8_t)b;
    }
  };
  auto lit_byte = [&](uint32_t b) {
    if (lit_ctrl < 0 || lit_len == 128) {
      if (lit_ctrl >= 0) patch(lit_ctrl, (uint32_t)(lit_len - 1));
      lit_ctrl = pos;
      put(0u);  // placeholder for the control byte
      lit_len = 0;
    }
    put(b);
    ++lit_len;
  };
  auto lit_close = [&]() {
    if (lit_ctrl >= 0) patch(lit_ctrl, (uint32_t)(lit_len - 1));
    lit_ctrl = -1;
    lit_len = 0;
  };
  int i = 0;
  uint32_t v = n > 0 ? rd.next() : 0u;
  while (i < n) {
    int run = 1;
    uint32_t nb = 0;
    bool more = false;
    while (i + run < n) {
      nb = rd.next();
      if (nb != v) {
        more = true;
        break;
      }
      ++run;
    }
    if (run >= 3) {
      lit_close();
      int r = run;
      while (r >= 3) {
        const int ch = r < 130 ? r : 130;
        put((uint32_t)(128 + ch - 3));
        put(v);
        r -= ch;
      }
      for (int k = 0; k < r; ++k) lit_byte(v);  // leftover < 3 starts a literal
    } else {
      for (int k = 0; k < run; ++k) lit_byte(v);
    }
    i += run;
    if (more) v = nb;
  }
  lit_close();
  if (pos & 3) sw[pos >> 2] = acc;  // the partial last word (bytes past pos are slack)
  *size_out = (uint64_t)pos;
}

__device__ __forceinline__ int block_stream(const StreamTab& st, int64_t b) {
  return (st.n > 1 && b >= st.first_block[1]) ? 1 : 0;
}

__global__ void __launch_bounds__(128) k_rle_encode(CodecArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > a.max_blocks) return;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) {
    a.sizes[b] = 0;
    return;
  }
  if (a.g.rle_whole) {  // the concatenated byte-padded streams (codecs.py:358-360)
    rle_encode_block(a.packed_in, (int)st.packed_bytes, a.slots, a.slot_bytes, a.sizes, a.status);
    return;
  }
  const int si = block_stream(st, b);
  const int w = st.w[si];
  const int64_t start = (b - st.first_block[si]) * a.g.block;
  const int64_t n = min(a.g.block, st.count[si] - start);
  const uint8_t* src = a.packed_in + st.byte_off[si] + start * w / 8;
  rle_encode_block(src, (n * w + 7) / 8, a.slots + b * a.slot_bytes, a.slot_bytes, a.sizes + b, a.status);
}

__global__ void __launch_bounds__(128) k_rle_decode(CodecArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const StreamTab st = *a.st;
  if (b >= st.nblocks) return;
  const int si = block_stream(st, b);
  const int w = st.w[si];
  const int64_t start = a.g.rle_whole ? 0 : (b - st.first_block[si]) * a.g.block;
  const int64_t n = min(a.g.block, st.count[si] - start);
  // whole-tensor rle: the block decodes to all packed streams, back to back
  const int64_t want = a.g.rle_whole ? st.packed_bytes : (n * w + 7) / 8;
  const uint64_t o0 = a.offsets_in[b], o1 = a.offsets_in[b + 1];
  // PackBits grows a block by at most one control byte per 128 literals
  if (o1 < o0 || o1 - o0 > (uint64_t)(want + want / 64 + 16) ||
      (a.payload_bytes >= 0 && o1 > (uint64_t)a.payload_bytes)) {
    atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  const uint8_t* in = a.payload_in + o0;
  const int len = (int)(o1 - o0);
  uint8_t* out = a.packed_out + (a.g.rle_whole ? 0 : st.byte_off[si] + start * w / 8);
  // input: aligned words, clamped to the word holding the block's last byte
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uint32_t* iw = reinterpret_cast<const uint32_t*>(ia & ~(uintptr_t)3);
  const int ilast = len > 0 ? (int)(((ia + len - 1) & ~(uintptr_t)3) - (ia & ~(uintptr_t)3)) / 4 : 0;
  int wi = 0, avail = 0;
  uint32_t cur = 0;
  int skip = (int)(ia & 3);
  auto rd = [&]() -> uint32_t {
    if (avail == 0) {
      cur = __ldg(iw + min(wi, ilast)) >> (8 * skip);
      avail = 4 - skip;
      skip = 0;
      ++wi;
    }
    const uint32_t b = cur & 0xFFu;
    cur >>= 8;
    --avail;
    return b;
  };
  // output: little-endian word accumulator (the block start is 4-aligned)
  const bool oal = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  uint32_t acc = 0;
  int o = 0;
  auto wr = [&](uint32_t b) {
    if (oal) {
      acc |= b << (8 * (o & 3));
      if ((o & 3) == 3) {
        reinterpret_cast<uint32_t*>(out)[o >> 2] = acc;
        acc = 0;
      }
    } else {
      out[o] = (uint8_t)b;
    }
    ++o;
  };
  int pos = 0;
  bool bad = false;
  while (pos < len) {  // codecs.py:155-174
    const uint32_t c = rd();
    ++pos;
    if (c < 128) {
      const int l = (int)c + 1;
      if (pos + l > len || o + l > want) { bad = true; break; }
      for (int k = 0; k < l; ++k) wr(rd());
      pos += l;
    } else {
      if (pos >= len) { bad = true; break; }
      const int l = (int)c - 125;
      if (o + l > want) { bad = true; break; }
      const uint32_t v = rd();
      ++pos;
      for (int k = 0; k < l; ++k) wr(v);
    }
  }
  if (oal && (o & 3)) {  // partial last word: bytes only (a neighbour may own the rest)
    for (int k = 0; k < (o & 3); ++k) out[(o & ~3) + k] = (uint8_t)(acc >> (8 * k));
  }
  if (bad || o != want) atomicOr(a.status, KVC_FLAG_CODEC);
}

// ---------------------------------------------------------- scan + gather
// one warp per block copies its slot bytes to payload[offsets[b]]: partial
// head / tail words byte by byte (they are shared with the neighbouring
// blocks), the aligned body as 32-bit words funnel-shifted out of the
// 16-byte-aligned slot
// one warp copies block b's bytes [o0, o1) of the payload from its slot: the
// unaligned head / tail bytewise, the body as 32-bit words funnel-shifted out
// of the 16-byte-aligned slot, U words per lane in flight
__device__ __forceinline__ void copy_block(const CodecArgs& a, int64_t b, uint64_t o0, uint64_t o1, int lane) {
  const uint32_t len = (uint32_t)(o1 - o0);
  const uint8_t* src = a.slots + b * a.slot_bytes;
  uint8_t* dst = a.payload_out + o0;
  const uint32_t head = min((uint32_t)((4u - (uint32_t)(o0 & 3u)) & 3u), len);
  const uint32_t words = (len - head) >> 2;
  const uint32_t tail = len - head - 4 * words;
  if (lane < (int)head) dst[lane] = src[lane];
  if (lane < (int)tail) dst[head + 4 * words + lane] = src[head + 4 * words + lane];
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
  const uint32_t sh = 8 * head;  // src byte offset of the body inside its first word
  // all loads of a round before any store (slots and payload never overlap,
  // but the compiler cannot know that and would serialize them)
  constexpr uint32_t U = 4;
  for (uint32_t w0 = lane; w0 < words; w0 += 32 * U) {
    uint32_t lo[U], hi[U];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t w = w0 + 32 * u;
      lo[u] = w < words ? __ldg(s32 + w) : 0u;
      hi[u] = (w < words && sh) ? __ldg(s32 + w + 1) : 0u;
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t w = w0 + 32 * u;
      if (w < words) d32[w] = sh ? __funnelshift_r(lo[u], hi[u], sh) : lo[u];
    }
  }
}

// Block offsets in one pass over the sizes (single-pass decoupled look-back,
// no library scan): CTAs take tiles of kScanTile block sizes in launch order
// (an atomic ticket, so every lower tile has started and will finish: the
// look-back cannot deadlock), scan them in shared memory, publish the tile
// aggregate, then thread 0 walks back over the predecessors' published
// aggregates / inclusive prefixes until it meets an inclusive one.
constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;
constexpr uint64_t kStAgg = 1ull << 62, kStInc = 2ull << 62, kStVal = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kScanThreads) k_scan_offsets(CodecArgs a, uint64_t* status, uint32_t* ticket) {
  __shared__ uint64_t warp_sum[kScanThreads / 32];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = (int64_t)atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t n = a.max_blocks + 1;  // sizes / offsets entries
  const int64_t b0 = tile * kScanTile + (int64_t)tid * kScanItems;
  // kScanItems consecutive sizes per thread, summed locally
  uint64_t v[kScanItems], mine = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = b0 + k < n ? a.sizes[b0 + k] : 0ull;
    mine += v[k];
  }
  uint64_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sum[warp] = incl;
  __syncthreads();
  uint64_t wpre = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    if (w < warp) wpre += warp_sum[w];
    agg += warp_sum[w];
  }
  if (tid == 0) {
    uint64_t prefix = 0;
    if (tile == 0) {
      st_status(status + tile, kStInc | agg);
    } else {
      st_status(status + tile, kStAgg | agg);
      for (int64_t t = tile - 1; t >= 0; --t) {
        uint64_t st;
        while (((st = ld_status(status + t)) & ~kStVal) == 0ull) {
        }
        prefix += st & kStVal;
        if (st & kStInc) break;
      }
      st_status(status + tile, kStInc | (prefix + agg));
    }
    s_prefix = prefix;
  }
  __syncthreads();
  uint64_t off = s_prefix + wpre + incl - mine;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (b0 + k < n) a.offsets[b0 + k] = off;
    off += v[k];
  }
}

// decode-side checks: offsets[0] == 0, offsets[nblocks] == payload bytes
// (codecs.py:412-413 / :429-430 trailing-byte rule), none: exact length.
__global__ void k_check_payload(CodecArgs a) {
  const StreamTab& st = *a.st;
  if (a.g.codec == C_NONE) {
    if (a.payload_bytes >= 0 && a.payload_bytes != st.packed_bytes) atomicOr(a.status, KVC_FLAG_CODEC);
    return;
  }
  if (a.offsets_in[0] != 0) atomicOr(a.status, KVC_FLAG_CODEC);
  if (a.payload_bytes >= 0 && a.offsets_in[st.nblocks] != (uint64_t)a.payload_bytes) atomicOr(a.status, KVC_FLAG_CODEC);
}

void widths_used(const Geo& g, bool used[9]) {
  for (int i = 0; i < 9; ++i) used[i] = false;
  if (g.quant == Q_UNIFORM || g.quant == Q_UCHAN) {
    used[g.bits] = true;
  } else {
    used[g.hi] = used[g.lo] = true;
  }
}

}  // namespace

// slots -> payload, one warp per block, grid-stride; the next block's offsets
// are loaded while the current one is copied
__global__ void __launch_bounds__(256) k_gather(CodecArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  const int64_t nb = a.st->nblocks;
  int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t o0 = 0, o1 = 0;
  if (b < nb) {
    o0 = a.offsets[b];
    o1 = a.offsets[b + 1];
  }
  for (; b < nb; b += nwarps) {
    const int64_t bn = b + nwarps;
    uint64_t n0 = 0, n1 = 0;
    if (bn < nb) {
      n0 = a.offsets[bn];
      n1 = a.offsets[bn + 1];
    }
    copy_block(a, b, o0, o1, lane);
    o0 = n0;
    o1 = n1;
  }
}

// look-back state: a ticket counter, then one status word per tile
size_t codec_scan_bytes(int64_t max_blocks) {
  const int64_t tiles = (max_blocks + 1 + kScanTile - 1) / kScanTile;
  return (size_t)(16 + 8 * tiles);
}

cudaError_t launch_codec_encode(const CodecArgs& args, int sm_count, cudaStream_t s) {
  (void)sm_count;
  CodecArgs a = args;
  if (a.g.codec == C_ENTROPY) {
    if (cudaError_t te = ensure_recip_tables(); te != cudaSuccess) return te;
    a.recip = recip_tables();
  }
  const unsigned grid = (unsigned)((a.max_blocks + 1 + 127) / 128);
  bool used[9];
  widths_used(a.g, used);
  if (a.g.codec == C_ENTROPY) {
    // one launch per width in use; each thread skips blocks of other widths
    for (int w = 1; w <= 8; ++w) {
      if (!used[w]) continue;
      cudaError_t e = w <= 4 ? launch_rc_small_encode(a, w, grid, s) : launch_rc_large_encode(a, w, s);
      if (e != cudaSuccess) return e;
    }
  } else {
    ProfScope ps("rle_encode", s);
    k_rle_encode<<<grid, 128, 0, s>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_codec_finish(a, s);
}

cudaError_t launch_codec_finish(const CodecArgs& a, cudaStream_t s) {
  const int64_t tiles = (a.max_blocks + 1 + kScanTile - 1) / kScanTile;
  uint32_t* ticket = reinterpret_cast<uint32_t*>(a.scan_tmp);
  uint64_t* status = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(a.scan_tmp) + 16);
  cudaError_t e = cudaMemsetAsync(a.scan_tmp, 0, codec_scan_bytes(a.max_blocks), s);
  if (e != cudaSuccess) return e;
  {
    ProfScope ps("offset_scan", s);
    k_scan_offsets<<<(unsigned)tiles, kScanThreads, 0, s>>>(a, status, ticket);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (a.max_blocks * 32 + 255) / 256 + 1;
  const int64_t cap = (int64_t)sms * 16;
  const unsigned ggrid = (unsigned)(want < cap ? want : cap);
  ProfScope ps("gather", s);
  k_gather<<<ggrid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_check_payload(const CodecArgs& a, cudaStream_t s) {
  ProfScope ps("check_payload", s);
  k_check_payload<<<1, 1, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_codec_decode(const CodecArgs& args, int sm_count, cudaStream_t s) {
  (void)sm_count;
  CodecArgs a = args;
  if (a.g.codec == C_ENTROPY) {
    if (cudaError_t te = ensure_recip_tables(); te != cudaSuccess) return te;
    a.recip = recip_tables();
  }
  cudaError_t ce = launch_check_payload(a, s);
  if (ce != cudaSuccess || a.g.codec == C_NONE) return ce;
  const unsigned grid = (unsigned)((a.max_blocks + 127) / 128 + 1);
  bool used[9];
  widths_used(a.g, used);
  if (a.g.codec == C_ENTROPY) {
    for (int w = 1; w <= 8; ++w) {
      if (!used[w]) continue;
      cudaError_t e = w <= 4 ? launch_rc_small_decode(a, w, grid, s) : launch_rc_large_decode(a, w, s);
      if (e != cudaSuccess) return e;
    }
  } else {
    ProfScope ps("rle_decode", s);
    k_rle_decode<<<grid, 128, 0, s>>>(a);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------ block CRC-32
// One thread per block, slicing-by-4 over 32-bit words with the four 256-entry
// tables in shared memory (built per CTA); unaligned head / tail bytes one at
// a time.  Blocks are a few hundred bytes, so this is a small fraction of an
// encode; it exists for the wire container's integrity check.
__global__ void __launch_bounds__(256) k_block_crc32(const uint8_t* payload, const uint64_t* offsets, int64_t nblocks,
                                                     uint32_t* crc) {
  __shared__ uint32_t tab[4][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    tab[0][i] = c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = tab[0][i];
    for (int t = 1; t < 4; ++t) {
      c = (c >> 8) ^ tab[0][c & 0xFFu];
      tab[t][i] = c;
    }
  }
  __syncthreads();
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const uint64_t o0 = offsets[b], o1 = offsets[b + 1];
  const uint8_t* p = payload + o0;
  uint64_t n = o1 > o0 ? o1 - o0 : 0;
  uint32_t c = 0xFFFFFFFFu;
  while (n && (reinterpret_cast<uintptr_t>(p) & 3u)) {
    c = (c >> 8) ^ tab[0][(c ^ *p++) & 0xFFu];
    --n;
  }
  const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
  for (; n >= 4; n -= 4) {
    const uint32_t x = c ^ __ldg(w++);
    c = tab[3][x & 0xFFu] ^ tab[2][(x >> 8) & 0xFFu] ^ tab[1][(x >> 16) & 0xFFu] ^ tab[0][x >> 24];
  }
  p = reinterpret_cast<const uint8_t*>(w);
  while (n--) c = (c >> 8) ^ tab[0][(c ^ *p++) & 0xFFu];
  crc[b] = c ^ 0xFFFFFFFFu;
}

cudaError_t launch_block_crc32(const uint8_t* payload, const uint64_t* offsets, int64_t nblocks, uint32_t* crc,
                               cudaStream_t s) {
  ProfScope ps("block_crc32", s);
  k_block_crc32<<<(unsigned)((nblocks + 255) / 256), 256, 0, s>>>(payload, offsets, nblocks, crc);
  return cudaGetLastError();
}

// ------------------------------------------------ device-length copy (P2P)
// The length lives in device memory, so a pipelined transfer never syncs to
// learn a data-dependent payload size.  16-byte vectors when both ends are
// 16-byte aligned (blob buffers are), bytes otherwise.
__global__ void __launch_bounds__(256) k_copy_device_length(uint8_t* dst, const uint8_t* src,
                                                            const uint64_t* nbytes_dev, int64_t max_bytes) {
  const uint64_t want = *nbytes_dev;
  const uint64_t n = want < (uint64_t)max_bytes ? want : (uint64_t)max_bytes;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
    const uint64_t nv = n >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint64_t i = tid; i < nv; i += stride) d4[i] = s4[i];
    for (uint64_t i = (nv << 4) + tid; i < n; i += stride) dst[i] = src[i];
  } else {
    for (uint64_t i = tid; i < n; i += stride) dst[i] = src[i];
  }
}

cudaError_t launch_copy_device_length(void* dst, const void* src, const uint64_t* nbytes_dev, int64_t max_bytes,
                                      cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (max_bytes / 16 + 255) / 256 + 1;
  // one CTA per SM moves bytes at link speed and leaves the SMs to the
  // encoder running beside it (pipelined transfers)
  const int64_t cap = (int64_t)sms;
  ProfScope ps("copy_device_length", s);
  k_copy_device_length<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(
      reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src), nbytes_dev, max_bytes);
  return cudaGetLastError();
}

// ------------------------------------------------------ squared error sum
// sum((a - b)^2) (b == nullptr: sum(a^2)) with every difference and square in
// fp64 (exact differences, like tensors.py:126's astype(float64) - ...), fp64
// accumulation; only the summation order differs from numpy's pairwise mean
__device__ __forceinline__ double sq_term(float a, float b) {
  const double d = (double)a - (double)b;
  return d * d;
}
// PARTIALS: block i adds its sum to out[i] (fixed work split and fixed
// reduction order: deterministic); else every block atomically adds to out[0]
template <typename T, bool HAS_B, bool PARTIALS = false>
__global__ void __launch_bounds__(256) k_sq_error(const T* a, const T* b, int64_t n, double* out) {
  constexpr int kVec = 16 / sizeof(T);
  const int64_t nv = n / kVec;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  const uint4* a4 = reinterpret_cast<const uint4*>(a);
  const uint4* b4 = reinterpret_cast<const uint4*>(b);
  for (int64_t i = tid; i < nv; i += stride) {
    const uint4 x = __ldg(a4 + i);
    const uint4 y = HAS_B ? __ldg(b4 + i) : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (sizeof(T) == 2) {
        acc += sq_term(__uint_as_float(xw[k] << 16), __uint_as_float(yw[k] << 16));
        acc += sq_term(__uint_as_float(xw[k] & 0xFFFF0000u), __uint_as_float(yw[k] & 0xFFFF0000u));
      } else {
        acc += sq_term(__uint_as_float(xw[k]), __uint_as_float(yw[k]));
      }
    }
  }
  for (int64_t i = nv * kVec + tid; i < n; i += stride) {
    float fa, fb = 0.0f;
    if constexpr (sizeof(T) == 2) {
      fa = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(a)[i] << 16);
      if (HAS_B) fb = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(b)[i] << 16);
    } else {
      fa = reinterpret_cast<const float*>(a)[i];
      if (HAS_B) fb = reinterpret_cast<const float*>(b)[i];
    }
    acc += sq_term(fa, fb);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    if (PARTIALS) out[blockIdx.x] += t;
    else atomicAdd(out, t);
  }
}

cudaError_t launch_sq_error(const void* a, const void* b, int64_t n, int dtype, double* out, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n / 8 + 255) / 256 + 1;
  const int64_t cap = (int64_t)sms * 8;
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  ProfScope ps("sq_error", s);
  const uint16_t* ah = reinterpret_cast<const uint16_t*>(a);
  const uint16_t* bh = reinterpret_cast<const uint16_t*>(b);
  const float* af = reinterpret_cast<const float*>(a);
  const float* bf = reinterpret_cast<const float*>(b);
  if (dtype == KVC_DTYPE_BF16) {
    if (b) k_sq_error<uint16_t, true><<<grid, 256, 0, s>>>(ah, bh, n, out);
    else k_sq_error<uint16_t, false><<<grid, 256, 0, s>>>(ah, bh, n, out);
  } else {
    if (b) k_sq_error<float, true><<<grid, 256, 0, s>>>(af, bf, n, out);
    else k_sq_error<float, false><<<grid, 256, 0, s>>>(af, bf, n, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_sq_error_partials(const void* a, const void* b, int64_t n, int dtype, double* partials,
                                     int64_t npartials, cudaStream_t s) {
  const unsigned grid = (unsigned)npartials;
  ProfScope ps("sq_error", s);
  const uint16_t* ah = reinterpret_cast<const uint16_t*>(a);
  const uint16_t* bh = reinterpret_cast<const uint16_t*>(b);
  const float* af = reinterpret_cast<const float*>(a);
  const float* bf = reinterpret_cast<const float*>(b);
  if (dtype == KVC_DTYPE_BF16) {
    if (b) k_sq_error<uint16_t, true, true><<<grid, 256, 0, s>>>(ah, bh, n, partials);
    else k_sq_error<uint16_t, false, true><<<grid, 256, 0, s>>>(ah, bh, n, partials);
  } else {
    if (b) k_sq_error<float, true, true><<<grid, 256, 0, s>>>(af, bf, n, partials);
    else k_sq_error<float, false, true><<<grid, 256, 0, s>>>(af, bf, n, partials);
  }
  return cudaGetLastError();
}

}  // namespace kvc
