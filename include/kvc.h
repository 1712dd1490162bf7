/*
 * kvc.h — C ABI of the B200 KV-cache compression codec (libkvc.so).
 *
 * Drop-in boundary for the reference's codec hot path
 * (/root/reference/pkg/src/kvpilot/pipeline/).  The reference is pure
 * Python, so "its FFI" is the pipeline's public call surface; each entry
 * point below names the reference function it replaces:
 *
 *   kvc_plan_create     <- parse_strategy_id + config validation
 *                          (strategy.py:68-109, quantize.py:26-62,
 *                           transforms.py:25-30, codecs.py:32-38)
 *   kvc_encode          <- the encode closure of compress():
 *                          apply_transform -> classify_heads -> quantize ->
 *                          encode_lossless (compress.py:122-125)
 *   kvc_decode          <- decompress()'s decode closure: decode_lossless ->
 *                          dequantize -> invert_transform (compress.py:150-151)
 *   kvc_decode_paged    <- same, writing into a paged KV cache (extension)
 *   kvc_read_status     <- the ValueError / CodecError raises of
 *                          tensors.py:41-42 and codecs.py:94,166,171,288,389,413,430
 *   kvc_last_error      <- exception message text
 *
 * Conventions: plain pointers and sizes only.  `kv`, `payload`, `metadata`,
 * `block_offsets`, `out` and `workspace` are DEVICE pointers owned by the
 * caller and sized with the query functions; `head_classes` is a HOST array.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  No call
 * allocates device memory; all device work is stream-ordered, and plans are
 * immutable after creation (safe to share across threads and streams).  A
 * workspace carries one operation's scratch and status word: operations in
 * flight at the same time (e.g. on two streams) need one workspace each.
 * Every function returns a kvc_status; on failure kvc_last_error() holds a
 * thread-local message.
 */
#ifndef KVC_H_
#define KVC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kvc_plan kvc_plan;

typedef enum {
  KVC_OK = 0,
  KVC_ERR_CONFIG = 1, /* ValueError: bad strategy id / shape / options      */
  KVC_ERR_CODEC = 2,  /* CodecError: malformed or mismatched payload          */
  KVC_ERR_CUDA = 3,   /* CUDA runtime failure                                 */
  KVC_ERR_VALUE = 4   /* ValueError raised by the data (non-finite values)    */
} kvc_status;

enum { KVC_DTYPE_BF16 = 0, KVC_DTYPE_F32 = 1 };

/* device status word flags (kvc_read_status) */
enum {
  KVC_FLAG_NONFINITE_INPUT = 1u,     /* tensors.py:41-42 on the input          */
  KVC_FLAG_NONFINITE_TRANSFORM = 2u, /* transform overflowed float32           */
  KVC_FLAG_CODEC = 4u,               /* truncated / trailing / length mismatch */
  KVC_FLAG_CAPACITY = 8u,            /* entropy block exceeded its scratch slot */
  KVC_FLAG_FP16_RANGE = 16u          /* a zero/scale overflowed float16 (the
                                        reference reproduces this; decode then
                                        yields +-inf and raises ValueError)    */
};

typedef struct {
  int64_t block_symbols; /* codec block (entropy / rle framing); multiple of 8; 0 -> 2048 */
  int32_t in_dtype;      /* KVC_DTYPE_BF16 (serving cache) or KVC_DTYPE_F32 (reference) */
  int32_t out_dtype;     /* decode output dtype                                 */
  int32_t reserved[8];
} kvc_options;

/* Create a plan for one KV tensor shape (layers, heads, tokens, channels)
 * and one strategy id, e.g. "t=hadamard;q=uniform,b=4,g=32;c=none".
 * Accepts the reference grammar (strategy.py:8-19) plus the extension kinds
 * t=affine, q=uchan / mixlayer / mixtok. */
int kvc_plan_create(kvc_plan** out, const char* strategy_id, int64_t layers, int64_t heads, int64_t tokens,
                    int64_t channels, const kvc_options* options);
int kvc_plan_destroy(kvc_plan* plan);

/* Canonical strategy id of the plan (NUL-terminated, owned by the plan). */
const char* kvc_plan_strategy_id(const kvc_plan* plan);

/* Kernel family kvc_encode / kvc_decode run for this plan: "fast128",
 * "fast128-cert+fp64+fixup" (Hadamard, bf16 input: the certified
 * float32 encoder, a float64 pass for the rows it cannot certify, then the
 * exact fixup; the environment variable KVC_HADAMARD_FP64=1 selects the
 * float64 encoder instead), "fast128+fixup", "uchan128", "fused_rc",
 * "delta128", or "generic: <why>" (the per-element correctness kernels, e.g.
 * float32 input).  Static strings. */
const char* kvc_plan_encode_path(const kvc_plan* plan);
const char* kvc_plan_decode_path(const kvc_plan* plan);

int64_t kvc_metadata_bytes(const kvc_plan* plan);  /* exact metadata size          */
int64_t kvc_payload_capacity(const kvc_plan* plan); /* upper bound on payload size   */
int64_t kvc_workspace_bytes(const kvc_plan* plan);  /* scratch needed by encode/decode */
int64_t kvc_max_blocks(const kvc_plan* plan);       /* block_offsets needs max_blocks+1 */

/* Payload bytes when they do not depend on the data (codec none), else -1:
 * then the size is block_offsets[nblocks] on the device after kvc_encode. */
int64_t kvc_static_payload_bytes(const kvc_plan* plan, const uint8_t* head_classes);
/* Number of codec blocks for these head classes (0 for codec none). */
int64_t kvc_num_blocks(const kvc_plan* plan, const uint8_t* head_classes);

/* Encode one KV tensor.  `kv` is (L,H,T,C) row-major in the plan's in_dtype.
 * `head_classes` (host, L*H bytes, nonzero = retrieval head) is required for
 * q=mixed / mixlayer and ignored otherwise.  Writes metadata (exactly
 * kvc_metadata_bytes), payload, and for rle/entropy the block offset table
 * (uint64, nblocks+1 entries, offsets into payload). */
int kvc_encode(const kvc_plan* plan, const void* kv, const uint8_t* head_classes, void* payload, void* metadata,
               uint64_t* block_offsets, void* workspace, void* stream);

/* kvc_encode reading the KV straight from a paged cache (the layout of
 * kvc_decode_paged: element (l,h,t,c) at
 *   page_base + l*layer_stride + (block_table[t / page_tokens]*page_tokens + t % page_tokens)*H*C + h*C + c),
 * in the plan's in_dtype.  The blob is byte-identical to kvc_encode of the
 * gathered contiguous tensor, with no gather pass.  The block table is trusted. */
int kvc_encode_paged(const kvc_plan* plan, const void* page_base, const int32_t* block_table, int64_t page_tokens,
                     int64_t layer_stride, const uint8_t* head_classes, void* payload, void* metadata,
                     uint64_t* block_offsets, void* workspace, void* stream);

/* Decode into a contiguous (L,H,T,C) tensor of the plan's out_dtype.
 * `payload_bytes` is the received payload length (checked like the
 * reference's trailing-byte rule, codecs.py:412-413 / :429-430): every block
 * offset is bounded by it, so any payload bytes and any offset table decode
 * or raise KVC_FLAG_CODEC, never read outside [payload, payload+payload_bytes).
 * Pass -1 for a device-resident blob this library encoded (its length is
 * block_offsets[nblocks]): the offsets are then trusted, not bounded. */
int kvc_decode(const kvc_plan* plan, const void* payload, int64_t payload_bytes, const void* metadata,
               const uint64_t* block_offsets, void* out, void* workspace, void* stream);

/* Decode into a paged cache: element (l,h,t,c) lands at
 *   base + l*layer_stride + (block_table[t / page_tokens]*page_tokens + t % page_tokens)*H*C + h*C + c
 * (vLLM layout [num_pages, page_tokens, heads, channels] per layer; strides in elements).
 * The block table is trusted: its entries must name pages inside page_base. */
int kvc_decode_paged(const kvc_plan* plan, const void* payload, int64_t payload_bytes, const void* metadata,
                     const uint64_t* block_offsets, void* page_base, const int32_t* block_table, int64_t page_tokens,
                     int64_t layer_stride, void* workspace, void* stream);

/* Synchronise `stream` and read (then clear) the device status word. */
int kvc_read_status(const kvc_plan* plan, void* workspace, void* stream, uint32_t* flags);

const char* kvc_last_error(void);
const char* kvc_version(void);

/* Per-block CRC-32 (IEEE 802.3 / zlib.crc32 polynomial, reflected, init and
 * final xor 0xFFFFFFFF) of an encoded payload: block b covers device bytes
 * [block_offsets[b], block_offsets[b+1]) of `payload`; `crc` (device,
 * nblocks entries) receives one checksum per block.  Used by the block-framed
 * wire container (the reference blob has no checksum,
 * codecs.py:41-59).  A whole-buffer checksum is nblocks = 1 with offsets
 * {0, len}. */
int kvc_block_crc32(const void* payload, const uint64_t* block_offsets, int64_t nblocks, uint32_t* crc, void* stream);

/* Copy a data-dependent number of bytes without a host round trip: copies
 * min(*nbytes_dev, max_bytes) bytes from src to dst, where *nbytes_dev is a
 * device-resident length (e.g. block_offsets[nblocks] of an encode).  src and
 * dst may live on different GPUs (peer access enabled with
 * kvc_enable_peer_access): the kernel runs on the stream's device and moves
 * 16-byte vectors over NVLink.  Used by the pipelined compress -> transfer ->
 * decompress path. */
int kvc_copy_device_length(void* dst, const void* src, const uint64_t* nbytes_dev, int64_t max_bytes, void* stream);

/* *sum_dev += sum over i < n of (a[i] - b[i])^2 (differences, squares and
 * accumulation in fp64; a, b device arrays of dtype KVC_DTYPE_BF16 or
 * KVC_DTYPE_F32; b may be NULL for sum a[i]^2): the RMSE / RMS terms of
 * quality_score (tensors.py:115-134) in one HBM-bound pass each. */
int kvc_sq_error(const void* a, const void* b, int64_t n, int dtype, double* sum_dev, void* stream);

/* Deterministic form of kvc_sq_error: npartials CTAs (1..65535) with a fixed
 * work split and reduction order; CTA i adds its share to partials[i] (device,
 * npartials doubles).  Summing the partials in order gives the same bits on
 * every call (the quality_score of the profiling evaluator must be a function
 * of its inputs, search.py:348-368). */
int kvc_sq_error_partials(const void* a, const void* b, int64_t n, int dtype, double* partials, int64_t npartials,
                          void* stream);

/* cudaDeviceEnablePeerAccess(peer) from `device` (already-enabled is OK). */
int kvc_enable_peer_access(int device, int peer);

/* Per-kernel timing (the native side of the StageTimer hook, compress.py:43-48).
 * When enabled, every kernel the library launches on the calling thread is
 * bracketed by CUDA events on its stream.  kvc_profile_collect synchronises,
 * accumulates elapsed milliseconds per kernel name into `ms` / `launches`
 * (up to `cap` distinct names, order of first launch), writes the names
 * (NUL-separated) into `names` (size `names_cap`), clears the record and
 * returns the number of names. */
int kvc_profile_enable(int on);
int kvc_profile_collect(char* names, int64_t names_cap, double* ms, int64_t* launches, int cap);

#ifdef __cplusplus
}
#endif

#endif /* KVC_H_ */
