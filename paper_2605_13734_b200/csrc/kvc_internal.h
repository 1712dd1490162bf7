// Internal plan / geometry shared by the host API and the CUDA kernels.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

#include "kvc.h"

namespace kvc {

enum Transform : int { T_IDENTITY = 0, T_DELTA = 1, T_HADAMARD = 2, T_AFFINE = 3 };
enum Quant : int { Q_UNIFORM = 0, Q_UCHAN = 1, Q_MIXED = 2, Q_MIXLAYER = 3, Q_MIXTOK = 4 };
enum Codec : int { C_NONE = 0, C_RLE = 1, C_ENTROPY = 2 };

constexpr int kAffinePrefix = 128;  // tokens used to calibrate t=affine
constexpr int kMaxStreams = 2;

// Everything a kernel needs to know about the tensor + strategy.  Passed by
// value (fits easily in the kernel parameter space).
struct Geo {
  int64_t L, H, T, C;
  int64_t LH;        // L*H heads
  int64_t E;         // total elements
  int transform, quant, codec;
  int bits, hi, lo, group;
  int64_t k_tok;     // mixtok: number of hi tokens (the most recent ones)
  int uchan;         // groups run along tokens
  int64_t rowlen;    // symbols per quant row (C, or T for uchan)
  int64_t G;         // groups per quant row
  int64_t ngroups;   // total groups (= scales count)
  int64_t meta_class_off;   // byte offset of the packed class map in metadata (or -1)
  int64_t meta_affine_off;  // byte offset of mu16||a16 in metadata (or -1)
  int64_t block;     // codec block in symbols
  int in_dtype, out_dtype;
  int rle_whole;     // rle with one block covering the whole tensor: the block is
                     // the concatenated packed width streams (codecs.py:358-360)
};

// Width streams (codecs.py:339-345): widths descending.
struct StreamTab {
  int n;
  int w[kMaxStreams];
  int64_t count[kMaxStreams];       // symbols
  int64_t byte_off[kMaxStreams];    // offset of the stream in the packed buffer
  int64_t first_block[kMaxStreams];
  int64_t nblocks;                  // total codec blocks
  int64_t packed_bytes;             // total packed bytes (== none payload)
};

// Per head entry for head-mixed strategies: width and bit offset of the
// head's first symbol in the packed buffer.
struct HeadEntry {
  int64_t bit;
  int32_t w;
  int32_t pad;
};

struct Plan {
  Geo g;
  char id[256];
  int64_t meta_bytes;
  int64_t payload_cap;
  int64_t max_blocks;
  int64_t ws_bytes;
  // workspace layout (byte offsets)
  int64_t ws_status, ws_streams, ws_heads, ws_packed, ws_slots, ws_sizes, ws_scan;
  int64_t ws_fix;       // fused Hadamard encode: fixup row list (count + rows), or -1
  int64_t ws_delta;     // chunked delta decode: chunk sums / carries / head flags, or -1
  int64_t slot_bytes;   // per-block scratch slot for entropy/rle encode
  int64_t scan_bytes;
  int sm_count;
};

}  // namespace kvc
