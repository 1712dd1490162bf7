/* The drop-in boundary used from plain C: no Python, no torch.  Builds
 * against include/kvc.h and libkvc.so only (plus the CUDA runtime for device
 * buffers), the way a serving engine or another language's FFI would.
 *
 * For each strategy: plan -> sizes -> encode -> status -> payload length
 * (static, or block_offsets[nblocks] read back) -> decode -> status; the
 * round trip must stay within the strategy's quantization error, encode must
 * be deterministic, decoding a truncated payload must report the codec flag,
 * and a bad strategy id must fail with a message.  Prints "abi ok".
 *
 *   nvcc -o abi tests/c/abi_roundtrip.c -Iinclude -Lpaper_2605_13734_b200 -lkvc
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "kvc.h"

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)
#define KV(x)                                                                        \
  do {                                                                               \
    int r_ = (x);                                                                    \
    if (r_ != KVC_OK) {                                                              \
      fprintf(stderr, "%s:%d kvc status %d: %s\n", __FILE__, __LINE__, r_, kvc_last_error()); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

static uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u); /* round to nearest even */
  return (uint16_t)(u >> 16);
}
static float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static double gauss(unsigned* s) {
  double u1, u2;
  *s = *s * 1664525u + 1013904223u;
  u1 = ((*s >> 8) + 1.0) / 16777217.0;
  *s = *s * 1664525u + 1013904223u;
  u2 = ((*s >> 8) + 1.0) / 16777217.0;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static int roundtrip(const char* sid, double tol) {
  const int64_t L = 2, H = 4, T = 512, C = 128, E = L * H * T * C;
  kvc_plan* plan = NULL;
  KV(kvc_plan_create(&plan, sid, L, H, T, C, NULL));
  const int64_t meta_b = kvc_metadata_bytes(plan), cap = kvc_payload_capacity(plan);
  const int64_t ws_b = kvc_workspace_bytes(plan), maxb = kvc_max_blocks(plan);
  uint16_t* h_kv = (uint16_t*)malloc(E * 2);
  uint16_t* h_out = (uint16_t*)malloc(E * 2);
  unsigned seed = 12345u;
  for (int64_t i = 0; i < E; ++i) h_kv[i] = f32_to_bf16((float)gauss(&seed));
  void *d_kv, *d_out, *d_pay, *d_pay2, *d_meta, *d_ws;
  uint64_t* d_off;
  CK(cudaMalloc(&d_kv, E * 2));
  CK(cudaMalloc(&d_out, E * 2));
  CK(cudaMalloc(&d_pay, cap));
  CK(cudaMalloc(&d_pay2, cap));
  CK(cudaMalloc(&d_meta, meta_b > 0 ? meta_b : 1));
  CK(cudaMalloc(&d_ws, ws_b));
  CK(cudaMalloc((void**)&d_off, 8 * (maxb + 1)));
  CK(cudaMemcpy(d_kv, h_kv, E * 2, cudaMemcpyHostToDevice));

  KV(kvc_encode(plan, d_kv, NULL, d_pay, d_meta, d_off, d_ws, NULL));
  uint32_t flags = 0;
  KV(kvc_read_status(plan, d_ws, NULL, &flags));
  if (flags) {
    fprintf(stderr, "%s: encode flags %u\n", sid, flags);
    return 1;
  }
  int64_t nbytes = kvc_static_payload_bytes(plan, NULL);
  const int64_t nblocks = kvc_num_blocks(plan, NULL);
  if (nbytes < 0) {
    uint64_t last = 0;
    CK(cudaMemcpy(&last, d_off + nblocks, 8, cudaMemcpyDeviceToHost));
    nbytes = (int64_t)last;
  }
  /* deterministic: a second encode gives the same bytes */
  KV(kvc_encode(plan, d_kv, NULL, d_pay2, d_meta, d_off, d_ws, NULL));
  unsigned char* a = (unsigned char*)malloc(nbytes);
  unsigned char* b = (unsigned char*)malloc(nbytes);
  CK(cudaMemcpy(a, d_pay, nbytes, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b, d_pay2, nbytes, cudaMemcpyDeviceToHost));
  if (memcmp(a, b, nbytes) != 0) {
    fprintf(stderr, "%s: encode not deterministic\n", sid);
    return 1;
  }

  KV(kvc_decode(plan, d_pay, nbytes, d_meta, d_off, d_out, d_ws, NULL));
  KV(kvc_read_status(plan, d_ws, NULL, &flags));
  if (flags) {
    fprintf(stderr, "%s: decode flags %u\n", sid, flags);
    return 1;
  }
  CK(cudaMemcpy(h_out, d_out, E * 2, cudaMemcpyDeviceToHost));
  double se = 0.0, sx = 0.0;
  for (int64_t i = 0; i < E; ++i) {
    const double x = bf16_to_f32(h_kv[i]), y = bf16_to_f32(h_out[i]);
    se += (x - y) * (x - y);
    sx += x * x;
  }
  const double rel = sqrt(se / sx);
  if (!(rel < tol)) {
    fprintf(stderr, "%s: relative rmse %g >= %g\n", sid, rel, tol);
    return 1;
  }
  /* a truncated payload is a codec error (codecs.py trailing / truncation rules) */
  KV(kvc_decode(plan, d_pay, nbytes - 1, d_meta, d_off, d_out, d_ws, NULL));
  KV(kvc_read_status(plan, d_ws, NULL, &flags));
  if (!(flags & KVC_FLAG_CODEC)) {
    fprintf(stderr, "%s: truncated payload not reported (flags %u)\n", sid, flags);
    return 1;
  }
  printf("%-45s encode=%-14s decode=%-12s payload=%lld B rel_rmse=%.4f\n", kvc_plan_strategy_id(plan),
         kvc_plan_encode_path(plan), kvc_plan_decode_path(plan), (long long)nbytes, rel);
  free(a);
  free(b);
  free(h_kv);
  free(h_out);
  cudaFree(d_kv);
  cudaFree(d_out);
  cudaFree(d_pay);
  cudaFree(d_pay2);
  cudaFree(d_meta);
  cudaFree(d_ws);
  cudaFree(d_off);
  KV(kvc_plan_destroy(plan));
  return 0;
}

int main(void) {
  kvc_plan* bad = NULL;
  if (kvc_plan_create(&bad, "t=hadamard;q=uniform,b=9,g=32;c=none", 1, 1, 8, 128, NULL) != KVC_ERR_CONFIG ||
      strlen(kvc_last_error()) == 0) {
    fprintf(stderr, "bad strategy id accepted\n");
    return 1;
  }
  printf("libkvc %s\n", kvc_version());
  int fails = 0;
  fails += roundtrip("t=hadamard;q=uniform,b=4,g=32;c=none", 0.15);
  fails += roundtrip("t=identity;q=uniform,b=2,g=32;c=entropy", 0.45);
  fails += roundtrip("t=identity;q=uchan,b=2,g=32;c=entropy", 0.45);
  fails += roundtrip("t=affine;q=uniform,b=8,g=32;c=entropy", 0.02);
  fails += roundtrip("t=identity;q=uniform,b=4,g=64;c=rle", 0.2);
  /* delta: quantization errors accumulate along the tokens of i.i.d. data */
  fails += roundtrip("t=delta;q=uniform,b=8,g=32;c=none", 1.0);
  if (fails) return 1;
  printf("abi ok\n");
  return 0;
}
