/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product library.
 *
 * Plain-C restatement of the reference's serial lossless codecs, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker for the CUDA kernels.  Follows:
 *   - range coder constants        pkg/src/kvpilot/pipeline/codecs.py:181-185
 *   - adaptive order-0 model       pkg/src/kvpilot/pipeline/codecs.py:188-242
 *   - encoder / renormalisation    pkg/src/kvpilot/pipeline/codecs.py:245-270
 *   - decoder                      pkg/src/kvpilot/pipeline/codecs.py:273-307
 *   - range_encode/range_decode    pkg/src/kvpilot/pipeline/codecs.py:310-331
 *   - PackBits-style RLE           pkg/src/kvpilot/pipeline/codecs.py:107-174
 *
 * The reference uses unbounded Python ints; `low + range` can reach exactly
 * 2^32, so every such sum is evaluated in 64 bits here.  The frequency model
 * is kept as a flat array: the Fenwick tree in the reference is only an
 * accelerator for prefix sums / searches and does not change any value.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>

#define RC_TOP (1u << 24)
#define RC_BOT (1u << 16)
#define FREQ_STEP 32u
#define FREQ_LIMIT (1u << 16)
#define MAX_ALPHA 65536

typedef struct {
  uint32_t alpha;
  uint32_t total;
  uint32_t* freq;
} model_t;

static int model_init(model_t* m, uint32_t alpha) {
  m->alpha = alpha;
  m->total = alpha;
  m->freq = (uint32_t*)malloc(sizeof(uint32_t) * (alpha ? alpha : 1));
  if (!m->freq) return -1;
  for (uint32_t s = 0; s < alpha; ++s) m->freq[s] = 1;
  return 0;
}

static uint32_t model_cum(const model_t* m, uint32_t s) {
  uint32_t c = 0;
  for (uint32_t i = 0; i < s; ++i) c += m->freq[i];
  return c;
}

/* symbol s with cum(s) <= target < cum(s+1); target < 0 maps to 0 like the
 * reference's Fenwick search (codecs.py:214-225). */
static uint32_t model_find(const model_t* m, int64_t target) {
  if (target < 0) return 0;
  uint64_t c = 0;
  for (uint32_t s = 0; s < m->alpha; ++s) {
    c += m->freq[s];
    if ((int64_t)c > target) return s;
  }
  return m->alpha; /* unreachable for target < total */
}

static void model_bump(model_t* m, uint32_t s) {
  m->freq[s] += FREQ_STEP;
  m->total += FREQ_STEP;
  if (m->total >= FREQ_LIMIT) {
    uint32_t t = 0;
    for (uint32_t i = 0; i < m->alpha; ++i) {
      uint32_t h = m->freq[i] >> 1;
      m->freq[i] = h ? h : 1;
      t += m->freq[i];
    }
    m->total = t;
  }
}

/* returns coded length, or -1 when `cap` is too small / bad args */
long oc_range_encode(const uint16_t* sym, size_t n, uint32_t alpha, uint8_t* out, size_t cap) {
  if (alpha < 1 || alpha > MAX_ALPHA) return -1;
  model_t m;
  if (model_init(&m, alpha)) return -1;
  uint32_t low = 0, range = 0xFFFFFFFFu;
  size_t pos = 0;
  for (size_t i = 0; i < n; ++i) {
    uint32_t s = sym[i];
    if (s >= alpha) { free(m.freq); return -1; }
    uint32_t unit = range / m.total;
    low += unit * model_cum(&m, s);
    range = unit * m.freq[s];
    for (;;) {
      uint64_t hi = (uint64_t)low + (uint64_t)range;
      if (((uint64_t)low ^ hi) < RC_TOP) {
      } else if (range < RC_BOT) {
        range = (0u - low) & (RC_BOT - 1);
      } else {
        break;
      }
      if (pos >= cap) { free(m.freq); return -1; }
      out[pos++] = (uint8_t)(low >> 24);
      low <<= 8;
      range <<= 8;
    }
    model_bump(&m, s);
  }
  for (int k = 0; k < 4; ++k) {
    if (pos >= cap) { free(m.freq); return -1; }
    out[pos++] = (uint8_t)(low >> 24);
    low <<= 8;
  }
  free(m.freq);
  return (long)pos;
}

/* 0 on success, -1 truncated stream (CodecError in the reference), -2 bad args */
int oc_range_decode(const uint8_t* data, size_t len, uint32_t alpha, size_t count, uint16_t* out) {
  if (alpha < 1 || alpha > MAX_ALPHA) return -2;
  model_t m;
  if (model_init(&m, alpha)) return -2;
  size_t pos = 0;
  uint32_t low = 0, range = 0xFFFFFFFFu, code = 0;
  for (int k = 0; k < 4; ++k) {
    if (pos >= len) { free(m.freq); return -1; }
    code = (code << 8) | data[pos++];
  }
  for (size_t i = 0; i < count; ++i) {
    uint32_t unit = range / m.total;
    int64_t diff = (int64_t)code - (int64_t)low;
    int64_t q = diff >= 0 ? diff / unit : -((-diff + unit - 1) / unit); /* floor division */
    int64_t target = q < (int64_t)m.total - 1 ? q : (int64_t)m.total - 1;
    uint32_t s = model_find(&m, target);
    low += unit * model_cum(&m, s);
    range = unit * m.freq[s];
    for (;;) {
      uint64_t hi = (uint64_t)low + (uint64_t)range;
      if (((uint64_t)low ^ hi) < RC_TOP) {
      } else if (range < RC_BOT) {
        range = (0u - low) & (RC_BOT - 1);
      } else {
        break;
      }
      if (pos >= len) { free(m.freq); return -1; }
      code = (code << 8) | data[pos++];
      low <<= 8;
      range <<= 8;
    }
    model_bump(&m, s);
    out[i] = (uint16_t)s;
  }
  free(m.freq);
  return 0;
}

/* ---------------------------------------------------------------- RLE */

static long emit_literal(const uint8_t* in, size_t from, size_t upto, uint8_t* out, size_t pos, size_t cap) {
  while (from < upto) {
    size_t chunk = upto - from < 128 ? upto - from : 128;
    if (pos + 1 + chunk > cap) return -1;
    out[pos++] = (uint8_t)(chunk - 1);
    memcpy(out + pos, in + from, chunk);
    pos += chunk;
    from += chunk;
  }
  return (long)pos;
}

/* returns encoded length or -1 when cap is too small */
long oc_rle_encode(const uint8_t* in, size_t n, uint8_t* out, size_t cap) {
  size_t pos = 0;
  size_t i = 0;
  int have_lit = 0;
  size_t lit_from = 0;
  while (i < n) {
    size_t j = i + 1;
    while (j < n && in[j] == in[i]) ++j;
    size_t run = j - i;
    if (run >= 3) {
      if (have_lit) {
        long r = emit_literal(in, lit_from, i, out, pos, cap);
        if (r < 0) return -1;
        pos = (size_t)r;
        have_lit = 0;
      }
      while (run >= 3) {
        size_t chunk = run < 130 ? run : 130;
        if (pos + 2 > cap) return -1;
        out[pos++] = (uint8_t)(128 + chunk - 3);
        out[pos++] = in[i];
        run -= chunk;
      }
      if (run) {
        have_lit = 1;
        lit_from = j - run;
      }
    } else if (!have_lit) {
      have_lit = 1;
      lit_from = i;
    }
    i = j;
  }
  if (have_lit) {
    long r = emit_literal(in, lit_from, n, out, pos, cap);
    if (r < 0) return -1;
    pos = (size_t)r;
  }
  return (long)pos;
}

/* returns decoded length; -1 truncated literal, -2 truncated repeat, -3 cap */
long oc_rle_decode(const uint8_t* in, size_t n, uint8_t* out, size_t cap) {
  size_t pos = 0, o = 0;
  while (pos < n) {
    uint8_t c = in[pos++];
    if (c < 128) {
      size_t len = (size_t)c + 1;
      if (pos + len > n) return -1;
      if (o + len > cap) return -3;
      memcpy(out + o, in + pos, len);
      o += len;
      pos += len;
    } else {
      if (pos >= n) return -2;
      size_t len = (size_t)c - 128 + 3;
      if (o + len > cap) return -3;
      memset(out + o, in[pos], len);
      o += len;
      pos += 1;
    }
  }
  return (long)o;
}

/* ------------------------------------------------- batched block framing
 * Block framing used by the GPU codec: a width stream is cut
 * into blocks of `block` symbols; each block's entropy payload is
 * BE32(len) || range_encode(block symbols)  (the reference's per-stream
 * framing, codecs.py:362-366, applied per block).  These batch entry points
 * exist so the CPU baseline can use every host core (pthreads).          */
#include <pthread.h>

typedef struct {
  int mode; /* 0 encode, 1 decode */
  const uint16_t* sym_in; uint16_t* sym_out;
  const uint8_t* payload; const uint64_t* offsets;
  uint8_t* out; size_t cap_per_block; uint64_t* sizes;
  size_t n, block, nb; uint32_t alpha;
  long next; long bad; pthread_mutex_t mu;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    long b0 = j->next; j->next += 16;
    pthread_mutex_unlock(&j->mu);
    if (b0 >= (long)j->nb) break;
    long b1 = b0 + 16 < (long)j->nb ? b0 + 16 : (long)j->nb;
    long bad = 0;
    for (long b = b0; b < b1; ++b) {
      size_t s0 = (size_t)b * j->block, cnt = j->n - s0 < j->block ? j->n - s0 : j->block;
      if (j->mode == 0) {
        uint8_t* dst = j->out + (size_t)b * j->cap_per_block;
        long r = oc_range_encode(j->sym_in + s0, cnt, j->alpha, dst + 4, j->cap_per_block - 4);
        if (r < 0) { bad++; j->sizes[b] = 0; continue; }
        dst[0] = (uint8_t)(r >> 24); dst[1] = (uint8_t)(r >> 16); dst[2] = (uint8_t)(r >> 8); dst[3] = (uint8_t)r;
        j->sizes[b] = (uint64_t)r + 4;
      } else {
        const uint8_t* src = j->payload + j->offsets[b];
        uint64_t avail = j->offsets[b + 1] - j->offsets[b];
        if (avail < 4) { bad++; continue; }
        uint64_t len = ((uint64_t)src[0] << 24) | ((uint64_t)src[1] << 16) | ((uint64_t)src[2] << 8) | src[3];
        if (len + 4 != avail || oc_range_decode(src + 4, len, j->alpha, cnt, j->sym_out + s0) != 0) bad++;
      }
    }
    if (bad) { pthread_mutex_lock(&j->mu); j->bad += bad; pthread_mutex_unlock(&j->mu); }
  }
  return NULL;
}

static long run_job(job_t* j, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  pthread_mutex_init(&j->mu, NULL);
  j->next = 0; j->bad = 0;
  int started = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tid[started], NULL, worker, j) == 0) started++;
  worker(j);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  pthread_mutex_destroy(&j->mu);
  return j->bad ? -1 : (long)j->nb;
}

long oc_entropy_encode_blocks(const uint16_t* sym, size_t n, uint32_t alpha, size_t block,
                              uint8_t* out, size_t cap_per_block, uint64_t* sizes, int threads) {
  if (block == 0) return -1;
  job_t j; memset(&j, 0, sizeof j);
  j.mode = 0; j.sym_in = sym; j.n = n; j.alpha = alpha; j.block = block;
  j.nb = n ? (n + block - 1) / block : 0; j.out = out; j.cap_per_block = cap_per_block; j.sizes = sizes;
  return run_job(&j, threads);
}

long oc_entropy_decode_blocks(const uint8_t* payload, const uint64_t* offsets, size_t n, uint32_t alpha,
                              size_t block, uint16_t* sym, int threads) {
  if (block == 0) return -1;
  job_t j; memset(&j, 0, sizeof j);
  j.mode = 1; j.payload = payload; j.offsets = offsets; j.n = n; j.alpha = alpha; j.block = block;
  j.nb = n ? (n + block - 1) / block : 0; j.sym_out = sym;
  return run_job(&j, threads);
}
