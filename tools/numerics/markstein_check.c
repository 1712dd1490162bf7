/* Exhaustive-over-scales check that the reciprocal+FMA quotient used by the
 * CUDA quantizer equals the IEEE fp32 quotient (quantize.py:152) for every
 * positive finite fp16 scale, on random and adversarial dividends. */
#include <stdio.h>
#include <stdint.h>
#include <math.h>
#include <string.h>
static float h2f(uint16_t h) {
  uint32_t s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
  float v;
  if (e == 0) v = ldexpf((float)m, -24);
  else v = ldexpf((float)(m | 1024), (int)e - 25);
  return s ? -v : v;
}
static uint64_t st = 88172645463325252ull;
static uint64_t rnd(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
int main(void) {
  long bad = 0, total = 0, badrint = 0;
  for (uint32_t h = 1; h < 0x7C00; ++h) {
    float s = h2f((uint16_t)h);
    float r = 1.0f / s; /* correctly rounded reciprocal */
    for (int k = 0; k < 4000; ++k) {
      float d;
      uint64_t u = rnd();
      int mode = k % 4;
      if (mode == 0) d = s * (float)(u % 70000) / 256.0f;                        /* typical range */
      else if (mode == 1) { float kk = (float)(u % 512) + 0.5f; d = kk * s;        /* near half-integers */
        uint32_t b; memcpy(&b, &d, 4); b += (int)((u >> 20) % 9) - 4; memcpy(&d, &b, 4); }
      else if (mode == 2) { uint32_t b = (uint32_t)(u >> 11); memcpy(&d, &b, 4); if (!isfinite(d)) d = 1.0f; d = fabsf(d); }
      else d = s * 255.0f * (float)((u >> 8) & 0xFFFFFF) / 16777216.0f;
      float q0 = fminf(d * r, 512.0f); /* clamp first: keeps the residual finite */
      float e = fmaf(-q0, s, d);
      float q1 = fmaf(e, r, q0);
      float ex = d / s;
      total++;
      if (rintf(fminf(fmaxf(q1, 0.f), 255.f)) != rintf(fminf(fmaxf(ex, 0.f), 255.f))) { badrint++; if (badrint < 5) printf("sym mismatch s=%a d=%a\n", s, d); }
      if (ex < 256.0f && d > 0x1p-100f && memcmp(&q1, &ex, 4) != 0) {
        bad++;
        if (bad < 10) printf("mismatch s=%a d=%a q1=%a ex=%a\n", s, d, q1, ex);
      }
    }
  }
  printf("checked %ld, quotient mismatches (d>2^-100, q<256) %ld, clamped-rint symbol mismatches %ld\n", total, bad, badrint);
  return (badrint != 0) || (bad != 0);
}
