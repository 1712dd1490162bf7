/* Exhaustive-over-scales check that the reciprocal+FMA quotient used by the
 * CUDA quantizer (numerics.cuh quant_magic) yields the same clipped rint as
 * the IEEE fp32 quotient of quantize.py:152, for every positive finite fp16
 * scale, on random and adversarial dividends with |d| <= 2^24 (always true
 * when the group's fp16 scale and zero are finite; infinite ones take the
 * exact slow path).  Build: gcc -O2 -ffp-contract=off markstein_check.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static float h2f(uint16_t h) {
  uint32_t s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
  float v = e == 0 ? ldexpf((float)m, -24) : ldexpf((float)(m | 1024), (int)e - 25);
  return s ? -v : v;
}
static uint64_t st = 88172645463325252ull;
static uint64_t rnd(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }

int main(void) {
  long bad = 0, total = 0, badsym = 0;
  for (uint32_t h = 1; h < 0x7C00; ++h) {
    float s = h2f((uint16_t)h);
    float r = 1.0f / s; /* correctly rounded reciprocal (__frcp_rn) */
    for (int k = 0; k < 4000; ++k) {
      float d;
      uint64_t u = rnd();
      int mode = k % 4;
      if (mode == 0) d = s * (float)(u % 70000) / 256.0f;        /* typical range */
      else if (mode == 1) {                                       /* near half-integers */
        d = ((float)(u % 512) + 0.5f) * s;
        uint32_t b; memcpy(&b, &d, 4); b += (int)((u >> 20) % 9) - 4; memcpy(&d, &b, 4);
      } else if (mode == 2) {                                     /* any magnitude up to 2^24 */
        uint32_t b = (uint32_t)(u >> 11); memcpy(&d, &b, 4);
        if (!isfinite(d)) d = 1.0f;
        d = fminf(fabsf(d), 16777216.0f);
      } else d = s * 255.0f * (float)((u >> 8) & 0xFFFFFF) / 16777216.0f;
      if (u & (1ull << 40)) d = -d * 0.01f;                         /* negative residues */
      float q0 = d * r;
      float e = fmaf(-q0, s, d);
      float q1 = fmaf(e, r, q0);
      float ex = d / s;
      total++;
      for (int lv = 1; lv <= 255; lv = 2 * lv + 1) {
        float a = rintf(fminf(fmaxf(q1, 0.f), (float)lv)), b = rintf(fminf(fmaxf(ex, 0.f), (float)lv));
        if (a != b) { badsym++; if (badsym < 5) printf("sym mismatch s=%a d=%a lv=%d\n", s, d, lv); }
      }
      if (fabsf(ex) < 256.0f && fabsf(d) > 0x1p-100f && memcmp(&q1, &ex, 4) != 0) bad++;
    }
  }
  printf("checked %ld (scale, dividend) pairs x 8 widths: quotient mismatches (|q|<256, |d|>2^-100) %ld, "
         "clipped-rint symbol mismatches %ld\n", total, bad, badsym);
  return (badsym != 0) || (bad != 0);
}
