/* Check of div6's integer path for tiny quotients (development aid, CPU):
 * for |s| below the FMA path's range (0x1.8p-1020 f64, 0x1.8p-124 f32) s is
 * an integer k of units 2^-1074 (2^-149); RN(s/6) is then k/6 rounded to
 * nearest-even in the same units, which is the bit pattern of the (subnormal
 * or smallest-normal) result.  Compared with the IEEE division: f32
 * exhaustive over the tiny range, f64 every k < 2^24 plus 5e8 random tiny
 * values.  gcc -O2 -o /tmp/d6t tools/div6_tiny_check.c && /tmp/d6t */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static uint64_t s64 = 88172645463325252ull;
static inline uint64_t xr(void) { s64 ^= s64 << 13; s64 ^= s64 >> 7; s64 ^= s64 << 17; return s64; }

static double div6_tiny(double s) {
  uint64_t b; memcpy(&b, &s, 8);
  const uint64_t sign = b & 0x8000000000000000ull, a = b & ~0x8000000000000000ull;
  const uint64_t E = a >> 52, m = a & 0xfffffffffffffull;
  const uint64_t k = E == 0 ? m : ((0x10000000000000ull | m) << (E - 1));
  uint64_t q = k / 6;
  const uint64_t r = k - 6 * q;
  if (r > 3 || (r == 3 && (q & 1))) ++q;
  const uint64_t o = sign | q;
  double d; memcpy(&d, &o, 8);
  return d;
}
static float div6_tiny_f(float s) {
  uint32_t b; memcpy(&b, &s, 4);
  const uint32_t sign = b & 0x80000000u, a = b & 0x7fffffffu;
  const uint32_t E = a >> 23, m = a & 0x7fffffu;
  const uint32_t k = E == 0 ? m : ((0x800000u | m) << (E - 1));
  uint32_t q = k / 6;
  const uint32_t r = k - 6 * q;
  if (r > 3 || (r == 3 && (q & 1))) ++q;
  const uint32_t o = sign | q;
  float d; memcpy(&d, &o, 4);
  return d;
}

int main(void) {
  long bad = 0, n = 0;
  const double lim = 0x1.8p-1020;
  uint64_t lb; memcpy(&lb, &lim, 8);
  for (uint64_t k = 0; k < (1ull << 24); ++k) {
    for (int sg = 0; sg < 2; ++sg) {
      uint64_t b = k | (sg ? 0x8000000000000000ull : 0);
      double s; memcpy(&s, &b, 8);
      double q = s / 6.0, t = div6_tiny(s);
      if (memcmp(&q, &t, 8)) { if (bad < 5) printf("bad s=%a q=%a t=%a\n", s, q, t); ++bad; }
      ++n;
    }
  }
  for (long i = 0; i < 500000000L; ++i) {
    uint64_t b = xr() % lb;
    if (i & 1) b |= 0x8000000000000000ull;
    double s; memcpy(&s, &b, 8);
    double q = s / 6.0, t = div6_tiny(s);
    if (memcmp(&q, &t, 8)) { if (bad < 10) printf("bad s=%a q=%a t=%a\n", s, q, t); ++bad; }
    ++n;
  }
  printf("f64 tiny path: %ld / %ld mismatches\n", bad, n);
  long badf = 0, nf = 0;
  const float limf = 0x1.8p-124f;
  uint32_t lf; memcpy(&lf, &limf, 4);
  for (uint32_t u = 0; u < lf; ++u) {
    for (int sg = 0; sg < 2; ++sg) {
      uint32_t b = u | (sg ? 0x80000000u : 0);
      float s; memcpy(&s, &b, 4);
      float q = s / 6.0f, t = div6_tiny_f(s);
      if (memcmp(&q, &t, 4)) { if (badf < 5) printf("badf s=%a q=%a t=%a\n", s, q, t); ++badf; }
      ++nf;
    }
  }
  printf("f32 tiny path (exhaustive): %ld / %ld mismatches\n", badf, nf);
  return (bad || badf) ? 1 : 0;
}
