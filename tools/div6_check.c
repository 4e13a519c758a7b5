#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s64 = 88172645463325252ull;
static inline uint64_t xr(void){ s64 ^= s64<<13; s64 ^= s64>>7; s64 ^= s64<<17; return s64; }
int main(void){
  const double y = 6.0, yi = 1.0/6.0;
  long bad = 0, n = 0;
  for (long k = 0; k < 400000000L; ++k) {
    uint64_t b = xr();
    uint64_t e = 1 + (xr() % 2045);         /* all normal exponents */
    b = (b & 0x800fffffffffffffull) | (e << 52);
    double s; memcpy(&s, &b, 8);
    double q0 = s * yi;
    double r = fma(-q0, y, s);
    double q1 = fma(r, yi, q0);
    double q = s / y;
    if (fabs(q) >= 0x1p-1022 && memcmp(&q, &q1, 8) != 0) { if (bad < 5) printf("bad s=%a q=%a q1=%a\n", s, q, q1); ++bad; }
    ++n;
  }
  /* subnormal and tiny inputs */
  for (long k = 0; k < 100000000L; ++k) {
    uint64_t b = xr() & 0x801fffffffffffffull;   /* exponent field 0 or 1 */
    double s; memcpy(&s, &b, 8);
    double q0 = s * yi, r = fma(-q0, y, s), q1 = fma(r, yi, q0), q = s / y;
    if (fabs(q) >= 0x1p-1022 && memcmp(&q, &q1, 8) != 0) { if (bad < 10) printf("bad(sub) s=%a q=%a q1=%a\n", s, q, q1); ++bad; }
    ++n;
  }
  printf("f64: %ld / %ld mismatches\n", bad, n);
  /* f32 exhaustive over all non-negative finite floats */
  const float yf = 6.0f, yif = 1.0f/6.0f; long badf = 0;
  for (uint32_t u = 0; u < 0x7f800000u; ++u) {
    float s; memcpy(&s, &u, 4);
    float q0 = s * yif, r = fmaf(-q0, yf, s), q1 = fmaf(r, yif, q0), q = s / yf;
    if (fabsf(q) >= 0x1p-126f && memcmp(&q, &q1, 4) != 0) { if (badf < 5) printf("badf s=%a q=%a q1=%a\n", s, q, q1); ++badf; }
  }
  printf("f32 exhaustive: %ld mismatches\n", badf);
  return 0;
}
