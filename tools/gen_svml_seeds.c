/* Generate paper_2509_20081_b200/csrc/svml_seeds.bin: the exact outputs of
 * the AVX-512 approximation instructions VRCP14PD and VRSQRT14PD, which seed
 * numpy's SVML atan2/asin (__svml_atan28_ha, __svml_asin8_ha). Measured facts
 * this file relies on (asserted below, on Sapphire Rapids):
 *   rcp14(2^e * 1.m)   depends only on e and the top 16 mantissa bits;
 *                      = 2^-e * rcp14(1.m); result mantissa has 16 bits;
 *                      exponent 0 for m == 0 else -1.
 *   rsqrt14(2^(2k+p) * 1.m) depends only on p and the top 15 mantissa bits;
 *                      = 2^-k * rsqrt14(2^p * 1.m); 16-bit result mantissa;
 *                      exponent 0 for p == 0 && m == 0 else -1.
 * Layout: uint16 rcp[65536] (index m16), uint16 rsqrt[65536] (index p*32768+m15),
 * little endian, each the top 16 bits of the result mantissa.
 * Build: gcc -O2 -mavx512f tools/gen_svml_seeds.c -o /tmp/gen && /tmp/gen out.bin */
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static double rcp14(double x) { double o[8]; _mm512_storeu_pd(o, _mm512_rcp14_pd(_mm512_set1_pd(x))); return o[0]; }
static double rsq14(double x) { double o[8]; _mm512_storeu_pd(o, _mm512_rsqrt14_pd(_mm512_set1_pd(x))); return o[0]; }
static uint64_t B(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double F(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

int main(int argc, char** argv) {
  static uint16_t tab[131072];
  for (uint64_t m = 0; m < 65536; ++m) {
    uint64_t r = B(rcp14(F((1023ull << 52) | (m << 36))));
    int ex = (int)(r >> 52) - 1023;
    if ((r & ((1ull << 36) - 1)) || ex != (m == 0 ? 0 : -1)) { fprintf(stderr, "rcp14 rule violated at %llu\n", (unsigned long long)m); return 1; }
    tab[m] = (uint16_t)((r >> 36) & 0xFFFF);
  }
  for (uint64_t p = 0; p < 2; ++p)
    for (uint64_t m = 0; m < 32768; ++m) {
      uint64_t r = B(rsq14(F(((1023ull + p) << 52) | (m << 37))));
      int ex = (int)(r >> 52) - 1023;
      if ((r & ((1ull << 36) - 1)) || ex != ((p == 0 && m == 0) ? 0 : -1)) { fprintf(stderr, "rsqrt14 rule violated\n"); return 1; }
      tab[65536 + p * 32768 + m] = (uint16_t)((r >> 36) & 0xFFFF);
    }
  FILE* f = fopen(argc > 1 ? argv[1] : "svml_seeds.bin", "wb");
  if (!f || fwrite(tab, 2, 131072, f) != 131072) { perror("write"); return 1; }
  fclose(f);
  return 0;
}
