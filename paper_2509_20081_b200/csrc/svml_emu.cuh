// svml_emu.cuh — bit-exact restatement of the two transcendental routines the
// reference's binning calls through numpy (kernels.py:49-57: np.arctan2,
// np.arcsin). numpy 2.3.5 dispatches float64 arctan2/arcsin on AVX512_SKX
// hosts (both the build container and the B200 box: Sapphire Rapids) to its
// vendored Intel SVML routines __svml_atan28_ha and __svml_asin8_ha
// (numpy/SVML, BSD-3). This file restates their per-lane algorithm: the same
// IEEE double operations (every mul/add/fma round-to-nearest, same order, same
// constants) so the device produces the identical bits numpy produces.
//
// The only non-IEEE steps in those routines are the AVX-512 approximation
// instructions VRCP14PD (atan2) and VRSQRT14PD (asin) that seed a Newton
// refinement. Their outputs depend only on the exponent and the top 16 / 15
// mantissa bits; svml_seeds.bin (generated from the instructions by
// tools/gen_svml_seeds.c) holds the 16-bit result mantissas.
//
// Scope: finite inputs. atan2 lanes SVML routes to its scalar "rare" helper
// (a nonzero component below 2^-1020 or above 2^993, NaN, inf) set *rare and
// the caller decides; x == 0 or y == 0 is handled exactly like SVML's vector
// special path. asin is restated for |x| <= 1 (the reference clips to
// [-1, 1]).
//
// License: the restated routines are BSD-3 (Intel SVML via numpy); see
// NOTICE.svml next to this file.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SVE_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define SVE_HD static inline
#endif

namespace svml {

#ifdef __CUDA_ARCH__
SVE_HD uint64_t bits(double d) { return (uint64_t)__double_as_longlong(d); }
SVE_HD double dbl(uint64_t u) { return __longlong_as_double((long long)u); }
SVE_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
SVE_HD double mul(double a, double b) { return __dmul_rn(a, b); }
SVE_HD double add(double a, double b) { return __dadd_rn(a, b); }
SVE_HD double sub(double a, double b) { return __dsub_rn(a, b); }
#else
SVE_HD uint64_t bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
SVE_HD double dbl(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
SVE_HD double fma_(double a, double b, double c) { return fma(a, b, c); }
SVE_HD double mul(double a, double b) { return a * b; }  // host TU built with -ffp-contract=off
SVE_HD double add(double a, double b) { return a + b; }
SVE_HD double sub(double a, double b) { return a - b; }
#endif

constexpr uint64_t kSign = 0x8000000000000000ull;
constexpr uint64_t kAbs = 0x7fffffffffffffffull;

// VRCP14PD for a positive normal x (seed table: uint16[65536] by top 16 bits)
SVE_HD double rcp14(double x, const uint16_t* tab) {
  const uint64_t u = bits(x);
  const int e = (int)((u >> 52) & 0x7FF) - 1023;
  const uint32_t m = (uint32_t)((u >> 36) & 0xFFFF);
  const int re = (m == 0 ? 0 : -1) - e;
  return dbl(((uint64_t)(re + 1023) << 52) | ((uint64_t)tab[m] << 36));
}

// VRSQRT14PD for a positive normal x (seed table: uint16[65536] by exponent
// parity and top 15 bits)
SVE_HD double rsqrt14(double x, const uint16_t* tab) {
  const uint64_t u = bits(x);
  const int e = (int)((u >> 52) & 0x7FF) - 1023;
  const int p = e & 1;
  const int k = (e - p) / 2;
  const uint32_t m = (uint32_t)((u >> 37) & 0x7FFF);
  const int re = ((p == 0 && m == 0) ? 0 : -1) - k;
  return dbl(((uint64_t)(re + 1023) << 52) | ((uint64_t)tab[65536 + p * 32768 + m] << 36));
}

// ---- __svml_atan28_ha (y, x), constants from __svml_datan2_ha_data_internal
SVE_HD double atan2(double y, double x, const uint16_t* rcp_tab, int* rare) {
  const uint64_t bx = bits(x), by = bits(y);
  const uint64_t sgnx = bx & kSign, sgny = by & kSign;
  const double ax = dbl(bx & kAbs), ay = dbl(by & kAbs);
  const bool xneg = x < 0.0;  // ordered compare with +0.0
  const uint32_t hx = (uint32_t)((bx & kAbs) >> 32), hy = (uint32_t)((by & kAbs) >> 32);
  const bool spx = (int32_t)(hx - 0x80300000u) >= (int32_t)0xfdd00000u;
  const bool spy = (int32_t)(hy - 0x80300000u) >= (int32_t)0xfdd00000u;
  *rare = 0;
  if (spx || spy) {
    // vector special path: a zero component (no NaN) -> exact constant
    const bool nan = (x != x) || (y != y);
    if (!nan && (ax == 0.0 || ay == 0.0)) {
      double base = (ay < ax) ? 0.0 : 1.5707963267948966;  // pi/2
      if (ax == 0.0 && ay == 0.0) base = 0.0;
      double v = dbl(bits(base) | sgnx);
      if (sgnx) v = add(v, 3.141592653589793);  // pi
      return dbl(bits(v) | sgny);
    }
    *rare = 1;  // tiny/huge nonzero, NaN, inf: SVML's scalar helper
    return 0.0;
  }
  const bool k5 = mul(ax, 0.4375) < ay;
  const bool k1 = mul(ax, 0.6875) < ay;
  const bool k2 = mul(ax, 1.1875) < ay;
  const bool k3 = mul(ax, 2.4375) < ay;
  double c = k1 ? 1.0 : 0.5;
  double hi = k1 ? dbl(0x3fe921fb54442d18ull) : dbl(0x3fddac670561bb4full);  // atan(1), atan(.5)
  double lo = k1 ? dbl(0x3c81a62633145c07ull) : dbl(0x3c7a2b7f222f65e2ull);
  if (k2) {
    c = k3 ? 1.0 : 1.5;
    hi = k3 ? dbl(0x3ff921fb54442d18ull) : dbl(0x3fef730bd281f69bull);  // pi/2, atan(1.5)
    lo = k3 ? dbl(0x3c91a62633145c07ull) : dbl(0x3c7007887af0cbbdull);
  }
  double B = k3 ? 0.0 : ax;
  if (k5) B = fma_(c, ay, B);
  const double r0 = rcp14(B, rcp_tab);
  const double e0 = fma_(-r0, B, 1.0);
  const double r1 = fma_(e0, r0, r0);
  const double e1 = fma_(-r1, B, 1.0);
  double A = k3 ? 0.0 : ay;
  if (k5) A = fma_(-c, ax, A);
  const double r2 = fma_(e1, r1, r1);
  const double q = mul(A, r2);
  const double q2 = mul(q, q);
  const double res = fma_(-q, B, A);
  const double q4 = mul(q2, q2);
  double corr = mul(r2, res);
  if (k5) corr = add(corr, lo);
  double p1 = fma_(dbl(0x3f8be4fbe6733718ull), q4, dbl(0x3fa6ad5558fe19c9ull));
  double p2 = fma_(dbl(0xbfa04cd71f92185eull), q4, dbl(0xbfaa9e755ca13d23ull));
  p1 = fma_(q4, p1, dbl(0x3fae12f1edf7c393ull));
  p2 = fma_(q4, p2, dbl(0xbfb1108d326c68edull));
  p1 = fma_(q4, p1, dbl(0x3fb3b132b731e73aull));
  p2 = fma_(q4, p2, dbl(0xbfb745d119677a4full));
  p1 = fma_(q4, p1, dbl(0x3fbc71c719f99f96ull));
  p2 = fma_(q4, p2, dbl(0xbfc2492492441a21ull));
  p1 = fma_(q4, p1, dbl(0x3fc9999999998f43ull));
  p2 = fma_(q4, p2, dbl(0xbfd5555555555552ull));
  const double P = fma_(q2, p1, p2);
  const double Pq2 = mul(P, q2);
  if (xneg) corr = add(corr, dbl(sgnx ^ 0x3ca1a64000000000ull));
  const double t = fma_(q, Pq2, corr);
  double s = add(q, t);
  if (k5) s = add(s, hi);
  s = dbl(bits(s) ^ sgnx);
  if (xneg) s = add(s, 3.141592653589793);
  return dbl(bits(s) | sgny);
}

// ---- __svml_asin8_ha (x), |x| <= 1, constants from __svml_dasin_ha_data_internal
SVE_HD double asin(double x, const uint16_t* rsqrt_tab) {
  const uint64_t b = bits(x);
  const double ax = dbl(b & kAbs);
  const uint64_t sgn = b & kSign;
  const double x2 = mul(ax, ax);
  const bool k2 = !(ax < 0.5);
  const double y = fma_(-0.5, ax, 0.5);
  const bool k1 = y < dbl(0x3000000000000000ull);  // 2^-255
  const double z = (x2 < y) ? x2 : y;               // vminpd(x2, y)
  const double r = k1 ? 0.0 : rsqrt14(y, rsqrt_tab);
  const double y2 = add(y, y);
  const double rr = mul(r, r);
  const double s0 = mul(y2, r);
  const double e = fma_(rr, y2, -2.0);
  const double lo = fma_(r, y2, -s0);
  double p = fma_(dbl(0xbf918000993b24c3ull), e, dbl(0x3fa400006f70d42dull));
  const double se = mul(s0, e);
  p = fma_(e, p, dbl(0xbfb7fffffffffe97ull));
  const double w1 = fma_(dbl(0x3f943f44bfbc3baeull), z, dbl(0x3f7a583395d45ed5ull));
  p = fma_(e, p, dbl(0x3fcfffffffffff9dull));
  const double w2 = fma_(dbl(0x3f9f1c72e13ad8beull), z, dbl(0x3fa6db6db3b445f8ull));
  p = fma_(se, p, -lo);
  double w3 = fma_(dbl(0x3fa07520c70eb909ull), z, dbl(0xbf90fb17f7dbb0edull));
  const double z2 = mul(z, z);
  double w4 = fma_(dbl(0x3f88f8dc2afccad6ull), z, dbl(0x3f8c6dbbcb88bd57ull));
  const double A = k2 ? sub(p, s0) : ax;
  w3 = fma_(z2, w3, w1);
  const double w5 = fma_(dbl(0x3f91c6dcf538ad2eull), z, dbl(0x3f96e89cebdefaddull));
  w4 = fma_(z2, w4, w5);
  const double z4 = mul(z2, z2);
  double P = fma_(z4, w3, w4);
  P = fma_(z2, P, w2);
  P = fma_(z, P, dbl(0x3fb333333337e0deull));
  P = fma_(z, P, dbl(0x3fc555555555529cull));
  const double Pz = mul(P, z);
  const double h = sub(1.5707963267948966, s0);
  const double pl = add(dbl(0x3c91a62633145c07ull), p);
  const double hh = sub(1.5707963267948966, h);
  const double d = sub(s0, hh);
  const double C = k2 ? sub(pl, d) : 0.0;
  const double res = fma_(A, Pz, C);
  const double out = add(k2 ? h : A, res);
  return dbl(bits(out) ^ sgn);
}

}  // namespace svml
