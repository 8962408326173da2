// libm_emu.cuh — bit-exact restatement of the C library's double sin/cos for
// the on-device deskew (integrator.py:91-123, §8(f)3).
//
// The reference deskews with scipy's Rotation/Slerp, whose Cython backend
// calls the C library's sin/cos once per point (from_euler("z"), from_rotvec).
// On the build container and the GPU box that is glibc 2.39's x86-64 libm,
// which dispatches sin/cos to its FMA-compiled variants. Those are the IBM
// Accurate Mathematical Library algorithm (glibc sysdeps/ieee754/dbl-64/
// s_sin.c, LGPL; the published algorithm is restated here, not its code):
//   * |x| < 2^-26 (sin) / 2^-27 (cos): x / 1;
//   * |x| < 0.855469: do_sin(x, 0) / do_cos(x, 0);
//   * |x| < 2.426265: the other function of pi/2 - |x| (two-double pi/2);
//   * |x| < 105414350: Cody-Waite reduction by pi/2 (four-part pi/2), then
//     do_sin / do_cos of the reduced (a, da) by quadrant.
// do_sin / do_cos split x = x_k + r with x_k = k/128 (rounded by adding
// 1.5 * 2^45), evaluate short Taylor polynomials of r and combine them with
// a table of sin/cos(x_k) as double-doubles; |x| < 0.126 takes a degree-9
// Taylor polynomial instead. The results are not correctly rounded (up to
// 0.52 ulp), so only the same operations in the same order give the same
// bits: every fused multiply-add below is one the compiler formed in the
// FMA variant (read from its instruction sequence), every other operation
// rounds on its own. The constants are the published ones.
//
// The table (sn, ssn, cs, ccs for k = 0..109: sin(k/128) and cos(k/128) as
// high + low doubles) is the C library's own data: its low parts are not
// the correctly rounded remainders, so it cannot be regenerated. The engine
// reads it from the loaded libm at run time (deskew.cu) and checks this
// restatement against the library's sin/cos before any device use.
//
// Scope: |x| < 105414350 (larger arguments, NaN and inf set *rare; the
// deskew never produces them: half-angles of at most ~pi).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define LM_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define LM_HD static inline
#endif

namespace libm_emu {

#ifdef __CUDA_ARCH__
LM_HD uint64_t bits(double d) { return (uint64_t)__double_as_longlong(d); }
LM_HD double dbl(uint64_t u) { return __longlong_as_double((long long)u); }
LM_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
LM_HD double mul(double a, double b) { return __dmul_rn(a, b); }
LM_HD double add(double a, double b) { return __dadd_rn(a, b); }
LM_HD double sub(double a, double b) { return __dsub_rn(a, b); }
#else
LM_HD uint64_t bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
LM_HD double dbl(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
LM_HD double fma_(double a, double b, double c) { return fma(a, b, c); }
LM_HD double mul(double a, double b) { return a * b; }  // host TU built with -ffp-contract=off
LM_HD double add(double a, double b) { return a + b; }
LM_HD double sub(double a, double b) { return a - b; }
#endif

constexpr int kTabEntries = 440;  // 110 x (sn, ssn, cs, ccs)

// polynomial coefficients of the table-based path (sin: x + sn3 x^3 +
// sn5 x^5; cos: cs2 x^2 + cs4 x^4 + cs6 x^6) and of the small-argument
// Taylor path (s1..s5)
constexpr double kSn3 = -0x1.5555555555515p-3, kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs2 = 0x1.0000000000000p-1, kCs4 = -0x1.5555555555535p-5, kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3, kS2 = 0x1.1111111110ecep-7, kS3 = -0x1.a01a019db08b8p-13,
                 kS4 = 0x1.71de27b9a7ed9p-19, kS5 = -0x1.addffc2fcdf59p-26;
constexpr double kBig = 0x1.8p45;                                        // rounds to multiples of 1/128
constexpr double kHp0 = 0x1.921fb54442d18p+0, kHp1 = 0x1.1a62633145c07p-54;  // pi/2 = hp0 + hp1
constexpr double kHpInv = 0x1.45f306dc9c883p-1, kToInt = 0x1.8p52;           // 2/pi, 1.5 * 2^52
constexpr double kMp1 = 0x1.921fb58000000p+0, kMp2 = -0x1.dde973c000000p-27;
constexpr double kPp3 = -0x1.cb3b398000000p-55, kPp4 = -0x1.d747f23e32ed7p-83;

LM_HD double fabs_(double x) { return dbl(bits(x) & 0x7fffffffffffffffull); }
LM_HD double copysign_(double m, double s) {
  return dbl((bits(m) & 0x7fffffffffffffffull) | (bits(s) & 0x8000000000000000ull));
}

// a + (xx (P(xx) a - da/2) + da): the degree-9 Taylor path (|a| < 0.126)
LM_HD double taylor_sin(double a, double da) {
  const double xx = mul(a, a);
  double p = fma_(xx, kS5, kS4);
  p = fma_(xx, p, kS3);
  p = fma_(xx, p, kS2);
  p = fma_(xx, p, kS1);
  const double t = fma_(p, a, -mul(0.5, da));
  return add(a, fma_(xx, t, da));
}

LM_HD void split(double ax, double* r, int* k) {
  const double u = add(kBig, ax);
  *r = sub(ax, sub(u, kBig));
  *k = (int)(bits(u) & 0xffffffffu) << 2;
}

// sin(x + dx) (glibc do_sin)
LM_HD double do_sin(double x, double dx, const double* tab) {
  if (fabs_(x) < 0.126) return taylor_sin(x, dx);
  if (x <= 0) dx = -dx;
  double r;
  int k;
  split(fabs_(x), &r, &k);
  const double xx = mul(r, r);
  const double s = add(r, fma_(mul(r, xx), fma_(xx, kSn5, kSn3), dx));
  const double c = fma_(r, dx, mul(xx, fma_(xx, fma_(xx, kCs6, kCs4), kCs2)));
  const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  const double cor = fma_(s, cs, fma_(-c, sn, fma_(s, ccs, ssn)));
  return copysign_(add(sn, cor), x);
}

// cos(x + dx) (glibc do_cos)
LM_HD double do_cos(double x, double dx, const double* tab) {
  if (x < 0) dx = -dx;
  double r;
  int k;
  split(fabs_(x), &r, &k);
  r = add(r, dx);
  const double xx = mul(r, r);
  const double s = fma_(mul(r, xx), fma_(xx, kSn5, kSn3), r);
  const double c = mul(xx, fma_(xx, fma_(xx, kCs6, kCs4), kCs2));
  const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  const double cor = fma_(-s, sn, fma_(-c, cs, fma_(-s, ssn, ccs)));
  return add(cs, cor);
}

// x = n pi/2 + (a + da), |x| < 105414350 (glibc reduce_sincos)
LM_HD int reduce(double x, double* a, double* da) {
  const double t = fma_(x, kHpInv, kToInt);
  const double xn = sub(t, kToInt);
  const int n = (int)(bits(t) & 3u);
  const double y = fma_(-xn, kMp2, fma_(-xn, kMp1, x));
  const double t2 = fma_(-xn, kPp3, y);
  double db = fma_(-kPp3, xn, sub(y, t2));
  const double b = fma_(-xn, kPp4, t2);
  db = add(db, fma_(-xn, kPp4, sub(t2, b)));
  *a = b;
  *da = db;
  return n;
}

LM_HD double do_sincos(double a, double da, int n, const double* tab) {
  const double r = (n & 1) ? do_cos(a, da, tab) : do_sin(a, da, tab);
  return (n & 2) ? -r : r;
}

LM_HD double sin(double x, const double* tab, int* rare) {
  const uint32_t k = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(x, 0.0, tab);
  if (k < 0x400368fdu) return copysign_(do_cos(sub(kHp0, fabs_(x)), kHp1, tab), x);
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce(x, &a, &da);
    return do_sincos(a, da, n, tab);
  }
  *rare = 1;
  return 0.0;
}

LM_HD double cos(double x, const double* tab, int* rare) {
  const uint32_t k = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(x, 0.0, tab);
  if (k < 0x400368fdu) {
    const double y = sub(kHp0, fabs_(x));
    const double a = add(y, kHp1);
    const double da = add(sub(y, a), kHp1);
    return do_sin(a, da, tab);
  }
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce(x, &a, &da);
    return do_sincos(a, da, n + 1, tab);
  }
  *rare = 1;
  return 0.0;
}

}  // namespace libm_emu
