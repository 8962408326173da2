// deskew.cuh — the reference's motion compensation (integrator.py:91-123)
// per point, bit for bit, for the device (prep_kernel) and a host build
// (tests/test_deskew.py).
//
// Per scan the host computes, with scipy exactly as the reference does, the
// few quantities that do not depend on the point: yaw mode y0, dy and the
// tilt quaternion _rot_z(-y1) * R1; se3 mode the start quaternion r0 and the
// Slerp rotation vector. Per point (time t) this file then restates what
// scipy's Cython backend and numpy do to it:
//   ts     = clip(timestamps or linspace(0, 1, n), 0, 1)
//   trans  = (1 - t) t0 + t t1
//   yaw    : q = normalize(compose((0, 0, sin(a/2), cos(a/2)), tilt)),
//            a = y0 + t dy                       (from_euler("z"), __mul__)
//   se3    : q = normalize(compose(r0, from_rotvec(rv t)))    (Slerp)
//   M      = as_matrix(q)
//   p_map  = einsum("nij,nj->ni", M, p) + trans  (numpy sums (j=0 + j=2) + j=1)
//   p_end  = (p_map - t1) @ R1                   (OpenBLAS: FMA chain over k)
// Each formula and operation order was checked against scipy 1.18.1 /
// numpy 2.3 on random inputs (tests/test_deskew.py runs the host build of
// this file against the reference's own motion_compensate). sin/cos are
// the C library's, restated in libm_emu.cuh.
#pragma once

#include "../../include/dbtsdf.h"
#include "libm_emu.cuh"

namespace deskew {

using libm_emu::add;
using libm_emu::fma_;
using libm_emu::mul;
using libm_emu::sub;

#ifdef __CUDA_ARCH__
LM_HD double sqrt_(double x) { return __dsqrt_rn(x); }
LM_HD double div_(double a, double b) { return __ddiv_rn(a, b); }
#else
LM_HD double sqrt_(double x) { return sqrt(x); }
LM_HD double div_(double a, double b) { return a / b; }
#endif

// per-scan constants (host-computed with scipy, see above; include/dbtsdf.h)
using Params = dbt_deskew;

// numpy.linspace(0, 1, n)[i]: i * (1 / (n - 1)), the last element exactly 1
LM_HD double linspace01(int64_t i, int64_t n) {
  if (n <= 1) return 0.0;
  if (i == n - 1) return 1.0;
  return mul((double)i, div_(1.0, (double)(n - 1)));
}

LM_HD double clip01(double t) { return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t); }

// scipy compose_quat (p * q), then normalization of the stored result
LM_HD void compose(const double p[4], const double q[4], double r[4]) {
  const double c0 = sub(mul(p[1], q[2]), mul(p[2], q[1]));
  const double c1 = sub(mul(p[2], q[0]), mul(p[0], q[2]));
  const double c2 = sub(mul(p[0], q[1]), mul(p[1], q[0]));
  r[0] = add(add(mul(p[3], q[0]), mul(q[3], p[0])), c0);
  r[1] = add(add(mul(p[3], q[1]), mul(q[3], p[1])), c1);
  r[2] = add(add(mul(p[3], q[2]), mul(q[3], p[2])), c2);
  r[3] = sub(sub(sub(mul(p[3], q[3]), mul(p[0], q[0])), mul(p[1], q[1])), mul(p[2], q[2]));
  const double n = sqrt_(add(add(add(mul(r[0], r[0]), mul(r[1], r[1])), mul(r[2], r[2])), mul(r[3], r[3])));
  for (int k = 0; k < 4; ++k) r[k] = div_(r[k], n);
}

// scipy from_rotvec (not normalized)
LM_HD void from_rotvec(const double v[3], double q[4], const double* tab, int* rare) {
  const double ang = sqrt_(add(add(mul(v[0], v[0]), mul(v[1], v[1])), mul(v[2], v[2])));
  double sc;
  if (ang <= 1e-3) {
    const double a2 = mul(ang, ang);
    sc = add(sub(0.5, div_(a2, 48.0)), div_(mul(a2, a2), 3840.0));
  } else {
    sc = div_(libm_emu::sin(div_(ang, 2.0), tab, rare), ang);
  }
  q[0] = mul(sc, v[0]);
  q[1] = mul(sc, v[1]);
  q[2] = mul(sc, v[2]);
  q[3] = libm_emu::cos(div_(ang, 2.0), tab, rare);
}

// scipy as_matrix
LM_HD void as_matrix(const double q[4], double m[9]) {
  const double x = q[0], y = q[1], z = q[2], w = q[3];
  const double x2 = mul(x, x), y2 = mul(y, y), z2 = mul(z, z), w2 = mul(w, w);
  const double xy = mul(x, y), zw = mul(z, w), xz = mul(x, z), yw = mul(y, w), yz = mul(y, z), xw = mul(x, w);
  m[0] = add(sub(sub(x2, y2), z2), w2);
  m[3] = mul(2.0, add(xy, zw));
  m[6] = mul(2.0, sub(xz, yw));
  m[1] = mul(2.0, sub(xy, zw));
  m[4] = add(sub(add(-x2, y2), z2), w2);
  m[7] = mul(2.0, add(yz, xw));
  m[2] = mul(2.0, add(xz, yw));
  m[5] = mul(2.0, sub(yz, xw));
  m[8] = add(add(sub(-x2, y2), z2), w2);
}

// The deskewed point in the end-of-sweep sensor frame (float64), given the
// point's time t (already clipped). *rare: a sin/cos argument outside the
// restated range (never for finite rotation inputs).
LM_HD void apply(const Params& P, double t, double p0, double p1, double p2, double out[3], const double* tab,
                 int* rare) {
  double tr[3];
  const double u = sub(1.0, t);
  for (int k = 0; k < 3; ++k) tr[k] = add(mul(u, P.t0[k]), mul(t, P.t1[k]));
  double q[4];
  if (P.mode == DBT_DESKEW_YAW) {
    const double h = div_(add(P.y0, mul(t, P.dy)), 2.0);
    const double qz[4] = {0.0, 0.0, libm_emu::sin(h, tab, rare), libm_emu::cos(h, tab, rare)};
    compose(qz, P.q, q);
  } else {
    const double v[3] = {mul(P.rv[0], t), mul(P.rv[1], t), mul(P.rv[2], t)};
    double qr[4];
    from_rotvec(v, qr, tab, rare);
    compose(P.q, qr, q);
  }
  double m[9];
  as_matrix(q, m);
  double d[3];
  for (int i = 0; i < 3; ++i) {
    const double pm = add(add(mul(m[3 * i], p0), mul(m[3 * i + 2], p2)), mul(m[3 * i + 1], p1));
    d[i] = sub(add(pm, tr[i]), P.t1[i]);
  }
  for (int j = 0; j < 3; ++j) out[j] = fma_(d[2], P.r1[6 + j], fma_(d[1], P.r1[3 + j], mul(d[0], P.r1[j])));
}

}  // namespace deskew
