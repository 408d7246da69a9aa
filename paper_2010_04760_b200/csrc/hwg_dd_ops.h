// Double-double scalar arithmetic shared by the device kernels and the CPU
// identity tests (tests/test_dd_identities.py compiles this header with g++
// -ffp-contract=off).  The operators replay DDReal
// (proj/include/hweno/precision.hpp:16-115) operation for operation; the
// mul_* / sum*_nn forms below are strength reductions that are BITWISE equal to
// the reference forms they replace (proofs in the comments, exhaustive
// random + edge-case checks in the tests).
#pragma once

#include <math.h>

#ifdef __CUDACC__
#define HWG_HD __host__ __device__ __forceinline__
#else
#define HWG_HD inline
#endif

namespace hwg {

struct dd {
  double hi, lo;
};

// ---- precision.hpp:16-33 error-free transforms
HWG_HD double dd_two_sum(double a, double b, double& e) {
  double s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
  return s;
}
HWG_HD double dd_qts(double a, double b, double& e) {
  double s = a + b;
  e = b - (s - a);
  return s;
}
HWG_HD double dd_two_prod(double a, double b, double& e) {
  double p = a * b;
  e = fma(a, b, -p);
  return p;
}
// ---- precision.hpp:53-115 operators (same overloads the reference calls)
HWG_HD dd operator+(dd a, dd b) {
  double s2, t2;
  double s1 = dd_two_sum(a.hi, b.hi, s2);
  double t1 = dd_two_sum(a.lo, b.lo, t2);
  s2 += t1;
  s1 = dd_qts(s1, s2, s2);
  s2 += t2;
  s1 = dd_qts(s1, s2, s2);
  return {s1, s2};
}
HWG_HD dd operator+(dd a, double b) {
  double s2;
  double s1 = dd_two_sum(a.hi, b, s2);
  s2 += a.lo;
  s1 = dd_qts(s1, s2, s2);
  return {s1, s2};
}
HWG_HD dd operator-(dd a) { return {-a.hi, -a.lo}; }
HWG_HD dd operator-(dd a, dd b) { return a + (-b); }
HWG_HD dd operator*(dd a, dd b) {
  double p2;
  double p1 = dd_two_prod(a.hi, b.hi, p2);
  p2 += a.hi * b.lo + a.lo * b.hi;
  p1 = dd_qts(p1, p2, p2);
  return {p1, p2};
}
HWG_HD dd operator*(dd a, double b) {
  double p2;
  double p1 = dd_two_prod(a.hi, b, p2);
  p2 += a.lo * b;
  p1 = dd_qts(p1, p2, p2);
  return {p1, p2};
}
HWG_HD dd D(double x) { return {x, 0.0}; }
// precision.hpp:103-112 operator/(DDReal, DDReal) with IEEE divisions (the
// stage kernels use their own branch-free form, hwg_dd.cuh div_dd)
HWG_HD dd dd_div_ieee(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = a - b * q1;
  const double q2 = r.hi / b.hi;
  r = r - b * q2;
  const double q3 = r.hi / b.hi;
  double s2;
  const double s1 = dd_qts(q1, q2, s2);
  return dd{s1, s2} + q3;
}
// precision.hpp sqrt(DDReal): one Karp-Markstein correction of the double
// estimate
HWG_HD dd dd_sqrt(dd a) {
  if (a.hi == 0.0 && a.lo == 0.0) return D(0.0);
  if (a.hi < 0.0) return D(nan(""));
  const double x = 1.0 / sqrt(a.hi);
  const double ax = a.hi * x;
  const dd d = a - D(ax) * D(ax);
  return D(ax) + d.hi * (x * 0.5);
}


// ---- strength reductions (bitwise equal to the reference forms)
//
// mul_c(a, c) == DDReal(c) * a for any a and any double c (a DD constant
// with lo == 0 on the left, as the reference writes TW(2) * f1, TW(4) *
// p[..], quarter * s, half * (..)).  The reference's dd * dd adds
// t = c*a.lo + 0*a.hi to the two_prod error; 0*a.hi is an exact (signed)
// zero, so fma(0, a.hi, c*a.lo) is t bit for bit (same rounding of the same
// exact sum, same zero-sign rule).  One product and one add become one fma
// — and nothing more: the "obvious" a * c (dd * double) differs in the sign
// of a zero lo limb when the two_prod error underflows to -0 (found by the
// identity test; subnormals do occur in this problem's far field).
HWG_HD dd mul_c(dd a, double c) {
  double p2;
  double p1 = dd_two_prod(c, a.hi, p2);
  p2 += fma(0.0, a.hi, c * a.lo);
  p1 = dd_qts(p1, p2, p2);
  return {p1, p2};
}
// mul_p2(a, c) == DDReal(c) * a for c = 2^k >= 1 (TW(2), TW(4), WorkReal(8),
// WorkReal(16) ...): c * a.hi is exact, so the two_prod error is an exact
// +0 and the reference's t = c*a.lo + 0*a.hi is c * a.lo (exact) with a zero
// made +0 — fma(c, a.lo, +0) in one operation; the renormalisation stays.
// 8 operations become 5 (identity test: every finite result).
HWG_HD dd mul_p2(dd a, double c) {
  const double p1 = c * a.hi;
  double p2 = fma(c, a.lo, 0.0);
  const double s = dd_qts(p1, p2, p2);
  return {s, p2};
}
// mul_x(b, x) == DDReal(x) * b (an fp64 weight promoted to DD, on the left
// as in the reference's w[0] * inv): t = x*b.lo + 0*b.hi, same argument.
HWG_HD dd mul_x(dd b, double x) {
  double p2;
  double p1 = dd_two_prod(x, b.hi, p2);
  p2 += fma(0.0, b.hi, x * b.lo);
  p1 = dd_qts(p1, p2, p2);
  return {p1, p2};
}
// sum3_nn(w0, w1, w2) == (DDReal(w0) + DDReal(w1)) + DDReal(w2) for finite
// w >= 0 (the fp64 WENO weights of the mixed mode).  DDReal(w0) + DDReal(w1)
// is two_sum(w0, w1) (exact) followed by two no-op renormalisations (the
// zero lo limbs add +0; the error of a two_sum of non-negative numbers is
// never -0); adding DDReal(w2) is then the dd + double form because the
// first quick_two_sum of the dd + dd form already yields an error-free
// pair (|lo| <= ulp(hi), Fast2Sum), so its second renormalisation is the
// identity.  20 + 20 operations become 7 + 10.
HWG_HD dd sum3_nn(double w0, double w1, double w2) {
  double e;
  const double s = dd_two_sum(w0, w1, e);
  return dd{s, e + 0.0} + w2;
}

// sum2_nn(w0, w1) == DDReal(w0) + DDReal(w1) for finite w >= 0 (the first
// step of sum3_nn): the exact two_sum with its error + 0.0
HWG_HD dd sum2_nn(double w0, double w1) {
  double e;
  const double s = dd_two_sum(w0, w1, e);
  return dd{s, e + 0.0};
}

}  // namespace hwg
