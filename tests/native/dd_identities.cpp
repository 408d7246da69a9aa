// CPU check of the double-double strength reductions in
// paper_2010_04760_b200/csrc/hwg_dd_ops.h: each reduced form must equal the
// reference form (DDReal operators, proj/include/hweno/precision.hpp:53-115)
// BIT FOR BIT on every finite input.  Random inputs over the whole exponent
// range plus edge cases (signed zeros, subnormals, lo = +-0, non-normalised
// pairs, powers of two, sums near 1).  Compiled by tests/test_dd_identities.py
// with g++ -O2 -ffp-contract=off (as the reference is built).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#include "../../paper_2010_04760_b200/csrc/hwg_dd_ops.h"

using hwg::dd;

static uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
static bool same(dd a, dd b) { return bits(a.hi) == bits(b.hi) && bits(a.lo) == bits(b.lo); }
static bool finite(dd a) { return std::isfinite(a.hi) && std::isfinite(a.lo); }

struct Gen {
  std::mt19937_64 r;
  explicit Gen(uint64_t s) : r(s) {}
  double uni() { return std::uniform_real_distribution<double>(0.0, 1.0)(r); }
  // a double with a random exponent in [emin, emax], random mantissa and sign
  double any(int emin = -1074, int emax = 1023, bool sign = true) {
    const int k = (int)(r() % 16);
    if (k == 0) return (sign && (r() & 1)) ? -0.0 : 0.0;
    if (k == 1) return std::ldexp(1.0, emin + (int)(r() % (uint64_t)(emax - emin + 1))) * ((sign && (r() & 1)) ? -1 : 1);
    if (k == 2) {  // subnormal
      uint64_t m = r() & ((1ull << 52) - 1);
      double x;
      std::memcpy(&x, &m, 8);
      return (sign && (r() & 1)) ? -x : x;
    }
    const int e = emin + (int)(r() % (uint64_t)(emax - emin + 1));
    double x = std::ldexp(1.0 + uni(), e);
    if (!std::isfinite(x)) x = std::ldexp(1.0 + uni(), 1000);
    return (sign && (r() & 1)) ? -x : x;
  }
  // a DD value: normalised (fl(hi + lo) == hi) or, 1 in 8, an arbitrary pair
  dd pair(int emin = -1000, int emax = 1000) {
    const double hi = any(emin, emax);
    const int k = (int)(r() % 8);
    if (k == 0) return {hi, any(emin - 60, emax)};
    if (k == 1) return {hi, (r() & 1) ? -0.0 : 0.0};
    double lo = hi * std::ldexp(uni() - 0.5, -52);
    if (r() & 1) lo = -lo;
    double e;
    const double s = hwg::dd_qts(hi, lo, e);
    return {s, e};
  }
};

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 4000000;
  Gen g(20260101);
  const double consts[] = {2, 3, 4, 5, 6, 7, 8, 9, 11, 16, 28, 30, 45, 56, 70, 0.25, 0.5};
  long bad[5] = {0, 0, 0, 0, 0}, tried[5] = {0, 0, 0, 0, 0};
  for (long i = 0; i < n; ++i) {
    // (1) mul_c(a, c) == DD(c) * a
    {
      const dd a = g.pair();
      const double c = (i & 3) ? consts[i % 17] : g.any(-600, 600);
      const dd r1 = hwg::mul_c(a, c), r2 = dd{c, 0.0} * a;
      if (finite(r2)) {
        ++tried[0];
        if (!same(r1, r2)) {
          if (bad[0]++ < 5)
            std::printf("mul_c a=(%a,%a) c=%a: %a %a vs %a %a\n", a.hi, a.lo, c, r1.hi, r1.lo, r2.hi, r2.lo);
        }
      }
    }
    // (1b) mul_p2(a, c) == DD(c) * a for c = 2^k >= 1
    {
      const dd a = g.pair();
      const double c = std::ldexp(1.0, (i & 1) ? (int)(i % 5) : (int)(g.r() % 200));
      const dd r1 = hwg::mul_p2(a, c), r2 = dd{c, 0.0} * a;
      if (finite(r2)) {
        ++tried[4];
        if (!same(r1, r2) && bad[4]++ < 5)
          std::printf("mul_p2 a=(%a,%a) c=%a: %a %a vs %a %a\n", a.hi, a.lo, c, r1.hi, r1.lo, r2.hi, r2.lo);
      }
    }
    // (2) mul_x(b, x) == DD(x) * b
    {
      const dd b = g.pair();
      const double x = g.any(-700, 700, (i & 1) != 0);
      const dd r1 = hwg::mul_x(b, x), r2 = dd{x, 0.0} * b;
      if (finite(r2)) {
        ++tried[1];
        if (!same(r1, r2) && bad[1]++ < 5)
          std::printf("mul_x b=(%a,%a) x=%a: %a %a vs %a %a\n", b.hi, b.lo, x, r1.hi, r1.lo, r2.hi, r2.lo);
      }
    }
    // (3) sum3_nn == (DD(w0) + DD(w1)) + DD(w2) for finite w >= 0: WENO
    // weights (near-partition of 1) and arbitrary non-negative values
    {
      double w0, w1, w2;
      if (i & 1) {
        w0 = g.uni(); w1 = g.uni() * (1 - w0); w2 = 1 - w0 - w1;
        if (i & 2) { w1 = std::ldexp(w1, -(int)(g.r() % 80)); }
        if (i & 4) { w0 = std::ldexp(w0, -(int)(g.r() % 1100)); }
      } else {
        w0 = std::fabs(g.any(-1074, 1020)); w1 = std::fabs(g.any(-1074, 1020));
        w2 = std::fabs(g.any(-1074, 1020));
      }
      if ((i % 5) == 0) w1 = w0;
      const dd r1 = hwg::sum3_nn(w0, w1, w2);
      const dd r2 = (dd{w0, 0.0} + dd{w1, 0.0}) + dd{w2, 0.0};
      if (finite(r2)) {
        ++tried[2];
        if (!same(r1, r2) && bad[2]++ < 5)
          std::printf("sum3 %a %a %a: %a %a vs %a %a\n", w0, w1, w2, r1.hi, r1.lo, r2.hi, r2.lo);
      }
      const dd s1 = hwg::sum2_nn(w0, w2), s2 = dd{w0, 0.0} + dd{w2, 0.0};
      if (finite(s2)) {
        ++tried[3];
        if (!same(s1, s2) && bad[3]++ < 5)
          std::printf("sum2 %a %a: %a %a vs %a %a\n", w0, w2, s1.hi, s1.lo, s2.hi, s2.lo);
      }
    }
  }
  std::printf("mul_c %ld/%ld  mul_p2 %ld/%ld  mul_x %ld/%ld  sum3_nn %ld/%ld  sum2_nn %ld/%ld mismatches\n",
              bad[0], tried[0], bad[4], tried[4], bad[1], tried[1], bad[2], tried[2], bad[3], tried[3]);
  return (bad[0] || bad[1] || bad[2] || bad[3] || bad[4]) ? 1 : 0;
}
