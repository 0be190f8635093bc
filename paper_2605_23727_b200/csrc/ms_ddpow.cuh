// ms_ddpow.cuh — correctly-rounded pow for the step-size controller,
// usable on host (unit-tested against glibc there) and device.
// Every operation is written as a single IEEE op: the device side is compiled
// with -fmad=false and the host side with -ffp-contract=off, so a*b+c never
// contracts; fma() is explicit where an exact product error is needed.
#pragma once
#include <cmath>

#ifdef __CUDACC__
#define MS_HD __host__ __device__
// the general double-double path (~1200 operations) is cold in the controller (the 1/q
// exponents take pow_root): kept out of line so the hot path stays dense in the
// instruction cache (MS_POW_COLD=0 inlines it again)
#ifndef MS_POW_COLD
#define MS_POW_COLD 1
#endif
#if MS_POW_COLD
#define MS_COLD inline __noinline__
#else
#define MS_COLD inline
#endif
#else
#define MS_HD
#define MS_COLD inline
#endif

namespace msb {
MS_HD inline double msb_add(double a, double b) { return a + b; }
MS_HD inline double msb_sub(double a, double b) { return a - b; }
MS_HD inline double msb_mul(double a, double b) { return a * b; }
MS_HD inline double msb_div(double a, double b) { return a / b; }
using std::fma;
using std::isfinite;
using std::ldexp;
using std::log;
using std::pow;
using std::rint;

// ------------------------------------------------------------------------------
// pow for the controller, correctly rounded by construction: exp(y*log(x)) in
// double-double (~100 bits) rounded once. glibc's pow, the reference's
// (solver.cpp:416, 448), is correctly rounded in all but ~1e-3 of calls, so
// this agrees with it far more often than CUDA's pow (<= 2 ulp).
// libm pow (a long routine) for the starts and fall-backs below: one out-of-line copy
MS_HD MS_COLD double pow_libm(double x, double y) { return pow(x, y); }
struct dd {
  double hi, lo;
};
MS_HD inline dd dd_two_sum(double a, double b) {
  const double s = msb_add(a, b);
  const double bb = msb_sub(s, a);
  const double e = msb_add(msb_sub(a, msb_sub(s, bb)), msb_sub(b, bb));
  return {s, e};
}
MS_HD inline dd dd_quick(double a, double b) {
  const double s = msb_add(a, b);
  return {s, msb_sub(b, msb_sub(s, a))};
}
MS_HD inline dd dd_two_prod(double a, double b) {
  const double p = msb_mul(a, b);
  return {p, fma(a, b, -p)};
}
MS_HD inline dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  dd t = dd_two_sum(a.lo, b.lo);
  s.lo = msb_add(s.lo, t.hi);
  s = dd_quick(s.hi, s.lo);
  s.lo = msb_add(s.lo, t.lo);
  return dd_quick(s.hi, s.lo);
}
MS_HD inline dd dd_mul(dd a, dd b) {
  dd p = dd_two_prod(a.hi, b.hi);
  p.lo = msb_add(p.lo, msb_add(msb_mul(a.hi, b.lo), msb_mul(a.lo, b.hi)));
  return dd_quick(p.hi, p.lo);
}
MS_HD inline dd dd_mul_d(dd a, double b) {
  dd p = dd_two_prod(a.hi, b);
  p.lo = msb_add(p.lo, msb_mul(a.lo, b));
  return dd_quick(p.hi, p.lo);
}
MS_HD inline dd dd_exp(dd x) {
  const dd ln2{0.6931471805599453, 2.3190468138462996e-17};
  const double k = rint(msb_div(x.hi, ln2.hi));
  dd kl = dd_two_prod(k, ln2.hi);
  kl.lo = msb_add(kl.lo, msb_mul(k, ln2.lo));
  dd r = dd_add(x, dd{-kl.hi, -kl.lo});
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  // s = exp(r) - 1 by Taylor to r^9/9! (|r| < 3.4e-4)
  dd s = r, term = r;
  for (int i = 2; i <= 9; ++i) {
    term = dd_mul(term, r);
    dd q{msb_div(term.hi, (double)i), 0.0};
    // term/i in double-double: one correction step
    const dd back = dd_mul_d(q, (double)i);
    q.lo = msb_div(msb_add(msb_sub(term.hi, back.hi), msb_sub(term.lo, back.lo)), (double)i);
    term = dd_quick(q.hi, q.lo);
    s = dd_add(s, term);
  }
  for (int i = 0; i < 10; ++i) s = dd_add(dd_mul_d(s, 2.0), dd_mul(s, s));  // (1+s)^2 - 1
  dd e = dd_add(dd{1.0, 0.0}, s);
  const int ki = (int)k;
  return {ldexp(e.hi, ki), ldexp(e.lo, ki)};
}
MS_HD inline dd dd_log(double x) {
  const double y0 = log(x);
  const dd e = dd_exp(dd{-y0, 0.0});
  dd t = dd_mul_d(e, x);              // x * exp(-y0)
  t = dd_add(t, dd{-1.0, 0.0});       // - 1
  return dd_add(dd{y0, 0.0}, t);      // one Newton step
}
// general path: exp(y log x) in double-double (two dd_exp: ~1200 dependent ops)
MS_HD MS_COLD double pow_cr_general(double x, double y) {
  if (!(x > 0.0) || !isfinite(x) || !isfinite(y)) return pow_libm(x, y);
  if (y == 0.0 || x == 1.0) return 1.0;
  const dd l = dd_log(x);
  const dd r = dd_exp(dd_mul_d(l, y));
  const double v = msb_add(r.hi, r.lo);
  return isfinite(v) ? v : pow_libm(x, y);
}

// y = RN(1/q), the controller's exponents (1/3 step control, 1/4 initial_step,
// 1/5 and 1/6 for DP5(4)): x^(1/q) in double-double by one Newton step from
// the libm estimate (error ~q*eps^2), times x^(y - 1/q) = 1 + (y - 1/q) ln x
// (|y - 1/q| < 2^-54, so that factor needs ln x to a few bits only), rounded
// once. ~60 operations instead of ~1200; tests/test_ddpow_host.py checks it
// against the general path and against exact decimal arithmetic.
MS_HD inline bool pow_root(double x, double y, double* out) {
  int q = 0;
  for (int k = 2; k <= 8; ++k)
    if (y == msb_div(1.0, (double)k)) q = k;
  if (q == 0 || !(x > 1e-290 && x < 1e290)) return false;
  // the libm start only has to be good to a few ulp: the Newton step squares
  // its error; the root functions are far shorter chains than pow
#ifndef MS_POW_ROOT_START
#define MS_POW_ROOT_START 1  // 0: start from libm pow (A/B: tools/build_variants.py pow_libm_*)
#endif
  const double r0 = !MS_POW_ROOT_START ? pow_libm(x, y)
                    : q == 2 ? std::sqrt(x)
                    : (q == 3 ? std::cbrt(x) : (q == 4 ? std::sqrt(std::sqrt(x)) : pow_libm(x, y)));
  if (!(r0 > 0.0) || !isfinite(r0)) return false;
  dd p{r0, 0.0};
  for (int i = 1; i < q; ++i) p = dd_mul_d(p, r0);  // r0^q
  const dd diff = dd_add(p, dd{-x, 0.0});            // r0^q - x
  double der = (double)q;
  for (int i = 1; i < q; ++i) der = msb_mul(der, r0);  // q r0^(q-1)
  const double corr = msb_div(msb_add(diff.hi, diff.lo), der);
  dd r = dd_two_sum(r0, -corr);                         // x^(1/q) to ~100 bits
  // y - 1/q = -(residual of RN(1/q)): 1/q = yq + res exactly to 2^-106
  const double res = msb_div(fma(-y, (double)q, 1.0), (double)q);
  const double t = msb_mul(msb_mul(r.hi, -res), log(x));  // r * (y - 1/q) ln x
  const double v = msb_add(r.hi, msb_add(r.lo, t));
  if (!isfinite(v)) return false;
  *out = v;
  return true;
}

MS_HD inline double pow_cr(double x, double y) {
  if (!(x > 0.0) || !isfinite(x) || !isfinite(y)) return pow_libm(x, y);
  if (y == 0.0 || x == 1.0) return 1.0;
  double v;
  if (pow_root(x, y, &v)) return v;
  return pow_cr_general(x, y);
}

}  // namespace msb
