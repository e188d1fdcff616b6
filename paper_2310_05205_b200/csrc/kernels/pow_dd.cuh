// pow_dd.cuh -- p^alpha rounded to the nearest double, for the PER priority
// exponent (reading Q7: key = Q_F(RN(p^alpha))).
//
// alpha in {1, 0, 0.5, 2} uses one IEEE operation (identity, 1, sqrt, p*p),
// which is correctly rounded by definition.  Any other alpha evaluates
// exp(alpha * log p) in double-double arithmetic (~2^-95 relative error over
// the range that can change a key) and returns the high word, i.e. the double
// nearest to that approximation: the correctly rounded p^alpha unless the
// exact value lies within 2^-95 (relative) of a rounding midpoint.
//
// Only values that can change a key need care: with F <= 62 and keys clamped
// to [1, q_max < 2^62], every p^alpha >= 2^62 maps to q_max and every
// p^alpha < 2^-64 maps to 1, so |alpha * log p| > 45 short-cuts to a value on
// the right side of those bounds.
#pragma once

#include <cstdint>

namespace gear {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}

__device__ __forceinline__ dd dd_fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}

__device__ __forceinline__ dd dd_two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}

__device__ __forceinline__ dd dd_add(dd x, dd y) {
  dd s = dd_two_sum(x.hi, y.hi);
  const dd t = dd_two_sum(x.lo, y.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = dd_fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return dd_fast_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }

__device__ __forceinline__ dd dd_mul(dd x, dd y) {
  dd p = dd_two_prod(x.hi, y.hi);
  p.lo = __fma_rn(x.hi, y.lo, p.lo);
  p.lo = __fma_rn(x.lo, y.hi, p.lo);
  return dd_fast_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ dd dd_mul_d(dd x, double d) {
  dd p = dd_two_prod(x.hi, d);
  p.lo = __fma_rn(x.lo, d, p.lo);
  return dd_fast_two_sum(p.hi, p.lo);
}

// x / d for a double d: two quotient digits.
__device__ __forceinline__ dd dd_div_d(dd x, double d) {
  const double q1 = __ddiv_rn(x.hi, d);
  const dd p = dd_two_prod(q1, d);
  const double r = __dadd_rn(__dsub_rn(__dsub_rn(x.hi, p.hi), p.lo), x.lo);
  return dd_fast_two_sum(q1, __ddiv_rn(r, d));
}

// x / y: three quotient digits.
__device__ __forceinline__ dd dd_div(dd x, dd y) {
  const double q1 = __ddiv_rn(x.hi, y.hi);
  dd r = dd_add(x, dd_neg(dd_mul_d(y, q1)));
  const double q2 = __ddiv_rn(r.hi, y.hi);
  r = dd_add(r, dd_neg(dd_mul_d(y, q2)));
  const double q3 = __ddiv_rn(r.hi, y.hi);
  dd q = dd_fast_two_sum(q1, q2);
  return dd_add(q, {q3, 0.0});
}

__device__ __forceinline__ dd dd_ln2() {
  return {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
}

// log(p) for a finite p > 0: p = m * 2^e with m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716, 23 series terms.
__device__ __forceinline__ dd dd_log(double p) {
  int e = 0;
  double m = frexp(p, &e);  // m in [0.5, 1)
  if (m < 0.70710678118654752) {
    m = __dmul_rn(m, 2.0);
    e -= 1;
  }
  const dd num = {__dsub_rn(m, 1.0), 0.0};  // exact (Sterbenz)
  const dd den = dd_two_sum(m, 1.0);        // exact
  const dd s = dd_div(num, den);
  const dd s2 = dd_mul(s, s);
  dd pw = s, acc = s;
#pragma unroll 1
  for (int k = 1; k <= 22; ++k) {
    pw = dd_mul(pw, s2);
    acc = dd_add(acc, dd_div_d(pw, (double)(2 * k + 1)));
  }
  acc = {__dmul_rn(acc.hi, 2.0), __dmul_rn(acc.lo, 2.0)};  // exact scaling
  return dd_add(dd_mul_d(dd_ln2(), (double)e), acc);
}

// exp(x) for |x| <= 45: x = k ln2 + r, |r| <= ln2/2; r' = r / 256;
// expm1(r') by 10 Taylor terms (Horner); 8 squarings of (1 + em1) kept in
// the em1 form; then 1 + em1 scaled by 2^k.
__device__ __forceinline__ dd dd_exp(dd x) {
  const double k = rint(__ddiv_rn(x.hi, 0.69314718055994531));
  const dd r = dd_add(x, dd_neg(dd_mul_d(dd_ln2(), k)));
  const dd rs = {__dmul_rn(r.hi, 1.0 / 256.0), __dmul_rn(r.lo, 1.0 / 256.0)};  // exact
  dd em1 = {0.0, 0.0};
#pragma unroll 1
  for (int i = 10; i >= 1; --i) em1 = dd_mul(dd_div_d(rs, (double)i), dd_add(em1, {1.0, 0.0}));
#pragma unroll 1
  for (int i = 0; i < 8; ++i) {  // (1 + e)^2 - 1 = 2e + e^2
    const dd e2 = dd_mul(em1, em1);
    em1 = dd_add({__dmul_rn(em1.hi, 2.0), __dmul_rn(em1.lo, 2.0)}, e2);
  }
  const dd y = dd_add({1.0, 0.0}, em1);
  const int ki = (int)k;
  return {scalbn(y.hi, ki), scalbn(y.lo, ki)};
}

// The general case, out of line so that it does not add to the register
// footprint of the kernels that quantise (most tables use alpha == 1).
static __device__ __noinline__ double pow_rn_dd(double p, double alpha) {
  const dd x = dd_mul_d(dd_log(p), alpha);
  if (x.hi > 45.0) return 0x1p+100;   // saturates every key at q_max
  if (x.hi < -45.0) return 0x1p-100;  // clamps every key to 1
  return dd_exp(x).hi;
}

// RN(p^alpha) for a finite p > 0 and a finite alpha >= 0 (alpha == 1: p),
// kept finite and positive: overflow gives DBL_MAX, underflow the least
// subnormal (both only matter through the key, which saturates / clamps).
__device__ __forceinline__ double pow_rn(double p, double alpha) {
  if (alpha == 1.0) return p;
  if (alpha == 0.0) return 1.0;
  if (alpha == 0.5) return __dsqrt_rn(p);
  double v;
  if (alpha == 2.0) {
    v = __dmul_rn(p, p);
    v = isinf(v) ? 0x1.fffffffffffffp+1023 : (v == 0.0 ? 0x1p-1074 : v);
  } else {
    v = pow_rn_dd(p, alpha);
  }
  return v;
}

}  // namespace gear
