// Numerics shared by the sm_100a kernels and the host (tests call the host
// instantiations through the C-ABI helpers psg_pow_cr / psg_hist_mass).
//
// The reference computes in fp64 with separate multiply and add (no FMA
// contraction).  Every accumulation below that must be
// bit-identical to the reference uses __dmul_rn / __dadd_rn explicitly, and
// the kernels are compiled with --fmad=false as a second guard.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define PSG_HD __host__ __device__ __forceinline__
#else
#define PSG_HD inline
#endif

namespace psg {

PSG_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
PSG_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
PSG_HD double dsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  volatile double r = a - b;
  return r;
#endif
}
PSG_HD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

// ---- double-double arithmetic (for a correctly rounded pow) -----------------
struct dd {
  double hi, lo;
};

PSG_HD dd two_sum(double a, double b) {
  const double s = dadd(a, b);
  const double bb = dsub(s, a);
  const double e = dadd(dsub(a, dsub(s, bb)), dsub(b, bb));
  return {s, e};
}
PSG_HD dd quick_two_sum(double a, double b) {
  const double s = dadd(a, b);
  return {s, dsub(b, dsub(s, a))};
}
PSG_HD dd two_prod(double a, double b) {
  const double p = dmul(a, b);
  return {p, dfma(a, b, -p)};
}
PSG_HD dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo = dadd(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = dadd(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
PSG_HD dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = dadd(p.lo, dadd(dmul(a.hi, b.lo), dmul(a.lo, b.hi)));
  return quick_two_sum(p.hi, p.lo);
}
PSG_HD dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = dadd(p.lo, dmul(a.lo, b));
  return quick_two_sum(p.hi, p.lo);
}

// exp of a double-double, relative error ~2^-100 for |x| < 700.
PSG_HD dd dd_exp(dd x) {
  const double ln2_hi = 6.93147180559945286227e-01;
  const double ln2_lo = 2.31904681384629955842e-17;
  const double k = rint(x.hi / ln2_hi);
  // r = x - k*ln2 in double-double
  dd r = dd_add(x, dd_mul_d(dd{-ln2_hi, -ln2_lo}, k));
  // scale down by 2^-10 then Taylor (degree 11), then square 10 times
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  // 1/n as double-doubles (|error| < 2^-106 relative): the Taylor terms are
  // scaled by multiplication instead of two fp64 divisions per term
  const double inv_hi[12] = {0, 0, 0x1p-1, 0x1.5555555555555p-2, 0x1p-2, 0x1.999999999999ap-3,
                             0x1.5555555555555p-3, 0x1.2492492492492p-3, 0x1p-3, 0x1.c71c71c71c71cp-4,
                             0x1.999999999999ap-4, 0x1.745d1745d1746p-4};
  const double inv_lo[12] = {0, 0, 0, 0x1.5555555555555p-56, 0, -0x1.999999999999ap-57,
                             0x1.5555555555555p-57, 0x1.2492492492492p-57, 0, 0x1.c71c71c71c71cp-58,
                             -0x1.999999999999ap-58, -0x1.745d1745d1746p-59};
  dd term = r;
  dd sum = r;  // expm1 accumulation
#pragma unroll
  for (int n = 2; n <= 9; ++n) {  // |r| <= 3.4e-4: the first omitted term r^10 / 10! < 2^-120 |r|
    term = dd_mul(dd_mul(term, r), dd{inv_hi[n], inv_lo[n]});
    sum = dd_add(sum, term);
  }
  // (1 + s)^2 - 1 = 2s + s^2 keeps the small quantity exact-ish
  for (int i = 0; i < 10; ++i) {
    dd s2 = dd_mul(sum, sum);
    dd twice = {dmul(sum.hi, 2.0), dmul(sum.lo, 2.0)};
    sum = dd_add(twice, s2);
  }
  dd one_plus = dd_add(dd{1.0, 0.0}, sum);
  const int ki = (int)k;
  return {ldexp(one_plus.hi, ki), ldexp(one_plus.lo, ki)};
}

// log of a positive double as double-double: one Newton step on exp.
PSG_HD dd dd_log(double x) {
  const double y0 = log(x);
  const dd e = dd_exp(dd{-y0, 0.0});       // exp(-y0)
  dd t = dd_mul_d(e, x);                    // x * exp(-y0) ~ 1
  t = dd_add(t, dd{-1.0, 0.0});             // x*exp(-y0) - 1
  return dd_add(dd{y0, 0.0}, t);
}

// x^y for x > 0 finite, correctly rounded except within ~2^-100 of a
// rounding boundary.  Used for the IRLS weight (optimizer.cpp:112-115) and
// the energy (optimizer.cpp:126-131), where the reference calls glibc pow.
PSG_HD double pow_cr(double x, double y) {
  if (x == 1.0 || y == 0.0) return 1.0;
  if (!(x > 0.0) || !isfinite(x) || !isfinite(y)) return pow(x, y);
  if (y == 1.0) return x;
  const dd l = dd_log(x);
  const dd p = dd_mul_d(l, y);
  if (p.hi > 709.0 || p.hi < -745.0) return pow(x, y);
  const dd e = dd_exp(p);
  return dadd(e.hi, e.lo);
}

// ---- exact histogram mass ------------------------------------------------------
// build_histograms adds inv = 1/P once per pixel into mass[b]
// (optimizer.cpp:76-86).  Every increment of a bin is the same double, so
// the sequential sum is a function of the count alone.  Within one binade a
// constant increment is exact after two in-binade steps (ties-to-even makes
// the ulp-count even after one tie step), which lets us jump in bulk.
// frexp exponent of a positive normal double, and 2^e, from the bit pattern
PSG_HD int exp_of(double x) {
  int64_t b;
  memcpy(&b, &x, sizeof b);
  return (int)((b >> 52) & 0x7ff) - 1022;
}
PSG_HD double pow2(int e) {  // 2^e for -1022 <= e <= 1023
  const int64_t b = (int64_t)(e + 1023) << 52;
  double x;
  memcpy(&x, &b, sizeof x);
  return x;
}

PSG_HD double hist_mass(int64_t count, double inv) {
  double m = 0.0;
  int64_t rem = count;
  while (rem > 0) {
    const double m1 = dadd(m, inv);
    --rem;
    if (rem == 0 || m == 0.0) { m = m1; continue; }
    // m, m1 >= inv > 0 are normal (inv = 1/P): exponents from the bits
    const int e0 = exp_of(m), e1 = exp_of(m1);
    if (e0 != e1) { m = m1; continue; }
    const double m2 = dadd(m1, inv);
    --rem;
    const int e2 = exp_of(m2);
    if (e2 != e1 || rem == 0) { m = m2; continue; }
    // steady state inside binade [2^(e2-1), 2^e2): ulp u = 2^(e2-53); the
    // differences below are multiples of u, so scaling by 1/u is exact
    const double inv_u = pow2(53 - e2);
    const double top = pow2(e2);
    const int64_t T = (int64_t)dmul(dsub(top, m2), inv_u);      // exact
    const int64_t delta = (int64_t)dmul(dsub(m2, m1), inv_u);   // exact
    const double u = pow2(e2 - 53);
    int64_t k = (T - 1) / delta;
    if (k > rem) k = rem;
    m = dadd(m2, dmul((double)k, (double)delta * u));  // exact: below top
    rem -= k;
  }
  return m;
}

// bin_of(float) evaluates floor(value * bins) in fp32 (optimizer.cpp:60-63).
PSG_HD int bin_of_f32(float v, int bins) {
#ifdef __CUDA_ARCH__
  const float p = __fmul_rn(v, (float)bins);
#else
  volatile float p = v * (float)bins;
#endif
  int b = (int)floorf(p);
  return b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
}

// build_histograms bins fp64 values (optimizer.cpp:81-82).
PSG_HD int bin_of_f64(double v, int bins) {
  int b = (int)floor(dmul(v, (double)bins));
  return b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
}

#ifdef __CUDACC__
// One 32-byte read-only global load (LDG.E.256 on sm_100): a padded 8-float
// exemplar pixel in one instruction, one sector per lane.
__device__ __forceinline__ void ldg256(const float* p, float4& lo, float4& hi) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
      : "l"(p));
}
#endif

}  // namespace psg
