// Lean fp64 transcendentals for the logistic terms, identical on host and device.
//
// The per-row work of every GLM kernel is  nll = (1-y)t + max(-t,0) + log1p(e),
// sigma(t) = (t >= 0 ? 1 : e) / (1 + e),  e = exp(-|t|)  (glm.py:186-192, 371).
// libdevice's exp/log1p handle every IEEE corner and materialise each 64-bit polynomial
// coefficient with two UMOVs (~140 SASS per row).  Here e lies in (0, 1] and 1+e in (1, 2],
// so no special cases are needed; coefficients live in __constant__ memory (DFMA reads
// them from the constant bank) and reciprocals are one fp32 MUFU seed + two fp64 Newton
// steps.  Accuracy (tests/test_abi.py::test_lean_math_accuracy, host == device bitwise
// because both use fused multiply-adds and IEEE-rounded seeds): a few ulp, far inside
// the 1e-10 parity budget of a sum over N rows.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PMM_HD __host__ __device__ __forceinline__
#else
#define PMM_HD inline
#endif

namespace pm {

// exp(-r) Taylor coefficients 1/n!, n = 0..12 (|r| <= ln2/2: truncation < 2e-16)
// log1p core (fdlibm-style, s = f/(2+f), R(s^2)) coefficients Lg1..Lg7
#define PM_MATH_COEFFS                                                                            \
  {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333,                  \
   0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06,       \
   2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09,                              \
   6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,                    \
   2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,                    \
   1.479819860511658591e-01,                                                                        \
   1.4426950408889634074, 6.93147180369123816490e-01, 1.90821492927058770002e-10,                   \
   6.93147180559945309417e-01}

enum {
  PMC_EXP0 = 0,    // .. PMC_EXP0 + 12
  PMC_LG1 = 13,    // .. PMC_LG1 + 6
  PMC_LOG2E = 20,
  PMC_LN2HI = 21,
  PMC_LN2LO = 22,
  PMC_LN2 = 23,
  PMC_N = 24
};

#if defined(__CUDACC__)
static __constant__ double c_pm_math[PMC_N] = PM_MATH_COEFFS;
#endif
static const double h_pm_math[PMC_N] = PM_MATH_COEFFS;

PMM_HD double pmc(int i) {
#if defined(__CUDA_ARCH__)
  return c_pm_math[i];
#else
  return h_pm_math[i];
#endif
}

PMM_HD double pm_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

// 1/x for x in [1, 4): fp32 reciprocal seed (IEEE-rounded on both sides) + 2 Newton steps
PMM_HD double pm_rcp_1_4(double x) {
#if defined(__CUDA_ARCH__)
  double y = double(__frcp_rn(__double2float_rn(x)));
#else
  double y = double(1.0f / float(x));
#endif
  double e = pm_fma(-x, y, 1.0);
  y = pm_fma(y, e, y);
  e = pm_fma(-x, y, 1.0);
  return pm_fma(y, e, y);
}

// exp(-a) for a >= 0 (0 for a > 708, where the result would be subnormal)
PMM_HD double pm_exp_neg(double a_in) {
  // branch-free (callers sit between warp shuffles): clamp, then select 0 past the range
  const double a = fmin(a_in, 708.0);
  const double kd = rint(a * pmc(PMC_LOG2E));
  double r = pm_fma(-kd, pmc(PMC_LN2HI), a);
  r = pm_fma(-kd, pmc(PMC_LN2LO), r);  // a = k ln2 + r, |r| <= ~0.347
  const double x = -r;
  double p = pmc(PMC_EXP0 + 12);
  for (int n = 11; n >= 0; --n) p = pm_fma(p, x, pmc(PMC_EXP0 + n));
  // scale by 2^-k, k in [0, 1022]
  const int64_t k = int64_t(kd);
  const uint64_t bits = uint64_t(1023 - k) << 52;
  double s;
  memcpy(&s, &bits, sizeof(s));
  return a_in > 708.0 ? 0.0 : p * s;
}

// log1p(e) for e in [0, 1]: e <= sqrt2-1 -> f = e, k = 0; else f = (e-1)/2, k = 1, so that
// s = f/(2+f) stays in |s| <= 0.1716, the range the Lg coefficients are fitted on
// (rounding of e-1 there costs < 2^-55 absolute in f)
PMM_HD double pm_log1p_unit(double e) {
  const bool hi = e > 0.41421356237309503;
  const double f = hi ? (e - 1.0) * 0.5 : e;
  const double s = f * pm_rcp_1_4(2.0 + f);
  const double z = s * s, w = z * z;
  const double t1 = w * pm_fma(w, pm_fma(w, pmc(PMC_LG1 + 5), pmc(PMC_LG1 + 3)), pmc(PMC_LG1 + 1));
  const double t2 =
      z * pm_fma(w, pm_fma(w, pm_fma(w, pmc(PMC_LG1 + 6), pmc(PMC_LG1 + 4)), pmc(PMC_LG1 + 2)), pmc(PMC_LG1 + 0));
  const double R = t1 + t2;
  const double hfsq = 0.5 * f * f;
  const double l = f - (hfsq - s * (hfsq + R));
  return hi ? l + pmc(PMC_LN2) : l;
}

// Per-row logistic terms: nll = (1-y) t + max(-t,0) + log1p(exp(-|t|)) and w = y - sigmoid(t)
PMM_HD void pm_row_terms(double t, double y, double& nll, double& w) {
  const double e = pm_exp_neg(fabs(t));
  nll = (1.0 - y) * t + fmax(-t, 0.0) + pm_log1p_unit(e);
  const double inv = pm_rcp_1_4(1.0 + e);
  const double sig = (t >= 0.0) ? inv : e * inv;
  w = y - sig;
}

PMM_HD double pm_row_nll(double t, double y) {
  const double e = pm_exp_neg(fabs(t));
  return (1.0 - y) * t + fmax(-t, 0.0) + pm_log1p_unit(e);
}

}  // namespace pm
