// Correctly rounded pow(x, -1.0/3.0) for the RKC2 step-size controller
// (host + device).
//
// The reference grows / shrinks the step with `0.8 * emax ** (-1.0 / 3.0)`
// (integrate.py:229,240): a Python float power, i.e. the C library's pow(),
// which glibc evaluates to within 0.52 ulp (in practice correctly rounded).
// CUDA's pow() carries up to 2 ulp of error, so device steps came out an ulp
// off and the adaptive trajectory drifted from the reference's at the next
// decision close to a threshold.
//
// The exponent is the double e = -(1/3)(1 - 2^-54), not -1/3, so the target
// is y = x^(-1/3) * (1 + eta), eta = ln(x) / (3 * 2^54) (|eta| < 1.5e-14).
// The CUDA result is a starting guess, moved to the nearest double by the
// sign of y - m at the midpoints m next to it:  m < y  <=>
// m^3 x - 1 < 3 eta + 3 eta^2, with m^3 x evaluated in double-double
// arithmetic (error ~2^-100, far below a midpoint's 2^-54 relative distance
// from y) and eta from a double log (its error enters at ~2^-98).
#pragma once

#include <cmath>
#include <cstring>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace ddpma {
namespace dev {

__host__ __device__ __forceinline__ double crp_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

#ifdef __CUDA_ARCH__
#define CRP_M(f) ::f
#else
#define CRP_M(f) std::f
#endif

// neighbour of a positive finite double (c > 0: the bit pattern is monotone)
__host__ __device__ __forceinline__ double crp_step(double c, int dir) {
  long long b;
  memcpy(&b, &c, 8);
  b += dir;
  double r;
  memcpy(&r, &b, 8);
  return r;
}

// sign of (c + d)^3 * x - 1 - (e3 + e3^2/3), with c + d an unevaluated sum,
// |d| <= ulp(c)/2 a power of two (so c*d is exact), e3 = 3 eta
__host__ __device__ inline int crp_cube_sign(double c, double d, double x, double e3) {
  // m^2 = c^2 + 2cd (+ d^2, below 2^-104 relative: dropped)
  double s_hi = c * c;
  double s_lo = crp_fma(c, c, -s_hi) + 2.0 * c * d;
  double t = s_hi + s_lo;                        // renormalise
  s_lo = s_lo - (t - s_hi);
  s_hi = t;
  // m^3 = m^2 * (c + d)
  double q_hi = s_hi * c;
  double q_lo = crp_fma(s_hi, c, -q_hi) + (s_lo * c + s_hi * d);
  t = q_hi + q_lo;
  q_lo = q_lo - (t - q_hi);
  q_hi = t;
  // m^3 * x
  double r_hi = q_hi * x;
  double r_lo = crp_fma(q_hi, x, -r_hi) + q_lo * x;
  const double g = ((r_hi - 1.0) - e3) + (r_lo - e3 * e3 * (1.0 / 3.0));   // r_hi - 1 is exact
  return g > 0.0 ? 1 : (g < 0.0 ? -1 : 0);
}

// pow(x, -1.0/3.0) rounded to nearest for positive finite x.
__host__ __device__ inline double pow_m13_rn(double x) {
  double c = CRP_M(pow)(x, -1.0 / 3.0);
  if (!(x > 0.0) || !CRP_M(isfinite)(x) || !CRP_M(isfinite)(c)) return c;
  const double e3 = CRP_M(log)(x) * 0x1p-54;
  for (int it = 0; it < 8; ++it) {
    const double up = crp_step(c, 1);
    const double dn = crp_step(c, -1);
    if (crp_cube_sign(c, 0.5 * (up - c), x, e3) < 0) {          // root above the upper midpoint
      c = up;
      continue;
    }
    if (crp_cube_sign(c, 0.5 * (dn - c), x, e3) > 0) {          // root below the lower midpoint
      c = dn;
      continue;
    }
    break;
  }
  return c;
}

}  // namespace dev
}  // namespace ddpma
