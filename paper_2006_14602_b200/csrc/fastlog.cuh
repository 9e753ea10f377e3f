// Table-driven natural logarithm for the hot kernel (host + device).
//
// CUDA's fp64 log() costs ~90 instructions per call and was 22% of the
// window kernel's instruction stream (ncu, persist.cu).  This restates the
// classic table method (Tang 1990; the same family numpy's AVX512 log uses):
//   x = 2^e m, m in [0.75, 1.5);  k = rn(128 m), c = k/128, inv = rn(1/c)
//   log x = e ln2 + T_k + log1p(r),  r = fma(m, inv, -1),  T_k = -log(inv)
// with m*inv split exactly (r + plo), T_k in double-double (tools/gen_logtable.py), ln2 split so e*ln2_hi is
// exact, and a degree-8 Taylor polynomial for log1p (|r| < 2^-7.5).  The
// bucket of 1.0 has inv = 1, T = 0, so log(1) = 0 exactly and x near 1 keeps
// full relative accuracy.  Max error measured by tools/test_fastlog.cpp (see its output in DESIGN.md).
#pragma once

#include <cmath>
#include <cstring>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

#include "logtable.h"

namespace ddpma {
namespace dev {

// log1p Taylor coefficients 1/7, -1/6, 1/5, 1/3 and ln2 = hi + lo
#define DDPMA_LOGPOLY \
  {0x1.2492492492492p-3, -0x1.5555555555555p-3, 0.2, 0x1.5555555555555p-2, kLn2Hi, kLn2Lo}
#ifdef __CUDACC__
__constant__ double kLogPolyD[6] = DDPMA_LOGPOLY;
#endif
static const double kLogPolyH[6] = DDPMA_LOGPOLY;

// The branch-free part of fastlog_t: x = 2^e * (mantissa given by xhi/xlo), a
// positive normal number (or a subnormal already scaled by the caller).
__host__ __device__ __forceinline__ double fastlog_core(unsigned xhi, unsigned xlo, int e,
                                                        const double (*tab)[3]) {
#ifdef __CUDA_ARCH__
#define DDPMA_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define DDPMA_FMA(a, b, c) std::fma((a), (b), (c))
#endif
  const unsigned hb = (xhi >> 19) & 1u;   // m0 >= 1.5 -> m = m0/2
  e += (int)hb;
  const unsigned mh = (xhi & 0x000FFFFFu) | ((1023u - hb) << 20);
  double m;
#ifdef __CUDA_ARCH__
  m = __hiloint2double((int)mh, (int)xlo);
#else
  {
    const unsigned long long b = ((unsigned long long)mh << 32) | xlo;
    memcpy(&m, &b, 8);
  }
#endif
  // k = (int)(m * 128.0 + 0.5), from the mantissa bits: m in [1, 1.5) ->
  // 128 + round-half-up(f * 128), m in [0.75, 1) -> 64 + round-half-up(f * 64)
  // (f = fraction; bits below the high word cannot move the floor)
  const unsigned f20 = xhi & 0x000FFFFFu;
  const int k = hb ? 64 + (int)((f20 + (1u << 13)) >> 14) : 128 + (int)((f20 + (1u << 12)) >> 13);
  const double* t = tab[k - 96];
  const double pm = m * t[0];                   // m*inv = pm + plo exactly
  const double plo = DDPMA_FMA(m, t[0], -pm);
  const double r = pm - 1.0;                    // exact (Sterbenz: pm in [1-2^-7.5, 1+2^-7.5])
#ifdef __CUDA_ARCH__
  const double* C = kLogPolyD;   // constant bank: DFMA takes c[][] operands directly
#else
  const double* C = kLogPolyH;
#endif
  double q = -0.125;
  q = DDPMA_FMA(q, r, C[0]);    // 1/7
  q = DDPMA_FMA(q, r, C[1]);    // -1/6
  q = DDPMA_FMA(q, r, C[2]);    // 0.2
  q = DDPMA_FMA(q, r, -0.25);
  q = DDPMA_FMA(q, r, C[3]);    // 1/3
  q = DDPMA_FMA(q, r, -0.5);
  const double r2 = r * r;
  const double ed = (double)e;
  const double big = ed * C[4];                 // ed * ln2_hi: exact
  const double s = big + t[1];
  const double err = (big - s) + t[1];          // Fast2Sum (|big| >= |T| or big = 0)
  // log1p(r + plo) = log1p(r) + plo/(1+r) + O(plo^2): plo/(1+r) ~ plo - plo*r
  const double lo = DDPMA_FMA(r2, q, (DDPMA_FMA(ed, C[5], t[2]) + err) + DDPMA_FMA(-plo, r, plo));
  const double a = s + r;                       // TwoSum(s, r): r and T partially cancel near 1
  const double bv = a - s;
  const double e2 = (s - (a - bv)) + (r - bv);
  return a + (e2 + lo);
#undef DDPMA_FMA
}

// x is a positive normal double: the test fastlog_t makes first.
__host__ __device__ __forceinline__ bool fastlog_normal(unsigned xhi) {
  return xhi - 0x00100000u < 0x7fe00000u;
}

// `tab` = the {inv_k, T_hi, T_lo} table (kLogTabD in global memory, or a
// shared-memory copy of it in the window kernel).
__host__ __device__ __forceinline__ double fastlog_t(double x, const double (*tab)[3]) {
#ifdef __CUDA_ARCH__
#define DDPMA_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define DDPMA_FMA(a, b, c) std::fma((a), (b), (c))
#endif
  // Decomposition on the high word only (32-bit integer ops; on the device the
  // 64-bit versions of these were ~20 instructions per call).
  unsigned xhi, xlo;
#ifdef __CUDA_ARCH__
  xhi = (unsigned)__double2hiint(x);
  xlo = (unsigned)__double2loint(x);
#else
  {
    unsigned long long b;
    memcpy(&b, &x, 8);
    xhi = (unsigned)(b >> 32);
    xlo = (unsigned)b;
  }
#endif
  int e;
  if (xhi - 0x00100000u < 0x7fe00000u) {   // positive normal: one unsigned compare
    e = (int)(xhi >> 20) - 1023;
  } else {
    if (!(x > 0.0)) return x == 0.0 ? -INFINITY : NAN;   // log(+-0) = -inf, log(<0 | NaN) = NaN
    if (x == INFINITY) return x;
    const double xs = x * 0x1p54;   // subnormal: scale into the normal range
#ifdef __CUDA_ARCH__
    xhi = (unsigned)__double2hiint(xs);
    xlo = (unsigned)__double2loint(xs);
#else
    unsigned long long b;
    memcpy(&b, &xs, 8);
    xhi = (unsigned)(b >> 32);
    xlo = (unsigned)b;
#endif
    e = (int)(xhi >> 20) - 1023 - 54;
  }
  return fastlog_core(xhi, xlo, e, tab);
#undef DDPMA_FMA
}

__host__ __device__ __forceinline__ double fastlog(double x) {
#ifdef __CUDA_ARCH__
  return fastlog_t(x, kLogTabD);
#else
  return fastlog_t(x, kLogTabH);
#endif
}

}  // namespace dev
}  // namespace ddpma
