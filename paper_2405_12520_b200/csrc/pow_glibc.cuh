// pow_glibc.cuh -- glibc's pow() restated for the device (and the host, for
// its validation), so the engine's IDM powers round exactly like CPython's
// `**` on the reference's platform (idm.py:25 `(v / v0_eff) ** delta`,
// idm.py:30 `(s_star / gap) ** 2`).
//
// CPython's float.__pow__ calls libm pow().  glibc >= 2.28 (2.39 here) uses
// the table-driven algorithm of ARM's optimized-routines: log(x) as a
// double-double from a 128-entry table plus a degree-7 polynomial, y*log(x)
// split exactly with an FMA, then exp() from a 128-entry 2^(k/N) table and a
// degree-5 polynomial.  On x86-64 the FMA ifunc variant (__pow_fma) is the
// one that runs, so the __FP_FAST_FMA branches are the ones restated here --
// and that variant is compiled with -mfma and GCC's default fp-contract=fast,
// so every a*b+c whose product has no other use became one fused operation;
// those contractions are restated with explicit fma() below.
// The tables are glibc's own (pow_tables.h, extracted from libm.so.6 by
// tools/gen_pow_tables.py).
//
// Provenance and licence: the algorithm and its constants come from glibc
// (sysdeps/ieee754/dbl-64/e_pow.c, e_pow_log_data.c, e_exp_data.c; GNU
// LGPL-2.1-or-later), which took them from ARM's optimized-routines
// (Copyright (c) 2018 Arm Limited; MIT OR Apache-2.0 WITH LLVM-exception).
// This file restates that published algorithm; the notices of both projects
// apply to it and to pow_tables.h.
//
// This is not a correctly-rounded pow: it is
// glibc's, rounding error for rounding error.  tests/test_pow_glibc.py checks
// the host build of this file against libm on millions of arguments.
//
// Only the domain the model needs is handled natively: x >= 0 (subnormals and
// zero included), finite y.  Anything else returns NaN (never reached: the
// model's bases are a speed ratio and a gap ratio).
#pragma once
// the overflow / underflow results below are intended (glibc builds them the same way)
#ifdef __CUDACC__
#pragma nv_diag_suppress 222
#endif
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define TSB_HD __host__ __device__ __forceinline__
#else
#define TSB_HD inline
#endif

#include "pow_tables.h"

namespace tsb {
namespace glibc_pow {

TSB_HD uint64_t asu64(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}
TSB_HD double asf64(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}
TSB_HD uint32_t top12(double x) { return (uint32_t)(asu64(x) >> 52); }

TSB_HD double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}

#ifdef __CUDA_ARCH__
#define POLY POLY_D
#define LOG_TAB LOG_TAB_D
#define EXP_TAB EXP_TAB_D
#else
#define POLY POLY_H
#define LOG_TAB LOG_TAB_H
#define EXP_TAB EXP_TAB_H
#endif

static constexpr uint64_t OFF = 0x3fe6955500000000ULL;

// log(x) = hi + *tail for the bits ix of a positive normal x (e_pow.c log_inline).
TSB_HD double log_inline(uint64_t ix, double* tail) {
  const uint64_t tmp = ix - OFF;
  const int i = (int)((tmp >> (52 - 7)) % 128);
  const int k = (int)((int64_t)tmp >> 52);  // arithmetic shift
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double z = asf64(iz);
  const double kd = (double)k;
  const double invc = LOG_TAB[i][0], logc = LOG_TAB[i][1], logctail = LOG_TAB[i][2];
  // __FP_FAST_FMA: exact r = z*invc - 1
  const double r = fma_(z, invc, -1.0);
  // k*Ln2 + log(c) + r
  const double t1 = fma_(kd, LN2HI, logc);
  const double t2 = t1 + r;
  const double lo1 = fma_(kd, LN2LO, logctail);
  const double lo2 = t1 - t2 + r;
  // evaluation is optimized assuming superscalar pipelined execution
  const double ar = POLY[0] * r;  // A[0] = -0.5
  const double ar2 = r * ar;
  const double ar3 = r * ar2;
  // k*Ln2 + log(c) + r + A[0]*r*r
  const double hi = t2 + ar2;
  const double lo3 = fma_(ar, r, -ar2);
  const double lo4 = t2 - hi + ar2;
  // p = log1p(r) - r - A[0]*r*r
  const double q = fma_(ar2, fma_(ar2, fma_(r, POLY[6], POLY[5]), fma_(r, POLY[4], POLY[3])), fma_(r, POLY[2], POLY[1]));
  const double lo = fma_(ar3, q, lo1 + lo2 + lo3 + lo4);  // + p, p = ar3 * q
  const double y = hi + lo;
  *tail = hi - y + lo;
  return y;
}

// exp(x + xtail) for |x| outside the fast range (e_pow.c specialcase).
TSB_HD double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    // k > 0: the exponent of scale might have overflowed by <= 460
    sbits -= 1009ULL << 52;
    const double scale = asf64(sbits);
    return 0x1p1009 * fma_(scale, tmp, scale);
  }
  // k < 0: special care in the subnormal range
  sbits += 1022ULL << 52;
  const double scale = asf64(sbits);
  // scale * tmp has two uses here, so the FMA build kept it a product
  const double st = scale * tmp;
  double y = scale + st;
  if ((y < 0.0 ? -y : y) < 1.0) {
    double one = 1.0;
    if (y < 0.0) one = -1.0;
    double lo = scale - y + st;
    const double hi = one + y;
    lo = one - hi + y + lo;
    y = (hi + lo) - one;
    if (y == 0) y = asf64(sbits & 0x8000000000000000ULL);
  }
  return 0x1p-1022 * y;
}

// exp(x + xtail) * (sign_bias ? -1 : 1) (e_pow.c exp_inline).
TSB_HD double exp_inline(double x, double xtail, uint32_t sign_bias) {
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
    if (abstop - top12(0x1p-54) >= 0x80000000u) {
      // tiny x: exp(x) ~ 1 + x (WANT_ROUNDING)
      const double one = 1.0 + x;
      return sign_bias ? -one : one;
    }
    if (abstop >= top12(1024.0)) {
      // overflow / underflow (__math_oflow / __math_uflow)
      const double big = (asu64(x) >> 63) ? 0x1p-767 * 0x1p-767 : 0x1p769 * 0x1p769;
      return sign_bias ? -big : big;
    }
    abstop = 0;  // large |x| is special cased below
  }
  // exp(x) = 2^(k/N) * exp(r), with exp(r) in [2^(-1/2N), 2^(1/2N)]
  // z = InvLn2N * x; kd = z + Shift (one fused operation in the FMA build);
  // z - kd is in [-1, 1] in non-nearest rounding modes (no toint intrinsics on x86-64)
  double kd = fma_(INVLN2N, x, SHIFT);
  const uint64_t ki = asu64(kd);
  kd -= SHIFT;
  double r = fma_(kd, NEGLN2LON, fma_(kd, NEGLN2HIN, x));
  // the code assumes 2^-200 < |xtail| < 2^-8/N
  r += xtail;
  // 2^(k/N) ~= scale * (1 + tail)
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = (ki + sign_bias) << (52 - 7);
  const double tail = asf64(EXP_TAB[idx]);
  // this is only a valid scale when -1023*N < k < 1024*N
  const uint64_t sbits = EXP_TAB[idx + 1] + top;
  // exp(x) = 2^(k/N) * exp(r) ~= scale + scale * (tail + exp(r) - 1)
  const double r2 = r * r;
  const double tmp = fma_(r2 * r2, fma_(r, C5, C4), fma_(r2, fma_(r, C3, C2), tail + r));
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  const double scale = asf64(sbits);
  return fma_(scale, tmp, scale);
}

// glibc pow(x, y) for x >= 0 and finite y (NaN otherwise).
TSB_HD double pow(double x, double y) {
  uint64_t ix = asu64(x);
  const uint64_t iy = asu64(y);
  const uint32_t topx = top12(x), topy = top12(y);
  if (topx - 0x001 >= 0x7ff - 0x001 || (topy & 0x7ff) - 0x3be >= 0x43e - 0x3be) {
    // zero, subnormal, inf/nan or negative x; |y| tiny or huge
    const bool y_zero_inf_nan = 2 * iy - 1 >= 2 * asu64(__builtin_inf()) - 1;
    if (y_zero_inf_nan) {
      if (2 * iy == 0) return 1.0;
      return asf64(0x7ff8000000000000ULL);  // not in the model's domain
    }
    if (2 * ix - 1 >= 2 * asu64(__builtin_inf()) - 1) {  // x is zero, inf or nan
      if (ix >> 63 || (ix & 0x7fffffffffffffffULL) > 0x7ff0000000000000ULL || ix == 0x7ff0000000000000ULL)
        return asf64(0x7ff8000000000000ULL);
      const double x2 = x * x;  // x == +0
      return (iy >> 63) ? 1 / x2 : x2;
    }
    if (ix >> 63) return asf64(0x7ff8000000000000ULL);  // negative x: not in the domain
    if ((topy & 0x7ff) - 0x3be >= 0x43e - 0x3be) {
      // |y| is tiny or huge
      if (ix == asu64(1.0)) return 1.0;
      if ((topy & 0x7ff) < 0x3be) return ix > asu64(1.0) ? 1.0 + y : 1.0 - y;  // |y| tiny
      return (ix > asu64(1.0)) == (topy < 0x800) ? 0x1p769 * 0x1p769 : 0x1p-767 * 0x1p-767;
    }
    if (topx == 0) {
      // normalize subnormal x so the exponent becomes negative
      ix = asu64(x * 0x1p52);
      ix &= 0x7fffffffffffffffULL;
      ix -= 52ULL << 52;
    }
  }
  double lo;
  const double hi = log_inline(ix, &lo);
  // __FP_FAST_FMA
  const double ehi = y * hi;
  const double elo = fma_(y, lo, fma_(y, hi, -ehi));
  return exp_inline(ehi, elo, 0);
}

#undef POLY
#undef LOG_TAB
#undef EXP_TAB
}  // namespace glibc_pow
}  // namespace tsb
