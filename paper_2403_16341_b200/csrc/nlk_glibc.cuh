// SPDX-License-Identifier: LGPL-2.1-or-later AND BSD-3-Clause (see NOTICE):
// glibc-derived libm ports (LGPL) and SVML-derived numpy exp/arctan (BSD-3).
// Bit-exact device (and host) ports of the glibc 2.39 x86-64 FMA-variant
// exp, pow (integer y), sin, cos and atan.
//
// nlkit evaluates its residuals with CPython's math module and numpy, which
// call glibc's libm; glibc is not correctly rounded (~0.1 % of results are
// one ulp off the true value), and CUDA's libdevice differs from it in the
// last bit far more often.  On chaotic problems (test23/trigonometric, boggs)
// those bits decide retcodes and iteration counts, so the device evaluates
// glibc's own algorithms: Szabolcs Nagy's table-driven exp/pow and the IBM
// Accurate Mathematical Library sin/cos/atan, with the operation order and
// FMA placement of the binary the reference actually runs (transcribed from
// its disassembly; tables extracted by tools/extract_glibc_tables.c).
// Verified bit-exact against libm on >10^7 inputs per function
// (tests/test_glibc_ports.py compiles this header for the host).
//
// sin/cos of |x| >= 105414350 go through a port of glibc's Payne-Hanek
// __branred.
#pragma once
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define NLK_HD __host__ __device__ __forceinline__
#else
#define NLK_HD inline
#endif

namespace nlk {
namespace glibc {

#define NLK_GLIBC_TABLE(name, n) static const uint64_t h_##name[n]
#include "nlk_glibc_tables.inc"
#undef NLK_GLIBC_TABLE
#if defined(__CUDACC__)
#define NLK_GLIBC_TABLE(name, n) static __device__ const uint64_t d_##name[n]
#include "nlk_glibc_tables.inc"
#undef NLK_GLIBC_TABLE
#endif

// table accessors: device copy in device code, host copy otherwise
#if defined(__CUDA_ARCH__)
#define NLK_GLIBC_ACCESSOR(name) \
  NLK_HD uint64_t tab_##name(int i) { return d_##name[i]; }
#else
#define NLK_GLIBC_ACCESSOR(name) \
  NLK_HD uint64_t tab_##name(int i) { return h_##name[i]; }
#endif
NLK_GLIBC_ACCESSOR(exp_tab)
NLK_GLIBC_ACCESSOR(pow_log_tab)
NLK_GLIBC_ACCESSOR(sincos_tab)
NLK_GLIBC_ACCESSOR(atan_tab)
NLK_GLIBC_ACCESSOR(toverp)
#undef NLK_GLIBC_ACCESSOR
#define NLK_PICK(name, i) tab_##name(i)

NLK_HD double asd(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
NLK_HD uint64_t asu(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}
NLK_HD double dfma(double a, double b, double c) { return fma(a, b, c); }

// ---- exp (sysdeps/ieee754/dbl-64/e_exp.c, FMA build) ------------------------
constexpr double kInvLn2N = 0x1.71547652b82fep+7, kShift = 0x1.8p52;
constexpr double kNegLn2hiN = -0x1.62e42fefap-8, kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
constexpr double kC2 = 0x1.ffffffffffdbdp-2, kC3 = 0x1.555555555543cp-3;
constexpr double kC4 = 0x1.55555cf172b91p-5, kC5 = 0x1.1111167a4d017p-7;

// exp_inline tail shared by exp and pow: exp(x + xtail) with sign bias
NLK_HD double exp_core(double x, double xtail, uint64_t sign_bias, bool pow_mode) {
  uint32_t abstop = (asu(x) >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) {
      double one = 1.0 + x;
      return sign_bias ? -one : one;
    }
    if (abstop > 0x408) {
      if (!pow_mode) {
        uint64_t ix = asu(x);
        if (ix == 0xfff0000000000000ull) return 0.0;
        if (abstop == 0x7ff) return 1.0 + x;
      }
      if (asu(x) >> 63) return sign_bias ? -0.0 : 0.0;
      return sign_bias ? -INFINITY : INFINITY;
    }
    abstop = 0;
  }
  const double z = dfma(x, kInvLn2N, kShift);
  const uint64_t ki = asu(z);
  const double kd = z - kShift;
  double r = dfma(kd, kNegLn2hiN, x);
  r = dfma(kd, kNegLn2loN, r);
  if (pow_mode) r = xtail + r;
  const int idx = static_cast<int>(2 * (ki & 0x7f));
  const uint64_t top = (ki + sign_bias) << 45;
  uint64_t sbits = NLK_PICK(exp_tab, idx + 1) + top;
  const double p23 = dfma(r, kC3, kC2);
  const double tr = r + asd(NLK_PICK(exp_tab, idx));
  const double r2 = r * r;
  const double p45 = dfma(r, kC5, kC4);
  const double t = dfma(p23, r2, tr);
  const double r4 = r2 * r2;
  const double tmp = dfma(p45, r4, t);
  if (abstop == 0) {
    if ((ki & 0x80000000u) == 0) {
      sbits -= 1009ull << 52;
      const double scale = asd(sbits);
      return dfma(scale, tmp, scale) * 0x1p1009;
    }
    sbits += 1022ull << 52;
    const double scale = asd(sbits);
    const double st = tmp * scale;
    double y = scale + st;
    if (1.0 > fabs(y)) {
      const double one = (pow_mode && y < 0.0) ? -1.0 : 1.0;
      double lo = scale - y;
      lo = lo + st;
      const double hi = y + one;
      double t1 = one - hi;
      t1 = t1 + y;
      t1 = t1 + lo;
      t1 = t1 + hi;
      y = t1 - one;
      if (y == 0.0) y = pow_mode ? asd(sbits & 0x8000000000000000ull) : 0.0;
    }
    return y * 0x1p-1022;
  }
  const double scale = asd(sbits);
  return dfma(scale, tmp, scale);
}

NLK_HD double exp(double x) { return exp_core(x, 0.0, 0, false); }

// ---- pow (sysdeps/ieee754/dbl-64/e_pow.c, FMA build), y integer-valued -------
constexpr double kLn2hi = 0x1.62e42fefa38p-1, kLn2lo = 0x1.ef35793c7673p-45;
constexpr double kP0 = -0.5, kP1 = -0x1.555555555556p-1, kP2 = 0x1.0000000000006p-1;
constexpr double kP3 = 0x1.999999959554ep-1, kP4 = -0x1.555555529a47ap-1;
constexpr double kP5 = -0x1.2495b9b4845e9p+0, kP6 = 0x1.0002b8b263fc3p+0;

// x ** y for y in {2, 3} (the exponents the reference's residuals use)
template <int Y>
NLK_HD double pow_int(double x) {
  constexpr double y = static_cast<double>(Y);
  uint64_t ix = asu(x);
  uint32_t topx = static_cast<uint32_t>(ix >> 52);
  uint64_t sign_bias = 0;
  if (topx - 1u > 0x7fdu) {
    if (2 * ix - 1 >= 2 * 0x7ff0000000000000ull - 1) {  // 0, inf, nan
      double x2 = x * x;
      if ((ix >> 63) && (Y & 1)) x2 = -x2;
      return x2;
    }
    if (ix >> 63) {  // negative finite x, integer y
      if (Y & 1) sign_bias = 0x40000;
      ix &= 0x7fffffffffffffffull;
      topx &= 0x7ff;
    }
    if (topx == 0) {  // subnormal
      ix = asu(asd(ix) * 0x1p52);
      ix &= 0x7fffffffffffffffull;
      ix -= 52ull << 52;
    }
  }
  const uint64_t tmp = ix - 0x3fe6955500000000ull;
  const int i = static_cast<int>((tmp >> 45) & 0x7f);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double z = asd(iz), kd = static_cast<double>(k);
  const double invc = asd(NLK_PICK(pow_log_tab, 4 * i));
  const double logc = asd(NLK_PICK(pow_log_tab, 4 * i + 2));
  const double logctail = asd(NLK_PICK(pow_log_tab, 4 * i + 3));
  const double t1 = dfma(kd, kLn2hi, logc);
  const double lo1 = dfma(kd, kLn2lo, logctail);
  const double r = dfma(z, invc, -1.0);
  const double ar = r * kP0;
  const double q12 = dfma(r, kP2, kP1);
  const double q34 = dfma(r, kP4, kP3);
  const double t2 = r + t1;
  const double lo2 = (t1 - t2) + r;
  const double ar2 = r * ar;
  const double ar3 = r * ar2;
  const double lo3 = dfma(ar, r, -ar2);
  const double hi = t2 + ar2;
  double q56 = dfma(r, kP6, kP5);
  const double lo4 = (t2 - hi) + ar2;
  q56 = dfma(q56, ar2, q34);
  const double p = dfma(ar2, q56, q12);
  double lo = ((lo1 + lo2) + lo3) + lo4;
  lo = dfma(ar3, p, lo);
  const double lhi = hi + lo;
  const double llo = (hi - lhi) + lo;
  const double ehi = y * lhi;
  const double elo0 = dfma(lhi, y, -ehi);
  const double elo = dfma(y, llo, elo0);
  return exp_core(ehi, elo, sign_bias, true);
}

// ---- sin / cos (sysdeps/ieee754/dbl-64/s_sin.c, FMA build) -------------------
constexpr double kBig = 0x1.8p45, kSn5 = 0x1.11110e829872fp-7, kSn3 = -0x1.5555555555515p-3;
constexpr double kCs6 = 0x1.6c16bedd9e239p-10, kCs4 = -0x1.5555555555535p-5, kCs2 = 0.5;
constexpr double kHp0 = 0x1.921fb54442d18p+0, kHp1 = 0x1.1a62633145c07p-54;
constexpr double kToint = 0x1.8p52, kHpinv = 0x1.45f306dc9c883p-1;
constexpr double kMp1 = 0x1.921fb58p+0, kMp2 = -0x1.dde973cp-27;
constexpr double kPp3 = -0x1.cb3b398p-55, kPp4 = -0x1.d747f23e32ed7p-83;
constexpr double kS5 = -0x1.addffc2fcdf59p-26, kS4 = 0x1.71de27b9a7ed9p-19;
constexpr double kS3 = -0x1.a01a019db08b8p-13, kS2 = 0x1.1111111110ecep-7;
constexpr double kS1 = -0x1.5555555555555p-3, kSmall = 0.126;

// NLK_GLIBC_CBANK: device code reads these constants from the constant bank
// (c[..] operands) instead of materialising each 64-bit value with two moves
// per use inside the out-of-line sincos calls.  Same values, same operations.
#ifndef NLK_GLIBC_CBANK
#define NLK_GLIBC_CBANK 1
#endif
#if defined(__CUDACC__) && NLK_GLIBC_CBANK
static __constant__ double cb_kBig = kBig;
static __constant__ double cb_kSn5 = kSn5;
static __constant__ double cb_kSn3 = kSn3;
static __constant__ double cb_kCs6 = kCs6;
static __constant__ double cb_kCs4 = kCs4;
static __constant__ double cb_kCs2 = kCs2;
static __constant__ double cb_kHp0 = kHp0;
static __constant__ double cb_kHp1 = kHp1;
static __constant__ double cb_kToint = kToint;
static __constant__ double cb_kHpinv = kHpinv;
static __constant__ double cb_kMp1 = kMp1;
static __constant__ double cb_kMp2 = kMp2;
static __constant__ double cb_kPp3 = kPp3;
static __constant__ double cb_kPp4 = kPp4;
static __constant__ double cb_kS5 = kS5;
static __constant__ double cb_kS4 = kS4;
static __constant__ double cb_kS3 = kS3;
static __constant__ double cb_kS2 = kS2;
static __constant__ double cb_kS1 = kS1;
static __constant__ double cb_kSmall = kSmall;
#endif
#if defined(__CUDA_ARCH__) && NLK_GLIBC_CBANK
#define K_(name) cb_##name
#else
#define K_(name) name
#endif
NLK_HD double sct(int i) { return asd(NLK_PICK(sincos_tab, i)); }

NLK_HD double taylor_sin(double a, double da) {
  const double xx = a * a;
  double p = dfma(xx, K_(kS5), K_(kS4));
  p = dfma(xx, p, K_(kS3));
  p = dfma(xx, p, K_(kS2));
  p = dfma(xx, p, K_(kS1));
  double t = dfma(p, a, -(da * 0.5));
  t = dfma(xx, t, da);
  return a + t;
}
NLK_HD double do_sin_tab(double a, double da) {
  if (!(0.0 < a)) da = -da;
  const double ax = fabs(a);
  const double u = ax + K_(kBig);
  const int k = static_cast<int>(static_cast<uint32_t>(asu(u)) << 2);
  const double xr = ax - (u - K_(kBig));
  const double xx = xr * xr;
  const double a5 = dfma(xx, K_(kSn5), K_(kSn3));
  double s = dfma(xr * xx, a5, da);
  double c = dfma(xx, K_(kCs6), K_(kCs4));
  c = dfma(xx, c, K_(kCs2));
  s = xr + s;
  const double cc = xx * c;
  c = dfma(xr, da, cc);
  double t = dfma(s, sct(k + 3), sct(k + 1));
  t = dfma(-c, sct(k), t);
  const double cor = dfma(s, sct(k + 2), t);
  return copysign(sct(k) + cor, a);
}
NLK_HD double do_cos_tab(double a, double da) {
  if (a < 0.0) da = -da;
  const double ax = fabs(a);
  const double u = ax + K_(kBig);
  const int k = static_cast<int>(static_cast<uint32_t>(asu(u)) << 2);
  const double xr = (ax - (u - K_(kBig))) + da;
  const double xx = xr * xr;
  const double a5 = dfma(xx, K_(kSn5), K_(kSn3));
  const double s = dfma(xr * xx, a5, xr);
  double c = dfma(xx, K_(kCs6), K_(kCs4));
  c = dfma(xx, c, K_(kCs2));
  const double cc = xx * c;
  double t = dfma(-s, sct(k + 1), sct(k + 3));
  t = dfma(-cc, sct(k + 2), t);
  t = dfma(-s, sct(k), t);
  return sct(k + 2) + t;
}
NLK_HD double do_sin(double a, double da) {
  if (fabs(a) < K_(kSmall)) return taylor_sin(a, da);
  return do_sin_tab(a, da);
}
NLK_HD int reduce_sincos(double x, double* a, double* da) {
  const double t = dfma(x, K_(kHpinv), K_(kToint));
  const int n = static_cast<int>(static_cast<uint32_t>(asu(t)) & 3);
  const double xn = t - K_(kToint);
  double y = dfma(-xn, K_(kMp1), x);
  y = dfma(-xn, K_(kMp2), y);
  const double t2 = dfma(-xn, K_(kPp3), y);
  const double db = dfma(-xn, K_(kPp3), y - t2);
  const double b = dfma(-xn, K_(kPp4), t2);
  const double e = dfma(-xn, K_(kPp4), t2 - b);
  *a = b;
  *da = db + e;
  return n;
}
// ---- __branred (sysdeps/ieee754/dbl-64/branred.c; no FMA in this build) ------
// Payne-Hanek reduction of 105414350 <= |x| < 2^1024 by pi/2 with the
// 24-bit digits of 2/pi (toverp): returns the quadrant, *a + *aa = x mod pi/2.
// Order of operations from the libm disassembly (SSE2, no contraction).
NLK_HD void branred_half(double xh, double* b_out, double* bb_out, double* sum_out) {
  constexpr double kTm24 = 0x1p-24, kBig = 0x1.8p52, kBig1 = 0x1.8p54;
  int k = static_cast<int>((asu(xh) >> 52) & 2047);
  k = (k - 450) / 24;
  if (k < 0) k = 0;
  double gor = asd(static_cast<uint64_t>(0x63f00000u - static_cast<uint32_t>((k * 24) << 20)) << 32);
  double r[6];
  for (int i = 0; i < 6; ++i) {
    r[i] = xh * asd(NLK_PICK(toverp, k + i)) * gor;
    gor *= kTm24;
  }
  double sum = 0.0, s;
  for (int i = 0; i < 3; ++i) {
    s = (r[i] + kBig) - kBig;
    sum += s;
    r[i] -= s;
  }
  double t = 0.0;
  for (int i = 0; i < 6; ++i) t += r[5 - i];
  double bb = (((((r[0] - t) + r[1]) + r[2]) + r[3]) + r[4]) + r[5];
  s = (t + kBig) - kBig;
  sum += s;
  t -= s;
  const double b = t + bb;
  bb = (t - b) + bb;
  s = (sum + kBig1) - kBig1;
  sum -= s;
  *b_out = b;
  *bb_out = bb;
  *sum_out = sum;
}
NLK_HD int branred(double x, double* a, double* aa) {
  constexpr double kTm600 = 0x1p-600, kSplit = 134217729.0;
  constexpr double kBrMp1 = 0x1.921fb58p+0, kBrMp2 = -0x1.dde974p-27;
  x *= kTm600;
  double t = x * kSplit;
  const double x1 = t - (t - x);
  const double x2 = x - x1;
  double b1, bb1, sum1, b2, bb2, sum2;
  branred_half(x1, &b1, &bb1, &sum1);
  branred_half(x2, &b2, &bb2, &sum2);
  double sum = sum1 + sum2;
  double b = b1 + b2;
  double bb = (fabs(b1) > fabs(b2)) ? (b1 - b) + b2 : (b2 - b) + b1;
  if (b > 0.5) {
    b -= 1.0;
    sum += 1.0;
  } else if (b < -0.5) {
    b += 1.0;
    sum -= 1.0;
  }
  double s = b + (bb + bb1 + bb2);
  t = ((b - s) + bb) + (bb1 + bb2);
  b = s * kSplit;
  const double t1 = b - (b - s);
  const double t2 = s - t1;
  b = s * kHp0;
  bb = (((t1 * kBrMp1 - b) + t1 * kBrMp2) + t2 * kBrMp1) + (t2 * kBrMp2 + s * kHp1 + t * kHp0);
  s = b + bb;
  t = (b - s) + bb;
  *a = s;
  *aa = t;
  return static_cast<int>(sum) & 3;
}

NLK_HD double sin(double x) {
  const uint32_t k = static_cast<uint32_t>(asu(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) {
    if (fabs(x) < kSmall) return taylor_sin(x, 0.0);
    return do_sin_tab(x, 0.0);
  }
  if (k < 0x400368fdu) return copysign(do_cos_tab(kHp0 - fabs(x), kHp1), x);
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce_sincos(x, &a, &da);
    const double r = (n & 1) ? do_cos_tab(a, da) : do_sin(a, da);
    return (n & 2) ? -r : r;
  }
  if (k >= 0x7ff00000u) return x / x;
  double a, da;
  const int n = branred(x, &a, &da);
  const double r = (n & 1) ? do_cos_tab(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}
NLK_HD double cos(double x) {
  const uint32_t k = static_cast<uint32_t>(asu(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos_tab(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = kHp0 - fabs(x);
    const double a = y + kHp1;
    const double da = (y - a) + kHp1;
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce_sincos(x, &a, &da) + 1;
    const double r = (n & 1) ? do_cos_tab(a, da) : do_sin(a, da);
    return (n & 2) ? -r : r;
  }
  if (k >= 0x7ff00000u) return x / x;
  double a, da;
  const int n = branred(x, &a, &da) + 1;
  const double r = (n & 1) ? do_cos_tab(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}

// sin and cos of the same argument in one evaluation, each bit-identical to
// glibc's separate sin() and cos().
NLK_HD void sincos(double x, double* s, double* c) {
  const uint32_t k = static_cast<uint32_t>(asu(x) >> 32) & 0x7fffffffu;
  if (k >= 0x7ff00000u) {  // inf / NaN -> NaN (glibc: x / x)
    *s = *c = x / x;
    return;
  }
  // Every range needs exactly one evaluation of glibc's sine kernel (do_sin:
  // Taylor below 0.126, else the table) and one of its cosine kernel
  // (do_cos), at range-dependent arguments.  Classify and reduce first, then
  // evaluate each kernel once: lanes of a warp in different ranges share the
  // table code instead of running it once per range (each result is the
  // value glibc's separate sin() / cos() above return).
  double as, das, ac, dac;
  int mode, n = 0;
  if (k < 0x3feb6000u) {  // |x| < 0.855469: sin(x), cos(x) directly
    as = ac = x;
    das = dac = 0.0;
    mode = 0;
  } else if (k < 0x400368fdu) {  // |x| < 2.426265: about pi/2
    const double y = kHp0 - fabs(x);
    ac = y;  // sin(x) = copysign(do_cos(y, hp1), x)
    dac = kHp1;
    as = y + kHp1;  // cos(x) = do_sin(a, da)
    das = (y - as) + kHp1;
    mode = 1;
  } else {  // Cody-Waite below 105414350, else Payne-Hanek
    double a, da;
    n = (k < 0x419921fbu) ? reduce_sincos(x, &a, &da) : branred(x, &a, &da);
    as = ac = a;
    das = dac = da;
    mode = 2;
  }
  const double vs = (fabs(as) < kSmall) ? taylor_sin(as, das) : do_sin_tab(as, das);
  const double vc = do_cos_tab(ac, dac);
  if (mode == 0) {
    *s = (k < 0x3e500000u) ? x : vs;
    *c = (k < 0x3e400000u) ? 1.0 : vc;
  } else if (mode == 1) {
    *s = copysign(vc, x);
    *c = vs;
  } else {
    const double rs = (n & 1) ? vc : vs;
    const double rc = ((n + 1) & 1) ? vc : vs;
    *s = (n & 2) ? -rs : rs;
    *c = ((n + 1) & 2) ? -rc : rc;
  }
}

// sincos of G independent arguments, each result bit-identical to sincos()
// above, written branch-free so that the G dependency chains interleave
// (one thread evaluates a residual's G transcendentals with G-way ILP instead
// of G serial calls).  Per argument: the classification of sincos() becomes
// selects, both sine kernels (Taylor and table) are evaluated and the one
// glibc would take is kept, and the table index of lanes that take neither
// is clamped to a valid entry.  Arguments outside the Cody-Waite range
// (|x| >= 105414350, inf, NaN) are rare: they take the scalar sincos()
// afterwards: sincos_n returns true when some argument needs that, and the
// caller re-evaluates those with sincos() (sincos_n leaves them unspecified).
NLK_HD bool sincos_slow(double x) {
  return (static_cast<uint32_t>(asu(x) >> 32) & 0x7fffffffu) >= 0x419921fbu;
}
template <int G>
NLK_HD bool sincos_n(const double* x, double* s, double* c) {
  double as[G], das[G], ac[G], dac[G];
  int n[G], mode[G];
  bool slow = false;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int g = 0; g < G; ++g) {
    const uint32_t k = static_cast<uint32_t>(asu(x[g]) >> 32) & 0x7fffffffu;
    const bool big = k >= 0x419921fbu;
    slow |= big;
    const double xs = big ? 0.5 : x[g];  // keeps every table index in range
    double a, da;
    const int nn = reduce_sincos(xs, &a, &da);
    const double y = K_(kHp0) - fabs(xs);
    const double a1 = y + K_(kHp1);
    const double da1 = (y - a1) + K_(kHp1);
    const int m = (k < 0x3feb6000u) ? 0 : ((k < 0x400368fdu) ? 1 : 2);
    mode[g] = m;
    n[g] = nn;
    as[g] = m == 0 ? xs : (m == 1 ? a1 : a);
    das[g] = m == 0 ? 0.0 : (m == 1 ? da1 : da);
    ac[g] = m == 0 ? xs : (m == 1 ? y : a);
    dac[g] = m == 0 ? 0.0 : (m == 1 ? K_(kHp1) : da);
  }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int g = 0; g < G; ++g) {
    const double vt = taylor_sin(as[g], das[g]);
    const double vb = do_sin_tab(as[g], das[g]);
    const double vs = (fabs(as[g]) < K_(kSmall)) ? vt : vb;
    const double vc = do_cos_tab(ac[g], dac[g]);
    const uint32_t k = static_cast<uint32_t>(asu(x[g]) >> 32) & 0x7fffffffu;
    const int nn = n[g];
    const double rs = (nn & 1) ? vc : vs;
    const double rc = ((nn + 1) & 1) ? vc : vs;
    const double s2 = (nn & 2) ? -rs : rs;
    const double c2 = ((nn + 1) & 2) ? -rc : rc;
    const double s0 = (k < 0x3e500000u) ? x[g] : vs;
    const double c0 = (k < 0x3e400000u) ? 1.0 : vc;
    s[g] = mode[g] == 0 ? s0 : (mode[g] == 1 ? copysign(vc, x[g]) : s2);
    c[g] = mode[g] == 0 ? c0 : (mode[g] == 1 ? vs : c2);
  }
  return slow;
}

#undef K_

// ---- atan (sysdeps/ieee754/dbl-64/s_atan.c, 2.35+ table version, FMA build) --
constexpr double kA0 = 0x1.375f08b31cbcep-4, kA1 = -0x1.7458022b13c25p-4;
constexpr double kA2 = 0x1.c71c6e5129a3bp-4, kA3 = -0x1.24924923f7603p-3;
constexpr double kA4 = 0x1.99999999997fdp-3, kA5 = -0x1.5555555555555p-2;

NLK_HD double ate(int i, int j) { return asd(NLK_PICK(atan_tab, 7 * i + j)); }
NLK_HD int atan_idx(double w) {
  return static_cast<int>(dfma(w, 256.0, 0x1p52) - 0x1p52) - 16;
}
NLK_HD double atan(double x) {
  const uint64_t ix = asu(x);
  if (((ix >> 52) & 0x7ff) == 0x7ff && (ix & 0xfffffffffffffull)) return x + x;
  const double ax = fabs(x);
  if (ax < 1.0) {
    if (ax >= 0.0625) {
      const int i = atan_idx(ax);
      const double t = ax - ate(i, 0);
      double p = dfma(t, ate(i, 6), ate(i, 5));
      p = dfma(t, p, ate(i, 4));
      p = dfma(t, p, ate(i, 3));
      p = dfma(t, p, ate(i, 2));
      return copysign(dfma(p, t, ate(i, 1)), x);
    }
    if (ax >= 0x1.bb67ap-27) {
      const double xx = x * x;
      double p = dfma(xx, kA0, kA1);
      p = dfma(xx, p, kA2);
      p = dfma(xx, p, kA3);
      p = dfma(xx, p, kA4);
      p = dfma(xx, p, kA5);
      return dfma(x * xx, p, x);
    }
    return x;
  }
  if (ax < 16.0) {
    const double w = 1.0 / ax;
    const double wx = w * ax;
    const double err = dfma(ax, w, -wx);
    const double res = (1.0 - wx) - err;
    const int i = atan_idx(w);
    const double t = dfma(res, w, w - ate(i, 0));
    double p = dfma(t, ate(i, 6), ate(i, 5));
    p = dfma(t, p, ate(i, 4));
    p = dfma(t, p, ate(i, 3));
    p = dfma(t, p, ate(i, 2));
    const double q = dfma(-p, t, kHp1);
    return copysign((kHp0 - ate(i, 1)) + q, x);
  }
  if (ax < 0x1.49ff2p+52) {
    const double w = 1.0 / ax;
    const double wx = w * ax;
    const double h = kHp0 - w;
    const double ww = w * w;
    double p = dfma(ww, kA0, kA1);
    p = dfma(ww, p, kA2);
    double c = kHp0 - h;
    p = dfma(ww, p, kA3);
    const double err = dfma(ax, w, -wx);
    double res = 1.0 - wx;
    p = dfma(ww, p, kA4);
    c = c - w;
    c = c + kHp1;
    p = dfma(ww, p, kA5);
    const double www = w * ww;
    res = res - err;
    res = dfma(-res, w, c);
    const double q = dfma(-www, p, res);
    return copysign(h + q, x);
  }
  return copysign(kHp0, x);
}

}  // namespace glibc

// ---- numpy's float64 exp on the reference host -------------------------------
// numpy 2.3 on an AVX512_SKX host evaluates np.exp (arrays and scalars) with
// Intel SVML's __svml_exp8_ha (DOUBLE_exp_AVX512_SKX), not glibc: it differs
// from glibc in the last bit on ~4.5 % of inputs.  Transcribed from the
// disassembly of numpy's _multiarray_umath (constants from
// __svml_dexp_ha_data_internal_avx512).  |x| >= 707.7 takes SVML's scalar
// "rare" path, which is not reproduced (glibc's exp is used there).
namespace svml {
#define NLK_SVML_TH {0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, \
  0x1.2387a6e756238p+0, 0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, \
  0x1.5ab07dd485429p+0, 0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, \
  0x1.9c49182a3f090p+0, 0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, \
  0x1.ea4afa2a490dap+0}
#define NLK_SVML_TL {0x0.0p+0, 0x1.79aa65d837b6dp-54, -0x1.01b15eaa59348p-55, \
  0x1.68efde3a8a894p-54, 0x1.34d754db0abb6p-55, 0x1.59f48a72a4c6dp-55, 0x1.690cebb7aafb0p-56, \
  0x1.063e1e21c5409p-54, -0x1.3b3efbf5e2228p-54, -0x1.b32dcb94da51dp-56, 0x1.db72fc1f0eab4p-55, \
  0x1.1affc2b91ce27p-56, 0x1.c1a7792cb3387p-55, 0x1.36eae30af0cb3p-56, 0x1.4a385a63d07a7p-56, \
  -0x1.ff7128fd391f0p-55}
static const double h_th[16] = NLK_SVML_TH;
static const double h_tl[16] = NLK_SVML_TL;
#if defined(__CUDACC__)
static __device__ const double d_th[16] = NLK_SVML_TH;
static __device__ const double d_tl[16] = NLK_SVML_TL;
#endif
NLK_HD double th(int j) {
#if defined(__CUDA_ARCH__)
  return d_th[j];
#else
  return h_th[j];
#endif
}
NLK_HD double tl(int j) {
#if defined(__CUDA_ARCH__)
  return d_tl[j];
#else
  return h_tl[j];
#endif
}
constexpr double kInvLn2 = 0x1.71547652b82fep+0, kShifter = 0x1.8000000003ff0p+48;
constexpr double kLn2hi = 0x1.62e42fefa39efp-1, kLn2lo = 0x1.abc9e3b39803fp-56;
constexpr double kRare = 0x1.61da04cbafe44p+9;

// fma rounded toward zero (the {rz-sae} of the first SVML instruction)
NLK_HD double fma_rz(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rz(a, b, c);
#else
  // host: exact product-sum in long double is not enough; use the FPU mode
  int old = fegetround();
  fesetround(FE_TOWARDZERO);
  volatile double r = fma(a, b, c);
  fesetround(old);
  return r;
#endif
}

NLK_HD double exp(double x) {
  if (!(fabs(x) < kRare)) return glibc::exp(x);
  const double s = fma_rz(x, kInvLn2, kShifter);
  const double n = s - kShifter;
  const int j = static_cast<int>(glibc::asu(s) & 15);
  double r = glibc::dfma(-n, kLn2hi, x);
  r = glibc::dfma(-n, kLn2lo, r);
  r = glibc::asd(glibc::asu(r) & 0xbfffffffffffffffull);
  const double r2 = r * r;
  const double p1 = glibc::dfma(0x1.7411836940c04p-10, r, 0x1.1101cbbc265c0p-7);
  const double p2 = glibc::dfma(0x1.55557242d68fep-5, r, 0x1.5555553939732p-3);
  const double p3 = glibc::dfma(0x1.000000000d008p-1, r, 0x1.fffffffffff70p-1);
  double P = glibc::dfma(p1, r2, p2);
  P = glibc::dfma(P, r2, p3);
  const double q = glibc::dfma(P, r, tl(j));
  const double y = glibc::dfma(q, th(j), th(j));
  // scalef(y, n): y * 2^floor(n), exact for the non-rare range
  return ldexp(y, static_cast<int>(floor(n)));
}

// ---- np.arctan on float64 = Intel SVML __svml_atan8_ha (numpy 2.3, AVX512_SKX)
// Transcribed lane-wise from the binary (tables from
// __svml_datan_ha_data_internal_avx512).  Differs from glibc's atan in ~0.17 %
// of inputs, which is why the float path (np.arctan) and the dual path
// (Dual.arctan -> math.atan = glibc) call different functions.
#define NLK_SVML_ATAN_HI {0x0.0p+0, 0x1.f5b75f92c80ddp-3, 0x1.dac670561bb4fp-2, \
  0x1.4978fa3269ee1p-1, 0x1.921fb54442d18p-1, 0x1.cac7c57846f9ep-1, 0x1.f730bd281f69bp-1, \
  0x1.0d38f2c5ba09fp+0, 0x1.1b6e192ebbe44p+0, 0x1.270ef55a53a25p+0, 0x1.30b6d796a4da8p+0, \
  0x1.38d6a6ce13353p+0, 0x1.3fc176b7a8560p+0, 0x1.45b54837351a0p+0, 0x1.4ae10fc6589a5p+0, \
  0x1.4f68dea672617p+0, 0x1.5368c951e9cfdp+0, 0x1.56f6f33a3e6a7p+0, 0x1.5a25052114e60p+0, \
  0x1.5d013c41adabdp+0, 0x1.5f97315254857p+0, 0x1.61f06c6a92b89p+0, 0x1.6414d44094c7cp+0, \
  0x1.660b02c736a06p+0, 0x1.67d8863bc99bdp+0, 0x1.698213a9d5053p+0, 0x1.6b0bae830c070p+0, \
  0x1.6c78c7edeb195p+0, 0x1.6dcc57bb565fdp+0, 0x1.6f08f07435fecp+0, 0x1.7030cf9403197p+0, \
  0x1.7145eac2088a4p+0}
#define NLK_SVML_ATAN_LO {0x0.0p+0, 0x1.8ab6e3cf7afbdp-57, 0x1.a2b7f222f65e2p-56, \
  0x1.2419a87f2a458p-56, 0x1.1a62633145c07p-55, 0x1.0dae13ad18a6bp-55, 0x1.007887af0cbbdp-56, \
  -0x1.bd0dc231bfd70p-54, 0x1.b1b466a88828ep-54, -0x1.a66b1af5f84fbp-54, 0x1.6254cb03bb199p-54, \
  -0x1.12c77e8a80f5cp-55, -0x1.441a3bd3f1084p-59, 0x1.9e4a72eedacc4p-56, -0x1.3b03e8a27f555p-54, \
  0x1.934f9f2b0020ep-54, -0x1.96f47948a99f1p-54, -0x1.df6edd6f1ec3bp-56, 0x1.8c2d0c89de218p-56, \
  0x1.f82bba194dd5dp-54, -0x1.31151a43b51cap-55, -0x1.487d50bceb1a5p-55, -0x1.c5f60a65c7397p-54, \
  -0x1.acb6afb332a0fp-56, -0x1.9b7bd2e1e8c9cp-54, -0x1.b9839085189e3p-54, -0x1.7d1ab82ffb70bp-54, \
  0x1.9239ad620ffe2p-54, -0x1.29c86447928e7p-54, -0x1.957a7170df016p-55, -0x1.cbe1896221608p-56, \
  -0x1.fda5797b32a0bp-54}
#define NLK_RCP14_TABLE static const uint16_t h_rcp14[65536]
#include "nlk_rcp14_table.inc"
#undef NLK_RCP14_TABLE
static const double h_atan_hi[32] = NLK_SVML_ATAN_HI;
static const double h_atan_lo[32] = NLK_SVML_ATAN_LO;
#if defined(__CUDACC__)
#define NLK_RCP14_TABLE static __device__ const uint16_t d_rcp14[65536]
#include "nlk_rcp14_table.inc"
#undef NLK_RCP14_TABLE
static __device__ const double d_atan_hi[32] = NLK_SVML_ATAN_HI;
static __device__ const double d_atan_lo[32] = NLK_SVML_ATAN_LO;
#endif
NLK_HD double atan_hi(int j) {
#if defined(__CUDA_ARCH__)
  return d_atan_hi[j];
#else
  return h_atan_hi[j];
#endif
}
NLK_HD double atan_lo(int j) {
#if defined(__CUDA_ARCH__)
  return d_atan_lo[j];
#else
  return h_atan_lo[j];
#endif
}
// VRCP14PD for a positive normal input (tools/extract_rcp14.c)
NLK_HD double rcp14(double d) {
  const uint64_t u = glibc::asu(d);
  const uint32_t e = static_cast<uint32_t>(u >> 52) & 0x7ffu;
  const uint32_t m16 = static_cast<uint32_t>(u >> 36) & 0xffffu;
#if defined(__CUDA_ARCH__)
  const uint64_t t = d_rcp14[m16];
#else
  const uint64_t t = h_rcp14[m16];
#endif
  const uint64_t oe = (m16 == 0 ? 2046u : 2045u) - e;
  return glibc::asd((oe << 52) | (t << 36));
}
// x86 MINPD: (a < b) ? a : b, the second operand on NaN
NLK_HD double minpd(double a, double b) { return a < b ? a : b; }

NLK_HD double atan(double x) {
  using glibc::dfma;
  constexpr double kS = 0x1.8p50, kS4 = 0x1.8000000000010p50, kBig = 0x1p128;
  const double ax = fabs(x);
  const bool k1 = ax < 7.875;  // table range; else atan(x) = pi/2 - atan(1/x)
  // reduced argument: vreducepd(ax, 0x28) = ax - RNE(4 ax) / 4 (exact)
  const double sh = ax + kS;
  const double b = sh - kS;  // RNE(4 ax) / 4
  const double t = k1 ? ax - b : -1.0;
  const int idx = static_cast<int>(glibc::asu(sh) & 15);
  const bool k2 = sh >= kS4;  // table row 16.. (b >= 4)
  const double den = k1 ? dfma(b, ax, 1.0) : minpd(kBig, ax);
  const double r0 = rcp14(den);
  const double dm1 = den - 1.0;
  const double dlo = dfma(b, ax, -dm1);
  const double ahi = k2 ? atan_hi(16 + idx) : atan_hi(idx);
  const double e = dfma(-r0, den, 1.0);
  const double e2 = e * e;
  double r = dfma(e, r0, r0);
  const double alo = k2 ? atan_lo(16 + idx) : atan_lo(idx);
  r = dfma(e2, r, r);
  const double q = r * t;
  const double dr = dlo * r;
  double c = dfma(-r, den, 1.0);
  const double qe = dfma(r, t, -q);
  c = dfma(q, c, qe);
  const double q2 = q * q;
  if (k1) c = dfma(-dr, q, c);
  const double hi = k1 ? ahi : 0x1.921fb54442d18p+0;
  const double lo = k1 ? alo : 0x1.1a62633145c07p-54;
  const double q4 = q2 * q2;
  const double q3 = q2 * q;
  double p1 = dfma(0x1.2e9b9f5c4fe97p-4, q2, -0x1.74257c46790ccp-4);
  const double p2 = dfma(0x1.c71bfeff916a0p-4, q2, -0x1.249248eef04dap-3);
  const double cl = c + lo;
  const double s = hi + q;
  p1 = dfma(q4, p1, p2);
  const double sh2 = s - hi;
  const double p3 = dfma(0x1.999999998741ep-3, q2, -0x1.555555555554dp-2);
  const double tail = q - sh2;
  p1 = dfma(q4, p1, p3);
  const double low = cl + tail;
  p1 = dfma(q3, p1, low);
  const double res = p1 + s;
  return glibc::asd(glibc::asu(res) ^ (glibc::asu(x) & 0x8000000000000000ull));
}
}  // namespace svml
}  // namespace nlk
