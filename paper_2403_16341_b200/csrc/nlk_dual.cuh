// Forward-mode dual numbers on the device.
//
// Operation-for-operation the arithmetic of nlkit's Dual
// (/root/reference/pkg/src/nlkit/autodiff.py:45-233) so the device Jacobian is
// bit-identical to the reference's (the library is compiled with
// -fmad=false: nothing is contracted unless written as fma()).  W is the seed
// width of one sweep; the kernels use W = n (one sweep per Jacobian) — every
// Dual op is componentwise in the partials, so any width gives the same bits
// as the reference's SEED_WIDTH = 8 chunks (SURVEY.md §7 "Register pressure").
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "nlk_glibc.cuh"

namespace nlk {

template <class T> struct Num;  // numeric constants per precision
template <> struct Num<double> {
  static constexpr double eps = 2.220446049250313e-16;   // np.finfo(float).eps
  static constexpr double tiny = 1e-300;                 // solvers.py:22, descent.py:231
  static constexpr double radius_floor = 1e-308;         // globalize.py:153
  static constexpr double radius_stop = 1e-300;          // globalize.py:212
  static constexpr double dbl_min = 2.2250738585072014e-308;
};
template <> struct Num<float> {
  static constexpr float eps = 1.1920929e-07f;
  static constexpr float tiny = 1e-37f;
  static constexpr float radius_floor = 1e-37f;
  static constexpr float radius_stop = 1e-36f;
  static constexpr float dbl_min = 1.17549435e-38f;
};

template <int W, class T>
struct Dual {
  T v;
  T d[W];
};

template <class S> struct ScalarOf { using type = S; };
template <int W, class T> struct ScalarOf<Dual<W, T>> { using type = T; };

// ---- elementary functions --------------------------------------------------------
// fp64: the reference host's own algorithms (nlk_glibc.cuh): glibc for
// CPython's math module, numpy's sin/cos and `x ** n`; Intel SVML for numpy's
// float64 exp and arctan (np.exp / np.arctan on the float path; the dual path
// calls math.exp / math.atan).
// fp32: CUDA's single-precision functions (no reference exists for fp32).
// Out of line: a residual like test23/trigonometric makes ~60 of these calls
// per iteration, and inlining each body blew the kernel up to ~25k
// instructions (instruction-fetch stalls dominated, ncu).
#ifndef NLK_INLINE_TRANS
#define NLK_INLINE_TRANS 0
#endif
#if NLK_INLINE_TRANS
#define NLK_TRANS_ATTR static __device__ __forceinline__
#else
#define NLK_TRANS_ATTR static __device__ __noinline__
#endif
NLK_TRANS_ATTR double nlk_exp(double x) { return glibc::exp(x); }      // math.exp (Dual path)
NLK_TRANS_ATTR double nlk_np_exp(double x) { return svml::exp(x); }   // np.exp on float64
NLK_TRANS_ATTR float nlk_exp(float x) { return expf(x); }
NLK_TRANS_ATTR double nlk_sin(double x) { return glibc::sin(x); }
NLK_TRANS_ATTR float nlk_sin(float x) { return sinf(x); }
NLK_TRANS_ATTR double nlk_cos(double x) { return glibc::cos(x); }
NLK_TRANS_ATTR float nlk_cos(float x) { return cosf(x); }
NLK_TRANS_ATTR double nlk_atan(double x) { return glibc::atan(x); }      // math.atan (Dual path)
NLK_TRANS_ATTR double nlk_np_atan(double x) { return svml::atan(x); }  // np.arctan on float64
NLK_TRANS_ATTR double nlk_pow2(double x) { return glibc::pow_int<2>(x); }
// sin and cos returned by value (registers): through pointers the call
// became two local-memory stores in the callee and two loads in the caller
struct SinCos { double s, c; };
NLK_TRANS_ATTR SinCos nlk_sincos_v(double x) {
  SinCos r;
  glibc::sincos(x, &r.s, &r.c);
  return r;
}
// two arguments per out-of-line call, evaluated branch-free side by side
// (glibc::sincos_n<2>; the rare Payne-Hanek / non-finite arguments take the
// scalar port inside the call): NLK_SINCOS_PAIRS
struct SinCos2 { double s0, c0, s1, c1; };
NLK_TRANS_ATTR SinCos2 nlk_sincos2_v(double x0, double x1) {
  double x[2] = {x0, x1}, sv[2], cv[2];
  if (glibc::sincos_n<2>(x, sv, cv)) {
    if (glibc::sincos_slow(x0)) glibc::sincos(x0, &sv[0], &cv[0]);
    if (glibc::sincos_slow(x1)) glibc::sincos(x1, &sv[1], &cv[1]);
  }
  return SinCos2{sv[0], cv[0], sv[1], cv[1]};
}
__device__ __forceinline__ void nlk_sincos(double x, double* s, double* c) {
  const SinCos r = nlk_sincos_v(x);
  *s = r.s;
  *c = r.c;
}
NLK_TRANS_ATTR void nlk_sincos(float x, float* s, float* c) { sincosf(x, s, c); }
NLK_TRANS_ATTR double nlk_pow3(double x) { return glibc::pow_int<3>(x); }
NLK_TRANS_ATTR float nlk_atan(float x) { return atanf(x); }
__device__ __forceinline__ double t_exp(double x) { return nlk_np_exp(x); }
__device__ __forceinline__ float t_exp(float x) { return nlk_exp(x); }
__device__ __forceinline__ double t_exp_math(double x) { return nlk_exp(x); }
__device__ __forceinline__ float t_exp_math(float x) { return nlk_exp(x); }
__device__ __forceinline__ double t_sin(double x) { return nlk_sin(x); }
__device__ __forceinline__ float t_sin(float x) { return nlk_sin(x); }
__device__ __forceinline__ double t_cos(double x) { return nlk_cos(x); }
__device__ __forceinline__ float t_cos(float x) { return nlk_cos(x); }
__device__ __forceinline__ double t_atan(double x) { return nlk_np_atan(x); }
__device__ __forceinline__ float t_atan(float x) { return nlk_atan(x); }
__device__ __forceinline__ double t_atan_math(double x) { return nlk_atan(x); }
__device__ __forceinline__ float t_atan_math(float x) { return nlk_atan(x); }
__device__ __forceinline__ double t_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float t_sqrt(float x) { return sqrtf(x); }
// Python `x ** 2` / `x ** 3` (numpy float64 scalars and CPython floats) call
// glibc pow, which is not correctly rounded; Dual ** 2 is v*v (autodiff.py:133).
__device__ __forceinline__ double t_pow2(double x) { return nlk_pow2(x); }
__device__ __forceinline__ float t_pow2(float x) { return x * x; }
__device__ __forceinline__ double t_pow3(double x) { return nlk_pow3(x); }
__device__ __forceinline__ float t_pow3(float x) { return x * x * x; }

// ---- Dual arithmetic (autodiff.py:66-154) ----------------------------------
#define NLK_D template <int W, class T> __device__ __forceinline__

NLK_D Dual<W, T> operator+(const Dual<W, T>& a, const Dual<W, T>& b) {
  Dual<W, T> r; r.v = a.v + b.v;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = a.d[i] + b.d[i];
  return r;
}
NLK_D Dual<W, T> operator+(const Dual<W, T>& a, T c) { Dual<W, T> r = a; r.v = a.v + c; return r; }
NLK_D Dual<W, T> operator+(T c, const Dual<W, T>& a) { Dual<W, T> r = a; r.v = a.v + c; return r; }
NLK_D Dual<W, T> operator-(const Dual<W, T>& a, const Dual<W, T>& b) {
  Dual<W, T> r; r.v = a.v - b.v;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = a.d[i] - b.d[i];
  return r;
}
NLK_D Dual<W, T> operator-(const Dual<W, T>& a, T c) { Dual<W, T> r = a; r.v = a.v - c; return r; }
NLK_D Dual<W, T> operator-(T c, const Dual<W, T>& a) {  // __rsub__
  Dual<W, T> r; r.v = c - a.v;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = -a.d[i];
  return r;
}
NLK_D Dual<W, T> operator-(const Dual<W, T>& a) {
  Dual<W, T> r; r.v = -a.v;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = -a.d[i];
  return r;
}
NLK_D Dual<W, T> operator*(const Dual<W, T>& a, const Dual<W, T>& b) {  // self.v*b + other.v*a
  Dual<W, T> r; r.v = a.v * b.v;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = a.v * b.d[i] + b.v * a.d[i];
  return r;
}
NLK_D Dual<W, T> operator*(const Dual<W, T>& a, T c) {
  Dual<W, T> r; r.v = a.v * c;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = c * a.d[i];
  return r;
}
NLK_D Dual<W, T> operator*(T c, const Dual<W, T>& a) { return a * c; }
NLK_D Dual<W, T> operator/(const Dual<W, T>& a, const Dual<W, T>& b) {  // reciprocal form
  T inv = T(1) / b.v;
  T q = a.v * inv;
  Dual<W, T> r; r.v = q;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = (a.d[i] - q * b.d[i]) * inv;
  return r;
}
NLK_D Dual<W, T> operator/(const Dual<W, T>& a, T c) {
  T inv = T(1) / c;
  Dual<W, T> r; r.v = a.v * inv;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = a.d[i] * inv;
  return r;
}
NLK_D Dual<W, T> operator/(T c, const Dual<W, T>& a) {  // __rtruediv__
  T inv = T(1) / a.v;
  T q = c * inv;
  Dual<W, T> r; r.v = q;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = -q * inv * a.d[i];
  return r;
}
NLK_D bool operator>(const Dual<W, T>& a, T c) { return a.v > c; }
NLK_D bool operator<(const Dual<W, T>& a, T c) { return a.v < c; }
NLK_D bool operator>=(const Dual<W, T>& a, T c) { return a.v >= c; }
NLK_D bool operator!=(const Dual<W, T>& a, T c) { return a.v != c; }

// __pow__ n == 2 / n == 3 (autodiff.py:132-136)
NLK_D Dual<W, T> t_pow2(const Dual<W, T>& a) {
  Dual<W, T> r; r.v = a.v * a.v;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = T(2) * a.v * a.d[i];
  return r;
}
NLK_D Dual<W, T> t_pow3(const Dual<W, T>& a) {
  T c = T(3) * t_pow2(a.v);
  Dual<W, T> r; r.v = t_pow3(a.v);
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = c * a.d[i];
  return r;
}
// elementary functions (autodiff.py:189-217)
NLK_D Dual<W, T> t_exp(const Dual<W, T>& a) {
  T e = t_exp_math(a.v);  // Dual.exp calls math.exp (autodiff.py:25-26, 189-191)
  Dual<W, T> r; r.v = e;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = e * a.d[i];
  return r;
}
NLK_D Dual<W, T> t_sqrt(const Dual<W, T>& a) {
  T s = t_sqrt(a.v);
  T c = T(0.5) / s;
  Dual<W, T> r; r.v = s;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = c * a.d[i];
  return r;
}
NLK_D Dual<W, T> t_sin(const Dual<W, T>& a) {
  T sv, c;
  nlk_sincos(a.v, &sv, &c);  // = math.sin(v), math.cos(v), one call
  Dual<W, T> r; r.v = sv;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = c * a.d[i];
  return r;
}
NLK_D Dual<W, T> t_cos(const Dual<W, T>& a) {
  T s, cv;
  nlk_sincos(a.v, &s, &cv);
  Dual<W, T> r; r.v = cv;
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = -s * a.d[i];
  return r;
}
NLK_D Dual<W, T> t_atan(const Dual<W, T>& a) {
  T c = T(1) / (T(1) + a.v * a.v);
  Dual<W, T> r; r.v = t_atan_math(a.v);  // Dual.arctan calls math.atan (autodiff.py:214-217)
#pragma unroll
  for (int i = 0; i < W; ++i) r.d[i] = c * a.d[i];
  return r;
}
#undef NLK_D

// sin and cos of one value (residuals that use both call this once)
__device__ __forceinline__ void t_sincos(double x, double& s, double& c) { nlk_sincos(x, &s, &c); }
__device__ __forceinline__ void t_sincos(float x, float& s, float& c) { nlk_sincos(x, &s, &c); }
template <int W, class T>
__device__ __forceinline__ void t_sincos(const Dual<W, T>& a, Dual<W, T>& s, Dual<W, T>& c) {
  T sv, cv;
  nlk_sincos(a.v, &sv, &cv);
  s.v = sv;
  c.v = cv;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    s.d[i] = cv * a.d[i];   // Dual.sin: c * a  (autodiff.py:202-204)
    c.d[i] = -sv * a.d[i];  // Dual.cos: -s * a (autodiff.py:206-208)
  }
}

__device__ __forceinline__ double value_of(double x) { return x; }
__device__ __forceinline__ float value_of(float x) { return x; }
template <int W, class T> __device__ __forceinline__ T value_of(const Dual<W, T>& x) { return x.v; }

}  // namespace nlk
