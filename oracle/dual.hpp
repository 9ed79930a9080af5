// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Forward-mode dual scalar restating nlkit's `Dual` class operation for
// operation (/root/reference/pkg/src/nlkit/autodiff.py:45-233).  Every
// method below names the Python method it restates; the rounding sequence is
// identical because each Python float operation is one IEEE double
// operation and nothing is contracted (compile with -ffp-contract=off).
#pragma once
#include <cmath>

#include "npatan.hpp"
#include "npexp.hpp"

namespace oracle {

constexpr int MAXW = 16;

// Transcendentals are called through volatile pointers so the compiler can
// neither constant-fold nor rewrite them (gcc turns pow(x, 2.0) into x*x,
// but glibc's pow is not correctly rounded, and Python's `float ** 2`
// calls glibc pow).
extern double (*volatile libm_pow)(double, double);
extern double (*volatile libm_exp)(double);
extern double (*volatile libm_sin)(double);
extern double (*volatile libm_cos)(double);
extern double (*volatile libm_atan)(double);

struct Dual {
  double v;
  double d[MAXW];
  int w;
};

inline Dual mk(double v, const Dual& like) { Dual r; r.v = v; r.w = like.w; return r; }

// __add__ / __radd__ (autodiff.py:66-76)
inline Dual operator+(const Dual& a, const Dual& b) {
  Dual r = mk(a.v + b.v, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = a.d[i] + b.d[i];
  return r;
}
inline Dual operator+(const Dual& a, double c) { Dual r = a; r.v = a.v + c; return r; }
inline Dual operator+(double c, const Dual& a) { Dual r = a; r.v = a.v + c; return r; }
// __sub__ (78-86), __rsub__ (88-93)
inline Dual operator-(const Dual& a, const Dual& b) {
  Dual r = mk(a.v - b.v, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = a.d[i] - b.d[i];
  return r;
}
inline Dual operator-(const Dual& a, double c) { Dual r = a; r.v = a.v - c; return r; }
inline Dual operator-(double c, const Dual& a) {
  Dual r = mk(c - a.v, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = -a.d[i];
  return r;
}
// __mul__ / __rmul__ (95-106): partial = self.value*b + other.value*a
inline Dual operator*(const Dual& a, const Dual& b) {
  Dual r = mk(a.v * b.v, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = a.v * b.d[i] + b.v * a.d[i];
  return r;
}
inline Dual operator*(const Dual& a, double c) {
  Dual r = mk(a.v * c, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = c * a.d[i];
  return r;
}
inline Dual operator*(double c, const Dual& a) { return a * c; }
// __truediv__ (108-117): multiply by the reciprocal
inline Dual operator/(const Dual& a, const Dual& b) {
  double inv = 1.0 / b.v;
  double q = a.v * inv;
  Dual r = mk(q, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = (a.d[i] - q * b.d[i]) * inv;
  return r;
}
inline Dual operator/(const Dual& a, double c) {
  double inv = 1.0 / c;
  Dual r = mk(a.v * inv, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = a.d[i] * inv;
  return r;
}
// __rtruediv__ (119-124): partial = -q * inv * a
inline Dual operator/(double c, const Dual& a) {
  double inv = 1.0 / a.v;
  double q = c * inv;
  Dual r = mk(q, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = -q * inv * a.d[i];
  return r;
}
// __neg__ (146-147)
inline Dual operator-(const Dual& a) {
  Dual r = mk(-a.v, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = -a.d[i];
  return r;
}
// comparisons act on the value (158-177)
inline bool operator>(const Dual& a, double c) { return a.v > c; }
inline bool operator<(const Dual& a, double c) { return a.v < c; }
inline bool operator>=(const Dual& a, double c) { return a.v >= c; }
inline bool operator!=(const Dual& a, double c) { return a.v != c; }
inline double value(const Dual& a) { return a.v; }
inline double value(double a) { return a; }

// __pow__ n == 2 (132-134)
inline Dual pow2(const Dual& a) {
  Dual r = mk(a.v * a.v, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = 2.0 * a.v * a.d[i];
  return r;
}
// __pow__ n == 3 (135-136): c = 3 * value**2 (Python float pow), value**3
inline Dual pow3(const Dual& a) {
  double c = 3.0 * libm_pow(a.v, 2.0);
  Dual r = mk(libm_pow(a.v, 3.0), a);
  for (int i = 0; i < a.w; ++i) r.d[i] = c * a.d[i];
  return r;
}
// exp (189-191) — math.exp
inline Dual np_exp(const Dual& a) {
  double e = libm_exp(a.v);
  Dual r = mk(e, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = e * a.d[i];
  return r;
}
// sqrt (197-200)
inline Dual np_sqrt(const Dual& a) {
  double s = std::sqrt(a.v);
  double c = 0.5 / s;
  Dual r = mk(s, a);
  for (int i = 0; i < a.w; ++i) r.d[i] = c * a.d[i];
  return r;
}
// sin (202-204)
inline Dual np_sin(const Dual& a) {
  double c = libm_cos(a.v);
  Dual r = mk(libm_sin(a.v), a);
  for (int i = 0; i < a.w; ++i) r.d[i] = c * a.d[i];
  return r;
}
// cos (206-208): partial = -s * a
inline Dual np_cos(const Dual& a) {
  double s = libm_sin(a.v);
  Dual r = mk(libm_cos(a.v), a);
  for (int i = 0; i < a.w; ++i) r.d[i] = -s * a.d[i];
  return r;
}
// arctan (214-217): c = 1/(1 + v*v)
inline Dual np_arctan(const Dual& a) {
  double c = 1.0 / (1.0 + a.v * a.v);
  Dual r = mk(libm_atan(a.v), a);
  for (int i = 0; i < a.w; ++i) r.d[i] = c * a.d[i];
  return r;
}

// Float-path counterparts: numpy float64 scalar / array ufuncs.  numpy's
// float64 sin/cos equal glibc's; numpy's exp and arctan are Intel SVML on the
// reference host (npexp.hpp, npatan.hpp), not glibc.
inline double pow2(double x) { return libm_pow(x, 2.0); }
inline double pow3(double x) { return libm_pow(x, 3.0); }
inline double np_exp(double x) { return svml_exp(x); }
inline double np_sqrt(double x) { return std::sqrt(x); }
inline double np_sin(double x) { return libm_sin(x); }
inline double np_cos(double x) { return libm_cos(x); }
inline double np_arctan(double x) { return svml_atan(x); }

}  // namespace oracle
