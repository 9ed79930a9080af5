// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// The built-in residuals of /root/reference/pkg/src/nlkit/problems.py,
// written once as templates over the scalar type S:
//   S = double : the reference's float path (numpy float64 scalars/arrays,
//                CountedResidual.at, core.py:119-123)
//   S = Dual   : the reference's dual path (object arrays of Dual,
//                autodiff.forward_sweep, autodiff.py:286-309)
// Where numpy evaluates the two paths differently (pairwise vs sequential
// sums, BLAS vs object matmul) the overloads below follow each path.
#pragma once
#include "blas_models.hpp"
#include "dual.hpp"

namespace oracle {

// ---- path-dependent reductions ---------------------------------------------
// numpy float64 add.reduce: pairwise with 8 accumulators for n >= 8,
// sequential from 0.0 below (numpy/_core/src/umath/loops_utils.h.src).
inline double np_sum(const double* x, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = r + x[i];
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = x[j];
  int nb = n - (n % 8);
  for (int i = 8; i < nb; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = r[j] + x[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (int i = nb; i < n; ++i) res = res + x[i];
  return res;
}
// object-array add.reduce: strictly left to right from the first element
inline Dual np_sum(const Dual* x, int n) {
  Dual r = x[0];
  for (int i = 1; i < n; ++i) r = r + x[i];
  return r;
}
inline double np_prod(const double* x, int n) {
  double r = 1.0;
  for (int i = 0; i < n; ++i) r = r * x[i];
  return r;
}
inline Dual np_prod(const Dual* x, int n) {
  Dual r = x[0];
  for (int i = 1; i < n; ++i) r = r * x[i];
  return r;
}
// A @ x with a float64 C-ordered A: BLAS dgemv (float path) or numpy's
// object matmul inner loop (first product, then sequential adds).
inline void np_matvec(const double* A, const double* x, double* y, int n) { gemv_A_x(n, A, x, y); }
inline void np_matvec(const double* A, const Dual* x, Dual* y, int n) {
  for (int i = 0; i < n; ++i) {
    Dual s = x[0] * A[i * n];
    for (int k = 1; k < n; ++k) s = s + x[k] * A[i * n + k];
    y[i] = s;
  }
}
// X @ X for a 3x3 X: dgemm on floats (sequential FMA chain from a plain
// product), object matmul on duals.
inline void np_matmul3(const double* X, double* R) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double t = X[i * 3 + 0] * X[0 * 3 + j];
      t = std::fma(X[i * 3 + 1], X[1 * 3 + j], t);
      t = std::fma(X[i * 3 + 2], X[2 * 3 + j], t);
      R[i * 3 + j] = t;
    }
}
inline void np_matmul3(const Dual* X, Dual* R) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      Dual s = X[i * 3 + 0] * X[0 * 3 + j];
      s = s + X[i * 3 + 1] * X[1 * 3 + j];
      s = s + X[i * 3 + 2] * X[2 * 3 + j];
      R[i * 3 + j] = s;
    }
}

inline double zero_like(double) { return 0.0; }
inline Dual zero_like(const Dual& x) { Dual r = x; r.v = 0.0; for (int i = 0; i < x.w; ++i) r.d[i] = 0.0; return r; }

constexpr double PI = 3.141592653589793;

// ---- the 23-member suite (problems.py:36-292) --------------------------------
template <class S> void r_rosenbrock(const S* x, const double*, S* out, int) {  // 36-40
  out[0] = 1.0 - x[0];
  out[1] = 10.0 * (x[1] - x[0] * x[0]);
}
template <class S> void r_powell_singular(const S* x, const double*, S* out, int) {  // 43-49
  out[0] = x[0] + 10.0 * x[1];
  out[1] = 2.23606797749979 * (x[2] - x[3]);  // math.sqrt(5.0)
  out[2] = pow2(x[1] - 2.0 * x[2]);
  out[3] = 3.1622776601683795 * pow2(x[0] - x[3]);  // math.sqrt(10.0)
}
template <class S> void r_powell_badly_scaled(const S* x, const double*, S* out, int) {  // 52-56
  out[0] = 1e4 * x[0] * x[1] - 1.0;
  out[1] = np_exp(-x[0]) + np_exp(-x[1]) - 1.0001;
}
template <class S> void r_wood(const S* x, const double*, S* out, int) {  // 59-67
  out[0] = -200.0 * x[0] * (x[1] - pow2(x[0])) - (1.0 - x[0]);
  out[1] = (200.0 * (x[1] - pow2(x[0])) + 20.2 * (x[1] - 1.0) + 19.8 * (x[3] - 1.0));
  out[2] = -180.0 * x[2] * (x[3] - pow2(x[2])) - (1.0 - x[2]);
  out[3] = (180.0 * (x[3] - pow2(x[2])) + 20.2 * (x[3] - 1.0) + 19.8 * (x[1] - 1.0));
}
template <class S> void r_helical_valley(const S* x, const double*, S* out, int) {  // 70-81
  const double twopi = 2.0 * PI;
  if (x[0] > 0.0) {
    S angle = np_arctan(x[1] / x[0]) / twopi;
    out[0] = 10.0 * (x[2] - 10.0 * angle);
  } else if (x[0] < 0.0) {
    S angle = np_arctan(x[1] / x[0]) / twopi + 0.5;
    out[0] = 10.0 * (x[2] - 10.0 * angle);
  } else {
    double angle = (x[1] >= 0.0) ? 0.25 : -0.25;
    out[0] = 10.0 * (x[2] - 10.0 * angle);
  }
  out[1] = 10.0 * (np_sqrt(x[0] * x[0] + x[1] * x[1]) - 1.0);
  out[2] = x[2];
}
template <class S> void r_watson(const S* x, const double*, S* out, int n) {  // 84-109
  bool started[16] = {false};
  for (int i = 1; i < 30; ++i) {
    double ti = i / 29.0;
    S sum1 = zero_like(x[0]);
    bool s1 = false;
    double temp = 1.0;
    for (int j = 1; j < n; ++j) {
      S term = (j * temp) * x[j];
      sum1 = s1 ? sum1 + term : 0.0 + term;
      s1 = true;
      temp = temp * ti;
    }
    S sum2 = zero_like(x[0]);
    temp = 1.0;
    for (int j = 0; j < n; ++j) {
      S term = temp * x[j];
      sum2 = (j > 0) ? sum2 + term : 0.0 + term;
      temp = temp * ti;
    }
    S temp1 = (s1 ? sum1 - sum2 * sum2 : 0.0 - sum2 * sum2) - 1.0;
    S temp2 = 2.0 * ti * sum2;
    temp = 1.0 / ti;
    for (int k = 0; k < n; ++k) {
      S term = temp * (double(k) - temp2) * temp1;
      out[k] = started[k] ? out[k] + term : 0.0 + term;
      started[k] = true;
      temp = temp * ti;
    }
  }
  S t = x[1] - x[0] * x[0] - 1.0;
  out[0] = out[0] + x[0] * (1.0 - 2.0 * t);
  out[1] = out[1] + t;
}
template <class S> void r_chebyquad(const S* x, const double*, S* out, int n) {  // 112-129
  bool started[16] = {false};
  for (int j = 0; j < n; ++j) {
    // t_prev starts as the float 1.0
    S t_cur = 2.0 * x[j] - 1.0;
    S scale = 2.0 * t_cur;
    S t_prev = zero_like(x[0]);
    bool prev_is_one = true;
    for (int i = 0; i < n; ++i) {
      out[i] = started[i] ? out[i] + t_cur : 0.0 + t_cur;
      started[i] = true;
      S t_next = prev_is_one ? scale * t_cur - 1.0 : scale * t_cur - t_prev;
      t_prev = t_cur;
      prev_is_one = false;
      t_cur = t_next;
    }
  }
  for (int k = 0; k < n; ++k) {
    out[k] = out[k] / double(n);
    if ((k + 1) % 2 == 0) out[k] = out[k] + 1.0 / (double((k + 1) * (k + 1)) - 1.0);
  }
}
template <class S> void r_brown_almost_linear(const S* x, const double*, S* out, int n) {  // 132-139
  S total = np_sum(x, n);
  for (int k = 0; k < n - 1; ++k) out[k] = x[k] + total - (n + 1.0);
  out[n - 1] = np_prod(x, n) - 1.0;
}
template <class S> void r_discrete_boundary_value(const S* x, const double*, S* out, int n) {  // 142-151
  double h = 1.0 / (n + 1);
  for (int k = 0; k < n; ++k) {
    double tk = (k + 1) * h;
    S a = 2.0 * x[k];
    a = (k > 0) ? a - x[k - 1] : a - 0.0;
    a = (k < n - 1) ? a - x[k + 1] : a - 0.0;
    out[k] = a + 0.5 * h * h * pow3(x[k] + tk + 1.0);
  }
}
template <class S> void r_discrete_integral(const S* x, const double*, S* out, int n) {  // 154-168
  double h = 1.0 / (n + 1);
  double t[16];
  for (int j = 0; j < n; ++j) t[j] = (j + 1) * h;
  S cubes[16];
  for (int j = 0; j < n; ++j) cubes[j] = pow3(x[j] + t[j] + 1.0);
  for (int k = 0; k < n; ++k) {
    S s1 = 0.0 + t[0] * cubes[0];
    for (int j = 1; j <= k; ++j) s1 = s1 + t[j] * cubes[j];
    S inner = (1.0 - t[k]) * s1;
    if (k + 1 < n) {
      S s2 = 0.0 + (1.0 - t[k + 1]) * cubes[k + 1];
      for (int j = k + 2; j < n; ++j) s2 = s2 + (1.0 - t[j]) * cubes[j];
      inner = inner + t[k] * s2;
    } else {
      inner = inner + t[k] * 0.0;
    }
    out[k] = x[k] + 0.5 * h * inner;
  }
}
template <class S> void r_trigonometric(const S* x, const double*, S* out, int n) {  // 171-177
  S c[16];
  for (int k = 0; k < n; ++k) c[k] = np_cos(x[k]);
  S cos_sum = np_sum(c, n);
  for (int k = 0; k < n; ++k)
    out[k] = double(n) - cos_sum + double(k + 1) * (1.0 - np_cos(x[k])) - np_sin(x[k]);
}
template <class S> void r_variably_dimensioned(const S* x, const double*, S* out, int n) {  // 180-188
  S w[16] = {};
  for (int k = 0; k < n; ++k) w[k] = double(k + 1) * (x[k] - 1.0);
  S s = np_sum(w, n);
  S temp = s * (1.0 + 2.0 * s * s);
  for (int k = 0; k < n; ++k) out[k] = x[k] - 1.0 + double(k + 1) * temp;
}
template <class S> void r_broyden_tridiagonal(const S* x, const double*, S* out, int n) {  // 191-198
  for (int k = 0; k < n; ++k) {
    S a = (3.0 - 2.0 * x[k]) * x[k];
    a = (k > 0) ? a - x[k - 1] : a - 0.0;
    a = (k < n - 1) ? a - 2.0 * x[k + 1] : a - 2.0 * 0.0;
    out[k] = a + 1.0;
  }
}
template <class S> void r_broyden_banded(const S* x, const double*, S* out, int n) {  // 201-210
  for (int k = 0; k < n; ++k) {
    S acc = zero_like(x[0]);
    bool first = true;
    int lo = k - 5 > 0 ? k - 5 : 0;
    int hi = k + 2 < n ? k + 2 : n;
    for (int j = lo; j < hi; ++j) {
      if (j == k) continue;
      S term = x[j] * (1.0 + x[j]);
      acc = first ? 0.0 + term : acc + term;
      first = false;
    }
    S a = x[k] * (2.0 + 5.0 * x[k] * x[k]) + 1.0;
    out[k] = first ? a - 0.0 : a - acc;
  }
}
template <class S> void r_matrix_sqrt_2x2(const S* x, const double*, S* out, int) {  // 213-220
  out[0] = x[0] * x[0] + x[1] * x[2] - 1e-4;
  out[1] = x[0] * x[1] + x[1] * x[3] - 1.0;
  out[2] = x[2] * x[0] + x[3] * x[2];
  out[3] = x[2] * x[1] + x[3] * x[3] - 1e-4;
}
template <class S> void r_matrix_sqrt_3x3(const S* x, const double*, S* out, int) {  // 223-230
  S R[9];
  np_matmul3(x, R);
  for (int k = 0; k < 9; ++k) {
    double a = (k == 0 || k == 4 || k == 8) ? 1e-4 : (k == 1 ? 1.0 : 0.0);
    out[k] = R[k] - a;
  }
}
template <class S> void r_dennis_schnabel(const S* x, const double*, S* out, int) {  // 233-237
  out[0] = x[0] * x[0] + x[1] * x[1] - 2.0;
  out[1] = np_exp(x[0] - 1.0) + pow3(x[1]) - 2.0;
}
template <class S> void r_product_exponential(const S* x, const double*, S* out, int) {  // 240-251
  if (x[0] != 0.0) out[0] = x[1] * x[1] * (1.0 - np_exp(-x[0] * x[0])) / x[0];
  else out[0] = 0.0 * x[1];
  if (x[1] != 0.0) out[1] = x[0] * (1.0 - np_exp(-x[1] * x[1])) / x[1];
  else out[1] = 0.0 * x[0];
}
template <class S> void r_cubic_radial(const S* x, const double*, S* out, int) {  // 254-260
  S r2 = x[0] * x[0] + x[1] * x[1];
  out[0] = x[0] * r2;
  out[1] = x[1] * r2;
}
template <class S> void r_double_root_scalar(const S* x, const double*, S* out, int) {  // 263-266
  out[0] = x[0] * pow2(x[0] - 5.0);
}
template <class S> void r_freudenstein_roth(const S* x, const double*, S* out, int) {  // 269-273
  out[0] = -13.0 + x[0] + ((5.0 - x[1]) * x[1] - 2.0) * x[1];
  out[1] = -29.0 + x[0] + ((1.0 + x[1]) * x[1] - 14.0) * x[1];
}
template <class S> void r_boggs(const S* x, const double*, S* out, int) {  // 276-280
  out[0] = x[0] * x[0] - x[1] + 1.0;
  out[1] = x[0] - np_cos(0.5 * PI * x[1]);
}
template <class S> void r_chandrasekhar(const S* x, const double*, S* out, int n) {  // 286-292
  double mu[16], A[256];
  for (int i = 0; i < n; ++i) mu[i] = ((i + 1) - 0.5) / n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A[i * n + j] = mu[i] / (mu[i] + mu[j]);
  S y[16];
  np_matvec(A, x, y, n);
  const double c = 0.9 / (2.0 * n);
  for (int i = 0; i < n; ++i) out[i] = x[i] - 1.0 / (1.0 - c * y[i]);
}

// ---- parametrised families (problems.py:358-387, 191-198) --------------------
template <class S> void r_generalized_rosenbrock(const S* x, const double*, S* out, int n) {  // 363-368
  out[0] = 1.0 - x[0];
  for (int i = 1; i < n; ++i) out[i] = 10.0 * (x[i] - x[i - 1] * x[i - 1]);
}
template <class S> void r_quadratic(const S* x, const double* p, S* out, int n) {  // 382-383
  for (int i = 0; i < n; ++i) out[i] = x[i] * x[i] - p[i];
}

}  // namespace oracle
