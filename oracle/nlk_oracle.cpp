// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's per-system solve path
// (/root/reference/pkg/src/nlkit) used as the parity checker for the CUDA
// kernels.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
// leg may load this library; the product (paper_2403_16341_b200) never does.
//
// What is restated, with the reference lines each function follows:
//   newton_raphson  solvers.py:179-287 (NR branch of run_newton_family)
//   trust_region    globalize.py:156-214 + descent.py:78-106 (dogleg)
//                   + globalize.py:116-153 (ratio, radius update)
//   quasi_newton    solvers.py:290-358 + quasinewton.py:66-198
//                   (dense inverse Broyden / diagonal Klement)
//   newton_linesearch solvers.py:263-276 + globalize.py:40-74
//   dfsane          builder-authored (the reference has no DFSane; SURVEY.md
//                   App. C) — parity UNPINNED against the reference
//   dense_jacobian  autodiff.py:286-309, 342-355 (one width-n sweep; the
//                   per-chunk nf accounting of SEED_WIDTH=8 is reproduced)
//   lu_factor       linalg.py:87-105 (+ blas_models.hpp getrf/getrs)
// Built by oracle/Makefile with -O2 -ffp-contract=off (no FMA contraction:
// numpy and CPython round every operation).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "blas_models.hpp"
#include "dual.hpp"
#include "residuals.hpp"

namespace oracle {

double (*volatile libm_pow)(double, double) = ::pow;
double (*volatile libm_exp)(double) = ::exp;
double (*volatile libm_sin)(double) = ::sin;
double (*volatile libm_cos)(double) = ::cos;
double (*volatile libm_atan)(double) = ::atan;

enum RetCode : int8_t {  // core.py:17-24, declaration order
  SUCCESS = 0, MAXITERS = 1, LINESEARCH_FAILED = 2, LINSOLVE_FAILED = 3,
  STALLED = 4, NONFINITE = 5
};
enum Alg : int { NR = 0, TR = 1, BROYDEN = 2, KLEMENT = 3, DFSANE = 4, NEWTON_LS = 5 };

using FloatRes = void (*)(const double*, const double*, double*, int);
using DualRes = void (*)(const Dual*, const double*, Dual*, int);

struct ProblemDef {
  const char* id;
  int n;          // 0 = any n (n-generic family)
  int m;          // params length: -1 means m == n
  FloatRes f;
  DualRes fd;
};

#define PROB(id, n, m, fn) {id, n, m, fn<double>, fn<Dual>}
// Handles follow the order below; the product registry uses the same ids.
static const ProblemDef kProblems[] = {
    PROB("test23/rosenbrock", 2, 0, r_rosenbrock),
    PROB("test23/powell-singular", 4, 0, r_powell_singular),
    PROB("test23/powell-badly-scaled", 2, 0, r_powell_badly_scaled),
    PROB("test23/wood", 4, 0, r_wood),
    PROB("test23/helical-valley", 3, 0, r_helical_valley),
    PROB("test23/watson", 2, 0, r_watson),
    PROB("test23/chebyquad", 2, 0, r_chebyquad),
    PROB("test23/brown-almost-linear", 10, 0, r_brown_almost_linear),
    PROB("test23/discrete-boundary-value", 10, 0, r_discrete_boundary_value),
    PROB("test23/discrete-integral", 10, 0, r_discrete_integral),
    PROB("test23/trigonometric", 10, 0, r_trigonometric),
    PROB("test23/variably-dimensioned", 10, 0, r_variably_dimensioned),
    PROB("test23/broyden-tridiagonal", 0, 0, r_broyden_tridiagonal),
    PROB("test23/broyden-banded", 10, 0, r_broyden_banded),
    PROB("test23/matrix-sqrt-2x2", 4, 0, r_matrix_sqrt_2x2),
    PROB("test23/matrix-sqrt-3x3", 9, 0, r_matrix_sqrt_3x3),
    PROB("test23/dennis-schnabel", 2, 0, r_dennis_schnabel),
    PROB("test23/product-exponential", 2, 0, r_product_exponential),
    PROB("test23/cubic-radial", 2, 0, r_cubic_radial),
    PROB("test23/double-root-scalar", 1, 0, r_double_root_scalar),
    PROB("test23/freudenstein-roth", 2, 0, r_freudenstein_roth),
    PROB("test23/boggs", 2, 0, r_boggs),
    PROB("test23/chandrasekhar", 10, 0, r_chandrasekhar),
    PROB("generalized_rosenbrock", 0, 0, r_generalized_rosenbrock),
    PROB("quadratic", 0, -1, r_quadratic),
};
static const int kNumProblems = sizeof(kProblems) / sizeof(kProblems[0]);

struct Ctx {
  const ProblemDef* prob;
  int n;
  const double* p;
  int nf = 0, njac = 0, nlinsolve = 0, nsteps = 0;
  int nudge = 0;  // +1/-1: move every float-residual component one ulp (sensitivity mask)

  void F(const double* u, double* f) {  // CountedResidual.at (core.py:119-123)
    nf += 1;
    prob->f(u, p, f, n);
    if (nudge)
      for (int i = 0; i < n; ++i) f[i] = std::nextafter(f[i], nudge > 0 ? INFINITY : -INFINITY);
  }
};

static inline bool all_finite(const double* x, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}
// np.max(np.abs(x)): NaN propagates
static inline double max_abs(const double* x, int n) {
  double m = 0.0;
  for (int i = 0; i < n; ++i) {
    double a = std::fabs(x[i]);
    if (std::isnan(a)) return a;
    if (i == 0 || a > m) m = a;
  }
  return m;
}
// check_convergence (core.py:94-98)
static inline bool converged(const double* f, int n, double abstol) {
  double m = max_abs(f, n);
  return std::isfinite(m) && m <= abstol;
}

// dense_jacobian through _DenseJac.materialize (jacobians.py:92-94,
// autodiff.py:342-355).  Returns false on NonFiniteValue.  nf grows by the
// number of SEED_WIDTH chunks the reference evaluates before it stops.
static bool dense_jacobian(Ctx& c, const double* u, double* J) {
  const int n = c.n;
  Dual ud[16] = {}, out[16] = {};
  for (int i = 0; i < n; ++i) {
    ud[i].v = u[i];
    ud[i].w = n;
    for (int j = 0; j < n; ++j) ud[i].d[j] = (i == j) ? 1.0 : 0.0;
  }
  c.njac += 1;
  c.prob->fd(ud, c.p, out, n);
  bool vals_ok = true;
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(out[i].v)) vals_ok = false;
  for (int lo = 0; lo < n; lo += 8) {
    int hi = std::min(lo + 8, n);
    c.nf += 1;
    if (!vals_ok) return false;
    for (int i = 0; i < n; ++i)
      for (int j = lo; j < hi; ++j)
        if (!std::isfinite(out[i].d[j])) return false;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) J[i * n + j] = out[i].d[j];
  return true;
}

// LuFactorization(A, strict=False) (linalg.py:87-105).  false = SingularMatrix.
static bool lu_factor(int n, double* A, int* piv) {
  double anorm = max_abs(A, n * n);
  if (anorm == 0.0 || !std::isfinite(anorm)) return false;
  getrf(n, A, piv);
  double mn = 0.0;
  bool nan = false;
  for (int i = 0; i < n; ++i) {
    double a = std::fabs(A[i * n + i]);
    if (std::isnan(a)) nan = true;
    if (i == 0 || a < mn) mn = a;
  }
  if (nan) return true;  // np.min propagates NaN; NaN <= 0 is False
  return !(mn <= 0.0);
}

struct Result {
  double u[16];
  double resid;
  int8_t code;
};

static void finish(Result& r, const double* u, const double* f, int n, int8_t code) {
  for (int i = 0; i < n; ++i) r.u[i] = u[i];
  r.resid = max_abs(f, n);  // resid_max_norm (core.py:101-103)
  r.code = code;
}

// ---- Newton-Raphson (solvers.py:179-287, descent newton, no globalization) ---
// With line_search=true: the "newton-backtracking" preset (solvers.py:613):
// merit_along + backtracking_search (globalize.py:40-74, c1=1e-4, rho=0.5,
// alpha0=1, 30 backtracks).
static void newton(Ctx& c, const double* u0, double abstol, int maxiters, bool line_search, Result& r) {
  const int n = c.n;
  double u[16], f[16], J[256], du[16], un[16], fn_[16];
  int piv[16];
  std::memcpy(u, u0, sizeof(double) * n);
  c.F(u, f);
  if (!all_finite(f, n)) return finish(r, u, f, n, NONFINITE);
  if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
  for (int k = 1; k <= maxiters; ++k) {
    if (!dense_jacobian(c, u, J)) return finish(r, u, f, n, NONFINITE);
    double Jc[256];
    std::memcpy(Jc, J, sizeof(double) * n * n);
    if (!lu_factor(n, Jc, piv)) return finish(r, u, f, n, LINSOLVE_FAILED);
    c.nlinsolve += 1;
    for (int i = 0; i < n; ++i) du[i] = -f[i];
    getrs(n, Jc, piv, du);
    double alpha = 1.0;
    if (line_search) {
      // merit_along (globalize.py:40-56): phi0 = 0.5*(f@f), dphi0 = f@(J@du)
      double phi0 = 0.5 * ddot(n, f, f);
      double Jdu[16];
      gemv_A_x(n, J, du, Jdu);
      double dphi0 = ddot(n, f, Jdu);
      // backtracking_search (globalize.py:59-74)
      if (!(dphi0 < 0.0)) return finish(r, u, f, n, LINESEARCH_FAILED);
      bool ok = false;
      for (int it = 0; it < 31; ++it) {
        double ut[16], ft[16];
        for (int i = 0; i < n; ++i) ut[i] = u[i] + alpha * du[i];
        c.F(ut, ft);
        double value = 0.5 * ddot(n, ft, ft);
        if (value <= phi0 + 1e-4 * alpha * dphi0) { ok = true; break; }
        alpha *= 0.5;
      }
      if (!ok) return finish(r, u, f, n, LINESEARCH_FAILED);
    }
    for (int i = 0; i < n; ++i) un[i] = u[i] + alpha * du[i];
    c.F(un, fn_);
    if (!(all_finite(un, n) && all_finite(fn_, n))) return finish(r, u, f, n, NONFINITE);
    std::memcpy(u, un, sizeof(double) * n);
    std::memcpy(f, fn_, sizeof(double) * n);
    c.nsteps += 1;
    if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
  }
  return finish(r, u, f, n, MAXITERS);
}

// ---- dogleg (descent.py:78-106) ------------------------------------------------
static void dogleg(int n, const double* J, const double* LU, const int* piv, const double* f,
                   double radius, double* out) {
  double newton[16];
  for (int i = 0; i < n; ++i) newton[i] = -f[i];
  getrs(n, LU, piv, newton);
  if (norm2(n, newton) <= radius) {
    std::memcpy(out, newton, sizeof(double) * n);
    return;
  }
  double g[16], Jg[16], cauchy[16], d[16];
  gemv_AT_x(n, J, f, g);  // J.T @ f
  gemv_A_x(n, J, g, Jg);  // J @ g
  double gg = ddot(n, g, g);
  double jgjg = ddot(n, Jg, Jg);
  // Python max(a, b) returns b only if b > a (NaN a stays NaN)
  double t_star = gg / ((1e-300 > jgjg) ? 1e-300 : jgjg);
  for (int i = 0; i < n; ++i) cauchy[i] = -t_star * g[i];
  double cnorm = norm2(n, cauchy);
  if (cnorm >= radius) {
    double s = -(radius / std::sqrt(gg));
    for (int i = 0; i < n; ++i) out[i] = s * g[i];
    return;
  }
  for (int i = 0; i < n; ++i) d[i] = newton[i] - cauchy[i];
  double a = ddot(n, d, d);
  double b = 2.0 * ddot(n, cauchy, d);
  double cc = cnorm * cnorm - radius * radius;
  double tau = (-b + std::sqrt(b * b - 4.0 * a * cc)) / (2.0 * a);
  for (int i = 0; i < n; ++i) out[i] = cauchy[i] + tau * d[i];
}

// ---- trust region (globalize.py:156-214, SIMPLE scheme) -------------------------
static void trust_region(Ctx& c, const double* u0, double abstol, int maxiters, Result& r) {
  const int n = c.n;
  const double EPS = 2.220446049250313e-16;
  double u[16], f[16], J[256], LU[256], du[16], ut[16], ft[16];
  int piv[16];
  std::memcpy(u, u0, sizeof(double) * n);
  c.F(u, f);
  if (!all_finite(f, n)) return finish(r, u, f, n, NONFINITE);
  if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
  // initial_trust_state (globalize.py:116-118)
  double mu = max_abs(u, n);
  double radius = (mu > 1.0) ? mu : 1.0;  // Python max(1.0, mu)
  const double radius_max = 1e3 * radius;
  bool cached = false;
  for (int k = 1; k <= maxiters; ++k) {
    if (!cached) {
      if (!dense_jacobian(c, u, J)) return finish(r, u, f, n, NONFINITE);
      std::memcpy(LU, J, sizeof(double) * n * n);
      if (!lu_factor(n, LU, piv)) return finish(r, u, f, n, LINSOLVE_FAILED);
      cached = true;
    }
    c.nlinsolve += 1;
    dogleg(n, J, LU, piv, f, radius, du);
    if (!all_finite(du, n)) return finish(r, u, f, n, LINSOLVE_FAILED);
    for (int i = 0; i < n; ++i) ut[i] = u[i] + du[i];
    c.F(ut, ft);
    double rho;
    if (all_finite(ft, n)) {
      // tr_ratio (globalize.py:121-134)
      double Jdu[16], model[16];
      gemv_A_x(n, J, du, Jdu);
      for (int i = 0; i < n; ++i) model[i] = f[i] + Jdu[i];
      double ff = ddot(n, f, f);
      double actual = ff - ddot(n, ft, ft);
      double predicted = ff - ddot(n, model, model);
      if (predicted < EPS * ff) rho = -INFINITY;
      else rho = actual / predicted;
    } else {
      rho = -INFINITY;
    }
    // tr_update (globalize.py:137-153)
    bool accept;
    if (rho >= 0.5) {
      double ex = 2.0 * radius;
      radius = (radius_max < ex) ? radius_max : ex;  // Python min(ex, radius_max)
      accept = true;
    } else if (rho >= 0.1) {
      accept = true;
    } else {
      double sh = 0.5 * radius;
      radius = (1e-308 > sh) ? 1e-308 : sh;  // Python max(sh, 1e-308)
      accept = false;
    }
    if (accept) {
      std::memcpy(u, ut, sizeof(double) * n);
      std::memcpy(f, ft, sizeof(double) * n);
      c.nsteps += 1;
      cached = false;
      if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
    }
    if (radius < 1e-300) break;
  }
  return finish(r, u, f, n, MAXITERS);
}

// ---- quasi-Newton (solvers.py:290-358, quasinewton.py) ------------------------
static void quasi_newton(Ctx& c, const double* u0, double abstol, int maxiters, bool diagonal, Result& r) {
  const int n = c.n;
  const double EPS = 2.220446049250313e-16;
  double u[16], f[16], du[16], un[16], fn_[16], s[16], t[16];
  double H[256], dg[16];
  std::memcpy(u, u0, sizeof(double) * n);
  c.F(u, f);
  if (!all_finite(f, n)) return finish(r, u, f, n, NONFINITE);
  if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
  auto init = [&]() {  // qn_init, IDENTITY_INIT (quasinewton.py:66-94)
    if (diagonal) for (int i = 0; i < n; ++i) dg[i] = 1.0;
    else for (int i = 0; i < n * n; ++i) H[i] = (i / n == i % n) ? 1.0 : 0.0;
  };
  init();
  int reinits = 0, since = 0;
  std::vector<double> hist;
  hist.reserve(64);
  hist.push_back(norm2(n, f));
  for (int k = 1; k <= maxiters; ++k) {
    // du = -qn_apply(state, f_u) (quasinewton.py:97-104)
    if (diagonal) {
      for (int i = 0; i < n; ++i) du[i] = -(f[i] / dg[i]);
    } else {
      double Hf[16];
      gemv_A_x(n, H, f, Hf);
      for (int i = 0; i < n; ++i) du[i] = -Hf[i];
    }
    c.nlinsolve += 1;
    for (int i = 0; i < n; ++i) un[i] = u[i] + 1.0 * du[i];
    c.F(un, fn_);
    if (!(all_finite(un, n) && all_finite(fn_, n))) return finish(r, u, f, n, NONFINITE);
    bool merit_decreased = norm2(n, fn_) < norm2(n, f);
    for (int i = 0; i < n; ++i) { s[i] = un[i] - u[i]; t[i] = fn_[i] - f[i]; }
    std::memcpy(u, un, sizeof(double) * n);
    std::memcpy(f, fn_, sizeof(double) * n);
    c.nsteps += 1;
    hist.push_back(norm2(n, f));
    if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
    // reinit_check (quasinewton.py:179-198)
    bool reinit;
    if (!diagonal) {  // NOT_DESCENT
      double mdu = max_abs(du, n);
      double mu = max_abs(u, n);
      double scale = (1.0 > mu) ? 1.0 : mu;
      bool tiny = mdu < EPS * scale;
      reinit = (!merit_decreased) || tiny;
    } else {  // STALLING, window 3
      size_t L = hist.size();
      if (L < 4) {
        reinit = false;
      } else {
        double prev_best = hist[0];
        for (size_t i = 1; i < L - 3; ++i) if (hist[i] < prev_best) prev_best = hist[i];
        double recent = hist[L - 3];
        for (size_t i = L - 2; i < L; ++i) if (hist[i] < recent) recent = hist[i];
        reinit = recent > prev_best * (1.0 - 1e-12);
      }
    }
    if (reinit) {
      if (reinits > 0 && since <= 1) return finish(r, u, f, n, STALLED);
      reinits += 1;
      init();
      since = 0;
      hist.clear();
      hist.push_back(norm2(n, f));
    } else {
      if (diagonal) {
        // klement_update (quasinewton.py:152-168)
        double thresh = 1e-9 * max_abs(s, n);
        for (int i = 0; i < n; ++i) {
          if (std::fabs(s[i]) > thresh) dg[i] = t[i] / s[i];
          double mag = std::fabs(dg[i]);
          if (mag < 1e-12) dg[i] = (dg[i] >= 0.0) ? 1e-12 : -1e-12;
        }
      } else {
        // broyden_update (quasinewton.py:107-121)
        double Ht[16], sH[16];
        gemv_A_x(n, H, t, Ht);
        gemv_AT_x(n, H, s, sH);  // s @ H == H.T @ s
        double denom = ddot(n, s, Ht);
        if (!(std::fabs(denom) < 1e-12 * norm2(n, s) * norm2(n, Ht))) {
          for (int i = 0; i < n; ++i) {
            double a = s[i] - Ht[i];
            for (int j = 0; j < n; ++j) H[i * n + j] = H[i * n + j] + a * sH[j] / denom;
          }
        }
      }
      since += 1;
    }
  }
  return finish(r, u, f, n, MAXITERS);
}

// ---- DFSane (builder-authored, La Cruz–Martínez–Raydan 2006) --
// Constants: sigma in [1e-10, 1e10], sigma0 = 1, memory M = 10, gamma = 1e-4,
// tau in [0.1, 0.5], merit ||F||_2^2, eta_k = ||F(x0)||^2 / k^2, at most 100
// line-search shrinks per iteration (then LineSearchFailed).  Mirrors
// oracle/dfsane_ref.py operation for operation.
static void dfsane(Ctx& c, const double* u0, double abstol, int maxiters, Result& r) {
  const int n = c.n;
  const int M = 10;
  double u[16], f[16], d[16], up[16], fp[16], um[16], fm[16];
  std::memcpy(u, u0, sizeof(double) * n);
  c.F(u, f);
  if (!all_finite(f, n)) return finish(r, u, f, n, NONFINITE);
  if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
  double fnorm = ddot(n, f, f);
  const double f0 = fnorm;
  double hist[M];
  for (int i = 0; i < M; ++i) hist[i] = fnorm;
  double sigma = 1.0;
  for (int k = 1; k <= maxiters; ++k) {
    double as = std::fabs(sigma);
    double cl = as < 1e-10 ? 1e-10 : (as > 1e10 ? 1e10 : as);
    sigma = (sigma >= 0.0) ? cl : -cl;
    for (int i = 0; i < n; ++i) d[i] = -sigma * f[i];
    double eta = f0 / (double(k) * double(k));
    double fbar = hist[0];
    for (int i = 1; i < M; ++i) if (hist[i] > fbar) fbar = hist[i];
    double ap = 1.0, am = 1.0;
    const double *ua = nullptr, *fa = nullptr;
    double fa_norm = 0.0;
    for (int ls = 0;; ++ls) {
      for (int i = 0; i < n; ++i) up[i] = u[i] + ap * d[i];
      c.F(up, fp);
      double np_ = ddot(n, fp, fp);
      if (np_ <= fbar + eta - 1e-4 * (ap * ap) * fnorm) { ua = up; fa = fp; fa_norm = np_; break; }
      for (int i = 0; i < n; ++i) um[i] = u[i] - am * d[i];
      c.F(um, fm);
      double nm = ddot(n, fm, fm);
      if (nm <= fbar + eta - 1e-4 * (am * am) * fnorm) { ua = um; fa = fm; fa_norm = nm; break; }
      if (ls == 100) return finish(r, u, f, n, LINESEARCH_FAILED);
      double atp = (ap * ap) * fnorm / (np_ + (2.0 * ap - 1.0) * fnorm);
      double atm = (am * am) * fnorm / (nm + (2.0 * am - 1.0) * fnorm);
      double lo = 0.1 * ap, hi = 0.5 * ap;
      ap = !(atp > lo) ? lo : (atp > hi ? hi : atp);
      lo = 0.1 * am; hi = 0.5 * am;
      am = !(atm > lo) ? lo : (atm > hi ? hi : atm);
    }
    if (!(all_finite(ua, n) && all_finite(fa, n))) return finish(r, u, f, n, NONFINITE);
    double s[16], y[16];
    for (int i = 0; i < n; ++i) { s[i] = ua[i] - u[i]; y[i] = fa[i] - f[i]; }
    std::memcpy(u, ua, sizeof(double) * n);
    std::memcpy(f, fa, sizeof(double) * n);
    fnorm = fa_norm;
    c.nsteps += 1;
    hist[k % M] = fnorm;
    if (converged(f, n, abstol)) return finish(r, u, f, n, SUCCESS);
    double ss = ddot(n, s, s);
    double sy = ddot(n, s, y);
    sigma = ss / sy;
    if (std::isnan(sigma)) sigma = 1.0;
  }
  return finish(r, u, f, n, MAXITERS);
}

static void solve_one(const ProblemDef* prob, int n, int alg, const double* u0, const double* p,
                      double abstol, int maxiters, int nudge, Result& r, int32_t* counters) {
  Ctx c;
  c.nudge = nudge;
  c.prob = prob;
  c.n = n;
  c.p = p;
  switch (alg) {
    case NR: newton(c, u0, abstol, maxiters, false, r); break;
    case NEWTON_LS: newton(c, u0, abstol, maxiters, true, r); break;
    case TR: trust_region(c, u0, abstol, maxiters, r); break;
    case BROYDEN: quasi_newton(c, u0, abstol, maxiters, false, r); break;
    case KLEMENT: quasi_newton(c, u0, abstol, maxiters, true, r); break;
    case DFSANE: dfsane(c, u0, abstol, maxiters, r); break;
  }
  counters[0] = c.nsteps;
  counters[1] = c.nf;
  counters[2] = c.njac;
  counters[3] = c.nlinsolve;
}

}  // namespace oracle

using namespace oracle;

extern "C" {

int oracle_num_problems() { return kNumProblems; }
const char* oracle_problem_id(int h) { return (h >= 0 && h < kNumProblems) ? kProblems[h].id : nullptr; }

// Resolve an nlkit problem id; n_override picks n for n-generic families.
int oracle_lookup(const char* id, int n_override, int* handle, int* n, int* m) {
  std::string s(id);
  for (int h = 0; h < kNumProblems; ++h) {
    if (s != kProblems[h].id) continue;
    int nn = kProblems[h].n ? kProblems[h].n : n_override;
    if (kProblems[h].n && n_override > 0 && n_override != kProblems[h].n) return -2;
    if (nn < 1 || nn > 16) return -3;
    *handle = h;
    *n = nn;
    *m = kProblems[h].m < 0 ? nn : kProblems[h].m;
    return 0;
  }
  return -1;
}

void oracle_residual(int h, int n, const double* x, const double* p, double* f) {
  kProblems[h].f(x, p, f, n);
}

// 1 = ok, 0 = NonFiniteValue; J row-major n x n
int oracle_jacobian(int h, int n, const double* x, const double* p, double* J) {
  Ctx c;
  c.prob = &kProblems[h];
  c.n = n;
  c.p = p;
  return dense_jacobian(c, x, J) ? 1 : 0;
}

// Batched solve, AoS: u0 [B][n], p [B][m] (or null), u_out [B][n].  nudge = +-1
// perturbs every float residual by one ulp (the roundoff-sensitivity probe).
int oracle_solve_batch(int h, int n, int alg, int64_t B, const double* u0, const double* p, int m,
                       double abstol, int maxiters, int nthreads, double* u_out, double* resid_out,
                       int8_t* retcode, int32_t* nsteps, int32_t* nf, int32_t* njac, int32_t* nlinsolve,
                       int nudge) {
  if (h < 0 || h >= kNumProblems || n < 1 || n > 16) return -1;
  if (alg < 0 || alg > 5) return -2;
  const ProblemDef* prob = &kProblems[h];
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(64);
      if (i >= B) break;
      int64_t e = std::min<int64_t>(i + 64, B);
      for (int64_t b = i; b < e; ++b) {
        Result r;
        int32_t cnt[4];
        solve_one(prob, n, alg, u0 + b * n, p ? p + b * m : nullptr, abstol, maxiters, nudge, r, cnt);
        for (int k = 0; k < n; ++k) u_out[b * n + k] = r.u[k];
        resid_out[b] = r.resid;
        retcode[b] = r.code;
        nsteps[b] = cnt[0];
        nf[b] = cnt[1];
        njac[b] = cnt[2];
        nlinsolve[b] = cnt[3];
      }
    }
  };
  if (nthreads <= 1) {
    worker();
  } else {
    std::vector<std::thread> ts;
    for (int t = 0; t < nthreads; ++t) ts.emplace_back(worker);
    for (auto& t : ts) t.join();
  }
  return 0;
}

// primitives, exported for tests/test_oracle_blas.py
double oracle_ddot(int n, const double* x, const double* y) { return ddot(n, x, y); }
void oracle_gemv_A_x(int n, const double* A, const double* x, double* y) { gemv_A_x(n, A, x, y); }
void oracle_gemv_AT_x(int n, const double* A, const double* x, double* y) { gemv_AT_x(n, A, x, y); }
void oracle_getrf(int n, double* A, int* piv) { getrf(n, A, piv); }
void oracle_getrs(int n, const double* LU, const int* piv, double* b) { getrs(n, LU, piv, b); }
void oracle_getrs_t(int n, const double* LU, const int* piv, double* b) { getrs_t(n, LU, piv, b); }

}  // extern "C"
