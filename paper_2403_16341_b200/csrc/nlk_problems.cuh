// Device residual registry: the built-in problems of nlkit's problem library
// (/root/reference/pkg/src/nlkit/problems.py), compiled into the solve kernels.
//
// Each residual is a template over the scalar type S:
//   S = T (double / float)  -> the float path (numpy float64 evaluation,
//                              CountedResidual.at, core.py:119-123)
//   S = Dual<W, T>          -> the dual path (object arrays of Dual,
//                              autodiff.forward_sweep, autodiff.py:286-309)
// Expression trees follow the Python source literally (left-associative,
// no contraction) so the float path and the Jacobian are bit-identical to the
// reference wherever only + - * / sqrt are involved.  Where numpy evaluates the
// two paths differently (pairwise vs sequential sums, BLAS vs object matmul),
// the helpers below branch on the path.
#pragma once
#include <type_traits>

#include "nlk_blas.cuh"

namespace nlk {

template <class S> struct IsDual { static constexpr bool value = false; };
template <int W, class T> struct IsDual<Dual<W, T>> { static constexpr bool value = true; };

#define NLK_FD __device__ __forceinline__
#define K(x) (static_cast<T>(x))

template <class S> NLK_FD S zero_of(const S& like) {
  S r = like;
  if constexpr (IsDual<S>::value) {
    r.v = 0;
#pragma unroll
    for (int i = 0; i < (int)(sizeof(r.d) / sizeof(r.d[0])); ++i) r.d[i] = 0;
  } else {
    r = S(0);
  }
  return r;
}

// numpy add.reduce: float64 arrays pairwise (8 accumulators for n >= 8,
// sequential from 0.0 below); object arrays strictly left to right.
template <int N, class S> NLK_FD S np_sum(const S* x) {
  using T = typename ScalarOf<S>::type;
  if constexpr (IsDual<S>::value) {
    S r = x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) r = r + x[i];
    return r;
  } else if constexpr (N < 8) {
    S r = K(0);
#pragma unroll
    for (int i = 0; i < N; ++i) r = r + x[i];
    return r;
  } else {
    S r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = x[j];
    constexpr int NB = N - (N % 8);
#pragma unroll
    for (int i = 8; i < NB; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = r[j] + x[i + j];
    S res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int i = NB; i < N; ++i) res = res + x[i];
    return res;
  }
}
template <int N, class S> NLK_FD S np_prod(const S* x) {
  using T = typename ScalarOf<S>::type;
  if constexpr (IsDual<S>::value) {
    S r = x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) r = r * x[i];
    return r;
  } else {
    S r = K(1);
#pragma unroll
    for (int i = 0; i < N; ++i) r = r * x[i];
    return r;
  }
}

// ---- transcendental memo ------------------------------------------------------
// nlkit evaluates the Jacobian's value path with the same libm calls, on the
// same point, as the residual evaluation that preceded it (F(u) always comes
// before J(u) in every driver), and each dense_jacobian chunk repeats them
// again.  Residuals route their memo-able transcendentals through `cx`:
//   MODE 1 (float path)  evaluates and records each value in order;
//   MODE 2 (dual path)   replays the recorded values (bit-identical, same
//                        function of the same input) and forms the partials;
//   MODE 0               plain evaluation, nothing recorded.
// Only functions whose float and dual paths call the same libm routine are
// memoised (np.sin/np.cos/x**3 == math.*; np.exp and np.arctan are SVML on
// float64, not glibc, so exp and atan are not), and only where both paths
// feed them the same bits.  `kMemo` = slots a residual records per evaluation.
// arguments per glibc::sincos_n group in Ctx::sincos_all (0: one call each)
#ifndef NLK_SINCOS_GROUP
#define NLK_SINCOS_GROUP 0
#endif
// 1: Newton-Raphson's residual evaluations take sincos in pairs per
// out-of-line call (nlk_sincos2_v; Base<..., SCPAIRS>)
#ifndef NLK_SINCOS_PAIRS_NR
#define NLK_SINCOS_PAIRS_NR 1
#endif
// (the trust region too since round 2: trig TR 63.3 -> 61.1 ms; in round 1,
// before the compressed Jacobian and the dogleg cache, its extra live state
// spilled and pairs measured slower there)
#ifndef NLK_SINCOS_PAIRS_TR
#define NLK_SINCOS_PAIRS_TR 1
#endif
template <class T, int MODE, bool SCPAIRS = false>
struct Ctx {
  T* m;
  int i;
  template <class S> NLK_FD void sincos(const S& x, S& s, S& c) {
    if constexpr (MODE == 2 && IsDual<S>::value) {
      const T sv = m[i], cv = m[i + 1];
      s.v = sv;
      c.v = cv;
#pragma unroll
      for (int j = 0; j < (int)(sizeof(x.d) / sizeof(x.d[0])); ++j) {
        s.d[j] = cv * x.d[j];   // Dual.sin (autodiff.py:202-204)
        c.d[j] = -sv * x.d[j];  // Dual.cos (autodiff.py:206-208)
      }
    } else {
      t_sincos(x, s, c);
      if constexpr (MODE == 1) { m[i] = value_of(s); m[i + 1] = value_of(c); }
    }
    i += 2;
  }
  // sincos of G arguments: the fp64 float path evaluates them together
  // (glibc::sincos_n, G-way ILP; same bits as G separate calls)
  template <int G, class S> NLK_FD void sincos_all(const S* x, S* s, S* c) {
    if constexpr (std::is_same<S, double>::value && SCPAIRS && G % 2 == 0) {
#pragma unroll
      for (int g = 0; g < G; g += 2) {
        const SinCos2 r = nlk_sincos2_v(x[g], x[g + 1]);
        s[g] = r.s0; c[g] = r.c0; s[g + 1] = r.s1; c[g + 1] = r.c1;
      }
      if constexpr (MODE == 1) {
#pragma unroll
        for (int g = 0; g < G; ++g) { m[i + 2 * g] = s[g]; m[i + 2 * g + 1] = c[g]; }
      }
      i += 2 * G;
    } else if constexpr (std::is_same<S, double>::value && NLK_SINCOS_GROUP > 0) {
      constexpr int GG = NLK_SINCOS_GROUP < G ? NLK_SINCOS_GROUP : G;
#pragma unroll
      for (int g0 = 0; g0 < G; g0 += GG) {
        constexpr int R = G % GG;
        if (g0 + GG <= G) {
          if (glibc::sincos_n<GG>(x + g0, s + g0, c + g0)) {
#pragma unroll
            for (int g = g0; g < g0 + GG; ++g)
              if (glibc::sincos_slow(x[g])) t_sincos(x[g], s[g], c[g]);
          }
        } else if constexpr (R > 0) {
          if (glibc::sincos_n<R>(x + g0, s + g0, c + g0)) {
#pragma unroll
            for (int g = g0; g < G; ++g)
              if (glibc::sincos_slow(x[g])) t_sincos(x[g], s[g], c[g]);
          }
        }
      }
      if constexpr (MODE == 1) {
#pragma unroll
        for (int g = 0; g < G; ++g) { m[i + 2 * g] = s[g]; m[i + 2 * g + 1] = c[g]; }
      }
      i += 2 * G;
    } else {
#pragma unroll
      for (int g = 0; g < G; ++g) sincos(x[g], s[g], c[g]);
    }
  }
  template <class S> NLK_FD S cos(const S& x) {
    S s, c;
    sincos(x, s, c);
    return c;
  }
  template <class S> NLK_FD S pow3(const S& x) {
    S r;
    if constexpr (MODE == 2 && IsDual<S>::value) {  // Dual.__pow__(3) (autodiff.py:135-136)
      const T c = T(3) * t_pow2(x.v);
      r.v = m[i];
#pragma unroll
      for (int j = 0; j < (int)(sizeof(x.d) / sizeof(x.d[0])); ++j) r.d[j] = c * x.d[j];
    } else {
      r = t_pow3(x);
      if constexpr (MODE == 1) m[i] = value_of(r);
    }
    i += 1;
    return r;
  }
};
template <class P, class = void> struct JacRankOneDiag { static constexpr bool value = false; };
template <class P>
struct JacRankOneDiag<P, std::void_t<decltype(P::kJacRankOneDiag)>> {
  static constexpr bool value = P::kJacRankOneDiag;
};
// Problems whose iteration counts are tight run on the static (grid-stride)
// schedule of nlk_kernel.cuh instead of the refilling one
// P::kStaticAlgs: bit a set = algorithm a (nlk_solvers.cuh Alg: 0 NR, 1 TR,
// 2 Broyden, 3 Klement, 4 DFSane, 5 NR + line search) runs the static schedule
template <class P, class = void> struct StaticAlgs { static constexpr int value = 0; };
template <class P>
struct StaticAlgs<P, std::void_t<decltype(P::kStaticAlgs)>> {
  static constexpr int value = P::kStaticAlgs;
};
template <class P, int ALG> struct StaticSchedule {
  static constexpr bool value = (StaticAlgs<P>::value >> ALG) & 1;
};
// Newton, trust region and Newton + line search (kStaticNewtonTR): suite
// problems whose iteration counts stay tight over C2's perturbed starts, at
// sigma = 0.1 and at the stress sigma = 1.0 (max 32 steps)
constexpr int kStaticNewtonTR = (1 << 0) | (1 << 1) | (1 << 5);
template <class P, class = void> struct MemoOf { static constexpr int value = 0; };
template <class P> struct MemoOf<P, std::void_t<decltype(P::kMemo)>> { static constexpr int value = P::kMemo; };

// ---- the 23-member suite (problems.py:36-292) -------------------------------
struct Rosenbrock {  // 36-40
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = K(1.0) - x[0];
    out[1] = K(10.0) * (x[1] - x[0] * x[0]);
  }
};
struct PowellSingular {  // 43-49
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 4, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = x[0] + K(10.0) * x[1];
    out[1] = K(2.23606797749979) * (x[2] - x[3]);     // math.sqrt(5.0)
    out[2] = t_pow2(x[1] - K(2.0) * x[2]);
    out[3] = K(3.1622776601683795) * t_pow2(x[0] - x[3]);  // math.sqrt(10.0)
  }
};
struct PowellBadlyScaled {  // 52-56
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = K(1e4) * x[0] * x[1] - K(1.0);
    out[1] = t_exp(-x[0]) + t_exp(-x[1]) - K(1.0001);
  }
};
struct Wood {  // 59-67
  static constexpr int N = 4, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = K(-200.0) * x[0] * (x[1] - t_pow2(x[0])) - (K(1.0) - x[0]);
    out[1] = (K(200.0) * (x[1] - t_pow2(x[0])) + K(20.2) * (x[1] - K(1.0)) + K(19.8) * (x[3] - K(1.0)));
    out[2] = K(-180.0) * x[2] * (x[3] - t_pow2(x[2])) - (K(1.0) - x[2]);
    out[3] = (K(180.0) * (x[3] - t_pow2(x[2])) + K(20.2) * (x[3] - K(1.0)) + K(19.8) * (x[1] - K(1.0)));
  }
};
struct HelicalValley {  // 70-81
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 3, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    const T twopi = K(6.283185307179586);  // 2.0 * math.pi
    if (x[0] > K(0)) {
      S angle = t_atan(x[1] / x[0]) / twopi;
      out[0] = K(10.0) * (x[2] - K(10.0) * angle);
    } else if (x[0] < K(0)) {
      S angle = t_atan(x[1] / x[0]) / twopi + K(0.5);
      out[0] = K(10.0) * (x[2] - K(10.0) * angle);
    } else {
      T angle = (x[1] >= K(0)) ? K(0.25) : K(-0.25);
      out[0] = K(10.0) * (x[2] - K(10.0) * angle);
    }
    out[1] = K(10.0) * (t_sqrt(x[0] * x[0] + x[1] * x[1]) - K(1.0));
    out[2] = x[2];
  }
};
struct Watson {  // 84-109 (n = 2)
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
#pragma unroll 1
    for (int i = 1; i < 30; ++i) {
      T ti = T(i) / K(29.0);
      // sum1 over j = 1 .. n-1 from the float 0.0
      T temp = K(1.0);
      S sum1 = K(0.0) + (K(1.0) * temp) * x[1];
      temp = temp * ti;
      S sum2 = K(0.0) + K(1.0) * x[0];
      temp = K(1.0) * ti;
      sum2 = sum2 + temp * x[1];
      S temp1 = sum1 - sum2 * sum2 - K(1.0);
      S temp2 = K(2.0) * ti * sum2;
      T tk = K(1.0) / ti;
      S t0 = tk * (K(0.0) - temp2) * temp1;
      tk = tk * ti;
      S t1 = tk * (K(1.0) - temp2) * temp1;
      if (i == 1) {
        out[0] = K(0.0) + t0;
        out[1] = K(0.0) + t1;
      } else {
        out[0] = out[0] + t0;
        out[1] = out[1] + t1;
      }
    }
    S t = x[1] - x[0] * x[0] - K(1.0);
    out[0] = out[0] + x[0] * (K(1.0) - K(2.0) * t);
    out[1] = out[1] + t;
  }
};
struct Chebyquad {  // 112-129 (n = 2)
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      S t_cur = K(2.0) * x[j] - K(1.0);
      S scale = K(2.0) * t_cur;
      S t_prev = t_cur;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        out[i] = (j == 0) ? K(0.0) + t_cur : out[i] + t_cur;
        S t_next = (i == 0) ? scale * t_cur - K(1.0) : scale * t_cur - t_prev;
        t_prev = t_cur;
        t_cur = t_next;
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      out[k] = out[k] / T(N);
      if ((k + 1) % 2 == 0) out[k] = out[k] + K(1.0) / (T((k + 1) * (k + 1)) - K(1.0));
    }
  }
};
struct BrownAlmostLinear {  // 132-139
  static constexpr int N = 10, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    S total = np_sum<N>(x);
#pragma unroll
    for (int k = 0; k < N - 1; ++k) out[k] = x[k] + total - K(N + 1.0);
    out[N - 1] = np_prod<N>(x) - K(1.0);
  }
};
struct DiscreteBoundaryValue {  // 142-151
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 10, M = 0;
  static constexpr int kMemo = N;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    const T h = K(1.0) / T(N + 1);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      T tk = T(k + 1) * h;
      S a = K(2.0) * x[k];
      a = (k > 0) ? a - x[k > 0 ? k - 1 : 0] : a - K(0.0);
      a = (k < N - 1) ? a - x[k < N - 1 ? k + 1 : 0] : a - K(0.0);
      out[k] = a + K(0.5) * h * h * cx.pow3(x[k] + tk + K(1.0));
    }
  }
};
struct DiscreteIntegral {  // 154-168
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 10, M = 0;
  static constexpr int kMemo = N;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    const T h = K(1.0) / T(N + 1);
    T t[N];
#pragma unroll
    for (int j = 0; j < N; ++j) t[j] = T(j + 1) * h;
    S cubes[N];
#pragma unroll
    for (int j = 0; j < N; ++j) cubes[j] = cx.pow3(x[j] + t[j] + K(1.0));
#pragma unroll
    for (int k = 0; k < N; ++k) {
      S s1 = K(0.0) + t[0] * cubes[0];
#pragma unroll
      for (int j = 1; j <= k; ++j) s1 = s1 + t[j] * cubes[j];
      S inner = (K(1.0) - t[k]) * s1;
      if (k + 1 < N) {
        S s2 = K(0.0) + (K(1.0) - t[k + 1 < N ? k + 1 : 0]) * cubes[k + 1 < N ? k + 1 : 0];
#pragma unroll
        for (int j = k + 2; j < N; ++j) s2 = s2 + (K(1.0) - t[j]) * cubes[j];
        inner = inner + t[k] * s2;
      } else {
        inner = inner + t[k] * K(0.0);
      }
      out[k] = x[k] + K(0.5) * h * inner;
    }
  }
};
struct Trigonometric {  // 171-177
  static constexpr int N = 10, M = 0;
  static constexpr int kMemo = 2 * N;
  // Jacobian structure: column j off the diagonal is d(n - cos_sum)/dx_j
  // plus exact zeros, so every off-diagonal entry of a column has the same
  // bits, except that the entries of an all-zero column (x_j = +-0) carry
  // row-dependent zero signs (checked against the reference's dense_jacobian
  // on 3,000 points incl. zeros).  Drivers that keep J may store it as
  // diagonal + one value per column + zero signs (RDJac, nlk_solvers.cuh).
  static constexpr bool kJacRankOneDiag = true;
  // The dual sweep's Jacobian in closed form, from the memo of F(u)
  // (memo[2j] = sin u_j, memo[2j+1] = cos u_j).  Column j of the sweep:
  // d(cos_sum) = -sin u_j exactly (one nonzero term among exact zeros), so
  // T(N) - cos_sum gives sin u_j; off the diagonal the other terms add exact
  // zeros, on it (j+1)*(-(-sin u_j)) and -cos u_j are added in the sweep's
  // order: d_j = (s_j + (j+1)*s_j) - c_j.  With s_j == 0 the zeros' signs
  // matter: decline, and the sweeps run.  (The sweep's value path is bounded:
  // always finite.)
  static constexpr bool kJacClosedForm = true;
  template <class T, class PUT>
  NLK_FD static bool jac_closed_form(const T* u, const T* memo, PUT&& put) {
    T sc[2 * N];  // without a memo: glibc sin/cos of u, as F(u) computed them
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (memo) { sc[2 * j] = memo[2 * j]; sc[2 * j + 1] = memo[2 * j + 1]; }
      else t_sincos(u[j], sc[2 * j], sc[2 * j + 1]);
    }
    bool ok = true;
#pragma unroll
    for (int j = 0; j < N; ++j) ok &= (sc[2 * j] != T(0));
    if (!ok) return false;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const T sj = sc[2 * j], cj = sc[2 * j + 1];
      const T dj = (sj + T(j + 1) * sj) - cj;
#pragma unroll
      for (int i = 0; i < N; ++i) put(i + j * N, i == j ? dj : sj);
    }
    return true;
  }
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    S c[N], sn[N];  // np.cos(x) and np.sin(x[k]): one sincos per component
    cx.template sincos_all<N>(x, sn, c);
    S cos_sum = np_sum<N>(c);
#pragma unroll
    for (int k = 0; k < N; ++k)
      out[k] = T(N) - cos_sum + T(k + 1) * (K(1.0) - c[k]) - sn[k];
  }
};
struct VariablyDimensioned {  // 180-188
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 10, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    S w[N];
#pragma unroll
    for (int k = 0; k < N; ++k) w[k] = T(k + 1) * (x[k] - K(1.0));
    S s = np_sum<N>(w);
    S temp = s * (K(1.0) + K(2.0) * s * s);
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = x[k] - K(1.0) + T(k + 1) * temp;
  }
};
template <int NN>
struct BroydenTridiagonal {  // 191-198 (n-generic)
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = NN, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      S a = (K(3.0) - K(2.0) * x[k]) * x[k];
      a = (k > 0) ? a - x[k > 0 ? k - 1 : 0] : a - K(0.0);
      a = (k < N - 1) ? a - K(2.0) * x[k < N - 1 ? k + 1 : 0] : a - K(2.0) * K(0.0);
      out[k] = a + K(1.0);
    }
  }
};
struct BroydenBanded {  // 201-210
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 10, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int lo = k - 5 > 0 ? k - 5 : 0;
      const int hi = k + 2 < N ? k + 2 : N;
      S acc = x[0];
      bool first = true;
#pragma unroll
      for (int j = lo; j < hi; ++j) {
        if (j == k) continue;
        S term = x[j] * (K(1.0) + x[j]);
        acc = first ? K(0.0) + term : acc + term;
        first = false;
      }
      out[k] = x[k] * (K(2.0) + K(5.0) * x[k] * x[k]) + K(1.0) - acc;
    }
  }
};
// The dual sweep's Jacobian of R = X @ X - A (object matmul, X = D x D,
// row-major) in closed form.  Entry (row i*D+j, column a*D+b) of the sweep is
// sum_l (X_il*[l==a][j==b] + X_lj*[i==a][l==b]) with every product formed
// (v*1 or v*0) and summed over l in order.  With every X entry nonzero the
// nonzero terms are exact and the zeros cannot change them: j==b, i!=a ->
// X_ia; i==a, j!=b -> X_bj; i==a, j==b -> X_aa + X_bb (a == b: X_aa + X_aa);
// otherwise all 2D products are zeros carrying the signs of X_il and X_lj, and
// the sum is -0 iff row i and column j of X are all negative.  Declines (the
// sweeps run) when an entry is zero, or large enough for the sweep's value
// path to overflow where the float path did not.
template <int D, class T, class PUT>
NLK_FD bool matsq_jac_closed_form(const T* x, PUT&& put) {
  bool ok = true;
#pragma unroll
  for (int e = 0; e < D * D; ++e) ok &= (x[e] != T(0)) && (fabs(x[e]) < T(1e150));
  if (!ok) return false;
  bool rneg[D], cneg[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    rneg[i] = cneg[i] = true;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      rneg[i] = rneg[i] && signbit(x[i * D + l]);
      cneg[i] = cneg[i] && signbit(x[l * D + i]);
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b)
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          T v;
          if (i == a && j == b) v = x[a * D + a] + x[b * D + b];
          else if (j == b) v = x[i * D + a];
          else if (i == a) v = x[b * D + j];
          else v = (rneg[i] && cneg[j]) ? -T(0) : T(0);
          put((i * D + j) + (a * D + b) * D * D, v);
        }
  return true;
}
struct MatrixSqrt2x2 {  // 213-220
  static constexpr int N = 4, M = 0;
  // out[i*2+j] = X_i0 X_0j + X_i1 X_1j (- A_ij): the object matmul of
  // matsq_jac_closed_form, written out
  static constexpr bool kJacClosedForm = true;
  template <class T, class PUT>
  NLK_FD static bool jac_closed_form(const T* x, const T*, PUT&& put) {
    return matsq_jac_closed_form<2>(x, put);
  }
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = x[0] * x[0] + x[1] * x[2] - K(1e-4);
    out[1] = x[0] * x[1] + x[1] * x[3] - K(1.0);
    out[2] = x[2] * x[0] + x[3] * x[2];
    out[3] = x[2] * x[1] + x[3] * x[3] - K(1e-4);
  }
};
struct MatrixSqrt3x3 {  // 223-230: R = X @ X - A
  static constexpr int N = 9, M = 0;
  static constexpr bool kTrNoFastFwd = true;  // no radius-exhaustion tails (TrustRegion)
  // closed-form Jacobian: matsq_jac_closed_form (above)
  static constexpr bool kJacClosedForm = true;
  template <class T, class PUT>
  NLK_FD static bool jac_closed_form(const T* x, const T*, PUT&& put) {
    return matsq_jac_closed_form<3>(x, put);
  }
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        S r;
        if constexpr (IsDual<S>::value) {  // object matmul: first product, then adds
          r = x[i * 3 + 0] * x[0 * 3 + j];
          r = r + x[i * 3 + 1] * x[1 * 3 + j];
          r = r + x[i * 3 + 2] * x[2 * 3 + j];
        } else {  // dgemm: FMA chain from a plain product
          r = x[i * 3 + 0] * x[0 * 3 + j];
          r = t_fma(x[i * 3 + 1], x[1 * 3 + j], r);
          r = t_fma(x[i * 3 + 2], x[2 * 3 + j], r);
        }
        const int k = i * 3 + j;
        const T a = (k == 0 || k == 4 || k == 8) ? K(1e-4) : (k == 1 ? K(1.0) : K(0.0));
        out[k] = r - a;
      }
  }
};
struct DennisSchnabel {  // 233-237
  static constexpr int N = 2, M = 0;
  static constexpr int kMemo = 1;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = x[0] * x[0] + x[1] * x[1] - K(2.0);
    out[1] = t_exp(x[0] - K(1.0)) + cx.pow3(x[1]) - K(2.0);
  }
};
struct ProductExponential {  // 240-251
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    if (x[0] != K(0)) out[0] = x[1] * x[1] * (K(1.0) - t_exp(-x[0] * x[0])) / x[0];
    else out[0] = K(0.0) * x[1];
    if (x[1] != K(0)) out[1] = x[0] * (K(1.0) - t_exp(-x[1] * x[1])) / x[1];
    else out[1] = K(0.0) * x[0];
  }
};
struct CubicRadial {  // 254-260
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    S r2 = x[0] * x[0] + x[1] * x[1];
    out[0] = x[0] * r2;
    out[1] = x[1] * r2;
  }
};
struct DoubleRootScalar {  // 263-266
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 1, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = x[0] * t_pow2(x[0] - K(5.0));
  }
};
struct FreudensteinRoth {  // 269-273
  static constexpr int N = 2, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = K(-13.0) + x[0] + ((K(5.0) - x[1]) * x[1] - K(2.0)) * x[1];
    out[1] = K(-29.0) + x[0] + ((K(1.0) + x[1]) * x[1] - K(14.0)) * x[1];
  }
};
struct Boggs {  // 276-280
  static constexpr int N = 2, M = 0;
  static constexpr int kMemo = 2;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = x[0] * x[0] - x[1] + K(1.0);
    out[1] = x[0] - cx.cos(K(1.5707963267948966) * x[1]);  // (0.5 * math.pi) * x1
  }
};
struct Chandrasekhar {  // 286-292
  static constexpr int kStaticAlgs = kStaticNewtonTR;
  static constexpr int N = 10, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    T mu[N];
#pragma unroll
    for (int i = 0; i < N; ++i) mu[i] = (T(i + 1) - K(0.5)) / T(N);
    const T c = K(0.9) / (K(2.0) * T(N));
    S y[N];
    if constexpr (IsDual<S>::value) {  // object matmul: first product, then adds
#pragma unroll
      for (int i = 0; i < N; ++i) {
        y[i] = x[0] * (mu[i] / (mu[i] + mu[0]));
#pragma unroll
        for (int k = 1; k < N; ++k) y[i] = y[i] + x[k] * (mu[i] / (mu[i] + mu[k]));
      }
    } else {  // BLAS dgemv_t on the C-ordered A (column-major copy here)
      T A[N * N];
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int k = 0; k < N; ++k) A[r + k * N] = mu[r] / (mu[r] + mu[k]);
      gemv_A_x<N>(A, x, y);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = x[i] - K(1.0) / (K(1.0) - c * y[i]);
  }
};

// ---- parametrised families (problems.py:358-387) ----------------------------
template <int NN>
struct GeneralizedRosenbrock {  // 363-368
  static constexpr int N = NN, M = 0;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T*, S* out, C& cx) {
    out[0] = K(1.0) - x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) out[i] = K(10.0) * (x[i] - x[i - 1] * x[i - 1]);
  }
};
template <int NN>
struct Quadratic {  // 382-383: u * u - theta
  static constexpr int N = NN, M = NN;
  // C1/C5 iteration counts are tight (4-8 steps): grid-stride schedule, every solver
  static constexpr int kStaticAlgs = 0x3f;
  template <class S, class T, class C> NLK_FD static void f(const S* x, const T* p, S* out, C& cx) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = x[i] * x[i] - p[i];
  }
  // residual with float u and dual θ (autodiff.param_jacobian, autodiff.py:400-427):
  // `u * u - td` = float64 product, then Dual.__rsub__
  template <class S, class T> NLK_FD static void f_param(const T* x, const S* p, S* out) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = x[i] * x[i] - p[i];
  }
};

#undef K
#undef NLK_FD
}  // namespace nlk
