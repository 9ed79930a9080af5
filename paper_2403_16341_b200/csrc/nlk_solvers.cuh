// Per-system solver state machines: one outer iteration per step() call.
//
// Each solver restates one nlkit driver for a single system held in
// registers; the persistent kernel (nlk_kernel.cuh) interleaves steps of
// different systems in the lanes of a warp and refills finished lanes.
//   NewtonRaphson  solvers.py:179-287   (+ line search: solvers.py:263-276,
//                                        globalize.py:40-74)
//   TrustRegion    globalize.py:156-214, descent.py:78-106, globalize.py:116-153
//   Broyden        solvers.py:290-358, quasinewton.py:66-121,179-193
//   Klement        solvers.py:290-358, quasinewton.py:152-168,194-198
//   DFSane         builder-authored (oracle/dfsane_ref.py)
// Counters follow the reference exactly: nf counts every residual evaluation
// including ceil(n/8) dual sweeps per Jacobian, njac Jacobians, nlinsolve
// linear solves (TR: loop iterations; QN: inverse applications), nsteps
// accepted steps.
#pragma once
#include "nlk_problems.cuh"
#include "nlk_smem_lu.cuh"

namespace nlk {

enum RetCode : int { SUCCESS = 0, MAXITERS = 1, LINESEARCH_FAILED = 2, LINSOLVE_FAILED = 3,
                     STALLED = 4, NONFINITE = 5, RUNNING = -1, DEFERRED = -2 };
enum Alg : int { ALG_NR = 0, ALG_TR = 1, ALG_BROYDEN = 2, ALG_KLEMENT = 3, ALG_DFSANE = 4,
                 ALG_NEWTON_LS = 5, NUM_ALGS = 6 };

#define NLK_FD __device__ __forceinline__

template <int N, class T> NLK_FD bool all_finite(const T* x) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < N; ++i) ok &= isfinite(x[i]);
  return ok;
}
// bitwise equality of two vectors (distinguishes -0/+0, NaN payloads)
template <int N, class T> NLK_FD bool same_bits(const T* a, const T* b) {
  bool eq = true;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if constexpr (sizeof(T) == 8) eq &= (__double_as_longlong(a[i]) == __double_as_longlong(b[i]));
    else eq &= (__float_as_int(a[i]) == __float_as_int(b[i]));
  }
  return eq;
}
// np.max(np.abs(x)) with NaN propagation
template <int N, class T> NLK_FD T max_abs(const T* x) {
  T m = fabs(x[0]);
  bool nan = (m != m);
#pragma unroll
  for (int i = 1; i < N; ++i) {
    T a = fabs(x[i]);
    nan |= (a != a);
    m = a > m ? a : m;
  }
  return nan ? T(NAN) : m;
}
template <int N, class T> NLK_FD bool converged(const T* f, T abstol) {  // core.py:94-98
  T m = max_abs<N>(f);
  return isfinite(m) && m <= abstol;
}

// Width of one dual sweep on the device (bits are independent of it; the
// reference sweeps in SEED_WIDTH = 8 chunks).  Small systems sweep all
// columns at once in registers; compact (n >= 7) systems also use a single
// sweep — repeating the value path per chunk would repeat every
// transcendental of the residual.
#ifndef NLK_SWEEP_MAX
#define NLK_SWEEP_MAX 4
#endif
template <int N> struct SweepWidth {
  static constexpr int value = N <= 4 ? N : (N < NLK_SWEEP_MAX ? N : NLK_SWEEP_MAX);
};

// J sinks: register array or shared-memory slice (column-major, e = i + j*N)
template <class T> NLK_FD void jput(T* J, int e, T v) { J[e] = v; }
template <int N, class T, int S> NLK_FD void jput(const SMat<N, T, S>& J, int e, T v) { J.v(e) = v; }

// A Jacobian whose off-diagonal entries of each column share one value
// (problems with kJacRankOneDiag): diagonal d, column values s, and the
// zero signs of the off-diagonal entries (only an all-zero column can carry
// different bits per row).  2N values + N*N bits instead of N*N values.
// Accessors rebuild every entry bit-exactly; ZS = false skips the zero-sign
// lookup (valid when no column value is zero, i.e. !zany).
template <int N, class T>
struct RDJac {
  T d[N], s[N];
  uint32_t zm[(N * N + 31) / 32];
  bool zany;
  NLK_FD void reset() {
#pragma unroll
    for (int w = 0; w < (N * N + 31) / 32; ++w) zm[w] = 0u;
    zany = false;
  }
};
template <int N, class T, bool ZS>
struct RDRef {
  RDJac<N, T>* J;
};
template <int N, class T, bool ZS>
NLK_FD T mat_at(const RDRef<N, T, ZS>& A, int e) {
  const int i = e % N, j = e / N;
  if (i == j) return A.J->d[i];
  if constexpr (!ZS) {
    return A.J->s[j];
  } else {
    const T v = A.J->s[j];
    const bool neg = (A.J->zm[e >> 5] >> (e & 31)) & 1u;
    return (v != T(0)) ? v : (neg ? -T(0) : T(0));
  }
}
template <int N, class T, bool ZS>
NLK_FD void jput(const RDRef<N, T, ZS>& A, int e, T v) {
  const int i = e % N, j = e / N;
  if (i == j) {
    A.J->d[i] = v;
    return;
  }
  if (i == (j == 0 ? 1 : 0)) {
    A.J->s[j] = v;
    A.J->zany |= (v == T(0));
  }
  if (v == T(0) && signbit(v)) A.J->zm[e >> 5] |= 1u << (e & 31);
}

// dense_jacobian (autodiff.py:342-355) into column-major J.  Returns -1 on
// success, else the index of the reference chunk (8 columns) whose check
// raised NonFiniteValue — nlkit evaluates chunks up to and including it.
// `memo` holds the transcendental values recorded by the last F(u) (see Ctx
// in nlk_problems.cuh); every sweep replays them.
template <class P, int N, class T, int KM, int C0, class JS>
NLK_FD void jac_sweeps(const T* u, const T* p, T* memo, JS J, bool& vals_ok, int& bad_col) {
  if constexpr (C0 < N) {
    constexpr int SW = SweepWidth<N>::value;
    constexpr int W = (N - C0) < SW ? (N - C0) : SW;
    Dual<W, T> xd[N], out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      xd[i].v = u[i];
#pragma unroll
      for (int j = 0; j < W; ++j) xd[i].d[j] = (i == C0 + j) ? T(1) : T(0);
    }
    Ctx<T, (KM > 0 ? 2 : 0)> cx{memo, 0};
    P::template f<Dual<W, T>, T>(xd, p, out, cx);
    if constexpr (C0 == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) vals_ok &= isfinite(out[i].v);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
      bool colok = true;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        colok &= isfinite(out[i].d[j]);
        jput(J, i + (C0 + j) * N, out[i].d[j]);
      }
      if (!colok && bad_col > C0 + j) bad_col = C0 + j;
    }
    jac_sweeps<P, N, T, KM, C0 + W>(u, p, memo, J, vals_ok, bad_col);
  }
}

// KM > 0: memo holds the KM transcendental values of F(u) (replayed)
// Problems with an exact closed form of their dual-sweep Jacobian
// (P::jac_closed_form(u, memo, put)) skip the sweeps when it applies: it
// must produce the sweeps' bits, entry by entry (put(e, v), column-major e),
// or decline (return false, nothing put) -- then the sweeps run.
template <class P, class = void> struct HasJacClosedForm { static constexpr bool value = false; };
template <class P>
struct HasJacClosedForm<P, std::void_t<decltype(P::kJacClosedForm)>> {
  static constexpr bool value = P::kJacClosedForm;
};
#ifndef NLK_JAC_CLOSED_FORM
#define NLK_JAC_CLOSED_FORM 1
#endif

// FAST (the fast kernel of a closed-form problem, nlk_kernel.cuh): a
// declined closed form returns kJacDefer instead of running the dual sweeps,
// and the system is re-solved from its start by the complete kernel.
constexpr int kJacDefer = -2;
template <class P, int N, class T, int KM, bool FAST = false, class JS>
NLK_FD int jacobian(const T* u, const T* p, T* memo, JS J) {
  if constexpr (NLK_JAC_CLOSED_FORM && HasJacClosedForm<P>::value && std::is_same<T, double>::value) {
    // memo = nullptr: the driver keeps no memo (the closed form evaluates
    // what it needs itself)
    if (P::jac_closed_form(u, KM > 0 ? memo : nullptr, [&](int e, T v) { jput(J, e, v); }))
      return -1;
    if constexpr (FAST) return kJacDefer;
  }
  bool vals_ok = true;
  int bad_col = N;
  jac_sweeps<P, N, T, KM, 0>(u, p, memo, J, vals_ok, bad_col);
  if (!vals_ok) return 0;
  if (bad_col < N) return bad_col / 8;
  return -1;
}

// MEMO: record F's transcendentals for the next Jacobian (drivers that
// never form a Jacobian -- quasi-Newton, DFSane -- pass false).
// SCPAIRS: residuals evaluate their sincos in pairs per out-of-line call
// (Ctx::sincos_all; measured faster for Newton, slower for the trust region,
// whose extra live state then spills)
template <class P, int N, class T, bool MEMO = true, bool SCPAIRS = false, bool FAST = false>
struct Base {
  static constexpr int M = P::M;
  T u[N], f[N];
  T p[M > 0 ? M : 1];
  int k, nsteps, nf, njac, nlinsolve;
  static constexpr int kSmemElems = 0;
  static constexpr int kStride = kSmStride;  // block size = stride of the smem slices
  T* sm;  // this thread's shared-memory slice (stride kStride), see kSmemElems

  static constexpr int KM = MEMO ? MemoOf<P>::value : 0;
  T memo[KM > 0 ? KM : 1];  // transcendentals of the last F call

  NLK_FD void F(const T* x, T* out) {  // CountedResidual.at (core.py:119-123)
    nf += 1;
    Ctx<T, (KM > 0 ? 1 : 0), SCPAIRS> cx{memo, 0};
    P::template f<T, T>(x, p, out, cx);
  }
  // Precondition (memo): the last F call was at u.  Holds at every call site:
  // start() evaluates F(u0); Newton accepts u = un right after F(un); the
  // trust region re-evaluates J only after accepting u = ut right after F(ut).
  template <class JS>
  NLK_FD int jac(JS J) {
    int bad = jacobian<P, N, T, KM, FAST>(u, p, memo, J);
    if (FAST && bad == kJacDefer) return kJacDefer;
    njac += 1;
    constexpr int chunks = (N + 7) / 8;
    nf += (bad < 0) ? chunks : bad + 1;
    return bad;
  }
  // FAST Newton: the LU's divisions take their inline fast path only
  // (FlagDiv, nlk_div.cuh); dbad marks one outside it -> the step defers the
  // system.  Measured: trig NR 162.6 -> 157.6 ms; the trust-region kernels
  // were slower with it (trig TR 45.3 -> 48.6, msqrt-3x3 TR 154.1 -> 158.6)
  // and keep `b / d`.
  bool dbad;
  NLK_FD auto divp() {
    if constexpr (FAST) return FlagDiv{&dbad};
    else return ExactDiv{nullptr};
  }
  // shared prologue of every driver: f(u0), NONFINITE / already-converged
  NLK_FD int start(T abstol) {
    k = nsteps = nf = njac = nlinsolve = 0;
    dbad = false;
    F(u, f);
    if (!all_finite<N>(f)) return NONFINITE;
    if (converged<N>(f, abstol)) return SUCCESS;
    return RUNNING;
  }
};

// ---- Newton-Raphson (optionally with backtracking line search) --------------
template <class P, int N, class T, bool LS, bool FAST = false>
struct NewtonRaphson : Base<P, N, T, true, NLK_SINCOS_PAIRS_NR, FAST> {
  using B = Base<P, N, T, true, NLK_SINCOS_PAIRS_NR, FAST>;
  using SL = UseSmemLU<N, T, NLK_SMEM_NR_MIN>;
  static constexpr bool SM = SL::value;
  static constexpr int kSmemElems = SM ? N * N + N : 0;
  static constexpr int kStride = SM ? SL::stride : kSmStride;
  using Mat = SMat<N, T, kStride>;
  NLK_FD int init(T abstol) { return B::start(abstol); }
  NLK_FD int step(T abstol, int maxiters) {
    B::k += 1;
    int piv[N];
    T Jf[LS ? N * N : 1];  // J kept for the line search's J @ du
    T du[N];
    if constexpr (SM) {  // J streams column by column into the smem slice
      const Mat A{B::sm}, rhs{B::sm + N * N * kStride};
      const int jb = B::jac(A);
      if (FAST && jb == kJacDefer) return DEFERRED;
      if (jb >= 0) return NONFINITE;
      if constexpr (LS) {
#pragma unroll
        for (int e = 0; e < N * N; ++e) Jf[e] = A.v(e);
      }
      if (!sm_lu_factor<N, true>(A, piv, B::divp())) {
        if (FAST && B::dbad) return DEFERRED;
        return LINSOLVE_FAILED;
      }
      B::nlinsolve += 1;
#pragma unroll
      for (int i = 0; i < N; ++i) rhs.v(i) = -B::f[i];
      sm_getrs<N>(A, piv, rhs, B::divp());
      if (FAST && B::dbad) return DEFERRED;
#pragma unroll
      for (int i = 0; i < N; ++i) du[i] = rhs.v(i);
    } else {
      T J[N * N];
      const int jb = B::jac(J);
      if (FAST && jb == kJacDefer) return DEFERRED;
      if (jb >= 0) return NONFINITE;
      if constexpr (LS) {
#pragma unroll
        for (int i = 0; i < N * N; ++i) Jf[i] = J[i];
      }
      if (!lu_factor<N>(J, piv)) return LINSOLVE_FAILED;
      B::nlinsolve += 1;
#pragma unroll
      for (int i = 0; i < N; ++i) du[i] = -B::f[i];
      getrs<N>(J, piv, du);
    }
    T alpha = T(1);
    T un[N], fn[N];
    if constexpr (LS) {
      // merit_along + backtracking_search (globalize.py:40-74)
      T phi0 = T(0.5) * ddot<N>(B::f, B::f);
      T Jdu[N];
      gemv_A_x<N>(Jf, du, Jdu);
      T dphi0 = ddot<N>(B::f, Jdu);
      if (!(dphi0 < T(0))) return LINESEARCH_FAILED;
      bool ok = false;
#pragma unroll 1
      for (int it = 0; it < 31; ++it) {
#pragma unroll
        for (int i = 0; i < N; ++i) un[i] = B::u[i] + alpha * du[i];
        B::F(un, fn);
        T value = T(0.5) * ddot<N>(fn, fn);
        if (value <= phi0 + T(1e-4) * alpha * dphi0) { ok = true; break; }
        alpha *= T(0.5);
      }
      if (!ok) return LINESEARCH_FAILED;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) un[i] = B::u[i] + alpha * du[i];
    B::F(un, fn);
    // one max|fn| for both tests: it is finite iff every fn_i is (max_abs
    // propagates NaN), and converged(fn) is isfinite(m) && m <= abstol
    const T mf = max_abs<N>(fn);
    if (!(all_finite<N>(un) && isfinite(mf))) return NONFINITE;
#pragma unroll
    for (int i = 0; i < N; ++i) { B::u[i] = un[i]; B::f[i] = fn[i]; }
    B::nsteps += 1;
    if (mf <= abstol) return SUCCESS;
    return B::k >= maxiters ? MAXITERS : RUNNING;
  }
};

// ---- trust region with Powell dogleg -----------------------------------------
#ifndef NLK_TR_MEMO
#define NLK_TR_MEMO 1
#endif
#ifndef NLK_TR_JSMEM
#define NLK_TR_JSMEM 0
#endif
// keep the dogleg's radius-independent values across rejected steps
#ifndef NLK_TR_DLCACHE
#define NLK_TR_DLCACHE 1
#endif
// fast-forward a radius-exhaustion tail of bit-identical rejections (step())
#ifndef NLK_TR_FASTFWD
#define NLK_TR_FASTFWD 1
#endif
template <class P, class = void> struct TrNoFastFwd { static constexpr bool value = false; };
template <class P>
struct TrNoFastFwd<P, std::void_t<decltype(P::kTrNoFastFwd)>> { static constexpr bool value = P::kTrNoFastFwd; };
template <class P, int N, class T, bool FAST = false>
struct TrustRegion : Base<P, N, T, NLK_TR_MEMO, NLK_SINCOS_PAIRS_TR, FAST> {
  using B = Base<P, N, T, NLK_TR_MEMO, NLK_SINCOS_PAIRS_TR, FAST>;
  using SL = UseSmemLU<N, T, NLK_SMEM_TR_MIN>;
  static constexpr bool SM = SL::value;
  static constexpr int kStride = SM ? SL::stride : kSmStride;
  using Mat = SMat<N, T, kStride>;
  // JSM: J also in shared memory (after LU and rhs) instead of registers
  static constexpr bool JSM =
      SM && NLK_TR_JSMEM && sizeof(T) * (2 * N * N + N) * kStride <= 227 * 1024;
  static constexpr int kSmemElems = SM ? (JSM ? 2 * N * N + N : N * N + N) : 0;
  // RD: a rank-one-plus-diagonal Jacobian kept as RDJac (2N values instead of
  // N^2 registers; test23/trigonometric: the cached J was what spilled)
#ifndef NLK_TR_RDJAC
#define NLK_TR_RDJAC 1
#endif
  static constexpr bool RD = !JSM && NLK_TR_RDJAC && JacRankOneDiag<P>::value;
  T J[(JSM || RD) ? 1 : N * N], LU[SM ? 1 : N * N];
  RDJac<N, T> jrd[RD ? 1 : 0];
  NLK_FD auto jmat() {
    if constexpr (JSM) return Mat{B::sm + (N * N + N) * kStride};
    else if constexpr (RD) return RDRef<N, T, true>{&jrd[0]};
    else return static_cast<T*>(J);
  }
  // f(J accessor); for RD the zero-sign lookups are skipped unless some
  // column value is zero
  template <class F> NLK_FD void with_j(F&& f) {
    if constexpr (RD && FAST) {
      // only the closed form fills jrd here, and it declines whenever a
      // column value would be zero: the zero-sign accessor is never needed
      f(RDRef<N, T, false>{&jrd[0]});
    } else if constexpr (RD) {
      if (jrd[0].zany) f(RDRef<N, T, true>{&jrd[0]});
      else f(RDRef<N, T, false>{&jrd[0]});
    } else {
      f(jmat());
    }
  }
  int piv[N];
  T radius, radius_max;
  bool cached;

  NLK_FD int init(T abstol) {
    int st = B::start(abstol);
    T mu = max_abs<N>(B::u);
    radius = (mu > T(1)) ? mu : T(1);  // initial_trust_state: max(1.0, |u0|_inf)
    radius_max = T(1e3) * radius;
    cached = false;
    return st;
  }
  // dogleg_direction (descent.py:78-106)
  NLK_FD void dogleg_plain(T* out) {
    T newton[N];
    if constexpr (SM) {
      const Mat A{B::sm}, rhs{B::sm + N * N * kStride};
#pragma unroll
      for (int i = 0; i < N; ++i) rhs.v(i) = -B::f[i];
      sm_getrs<N>(A, piv, rhs);
#pragma unroll
      for (int i = 0; i < N; ++i) newton[i] = rhs.v(i);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) newton[i] = -B::f[i];
      getrs<N>(LU, piv, newton);
    }
    if (norm2<N>(newton) <= radius) {
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = newton[i];
      return;
    }
    T g[N], Jg[N], cauchy[N];
    with_j([&](auto Jm) {
      gemv_AT_x<N>(Jm, B::f, g);
      gemv_A_x<N>(Jm, g, Jg);
    });
    T gg = ddot<N>(g, g);
    T jj = ddot<N>(Jg, Jg);
    T t_star = gg / ((Num<T>::tiny > jj) ? Num<T>::tiny : jj);
#pragma unroll
    for (int i = 0; i < N; ++i) cauchy[i] = -t_star * g[i];
    T cnorm = norm2<N>(cauchy);
    if (cnorm >= radius) {
      T s = -(radius / sqrt(gg));
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = s * g[i];
      return;
    }
    T d[N];
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = newton[i] - cauchy[i];
    T a = ddot<N>(d, d);
    T b = T(2) * ddot<N>(cauchy, d);
    T c = cnorm * cnorm - radius * radius;
    T tau = (-b + sqrt(b * b - T(4) * a * c)) / (T(2) * a);
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = cauchy[i] + tau * d[i];
  }
  // The same dogleg with its radius-independent part kept across rejected
  // steps (shared-memory path, NLK_TR_DLCACHE).  A rejection leaves u, f, J
  // and the LU unchanged and only shrinks the radius, so the Newton step and
  // its norm, g = J^T f, J g, the Cauchy point and its norm are the same at
  // the next iteration; only the radius-dependent tail is re-evaluated, with
  // the same operations on the same values (bit-identical).  On MaxIters-bound
  // runs most iterations are rejections (test23/trigonometric, sigma = 0.1:
  // 94 %).  dl: 0 nothing cached; 1 Newton step in the rhs slot + its norm;
  // 2 + gg, t_star, |cauchy|; 3 g in the rhs slot instead -- set once the
  // scaled-gradient branch is taken: the radius only shrinks until the next
  // accepted step, so the Newton step and the segment are not needed again.
  // Measured (C2 jobs, B = 2^20): trigonometric 326 -> 283 ms; on the
  // register-LU path the extra loop-carried state cost more than it saved
  // (matrix-sqrt-2x2 with a register LU: 36 -> 47 ms), so it keeps
  // dogleg_plain.
  // Round 2: below n = NLK_TR_DLCACHE_MIN_N the cache's loop-carried state
  // costs more than the rejections it saves (matrix-sqrt-2x2 TR 29.4 -> 28.0
  // ms without it; matrix-sqrt-3x3 TR 158.7 -> 166.9 ms and spills without it).
#ifndef NLK_TR_DLCACHE_MIN_N
#define NLK_TR_DLCACHE_MIN_N 5
#endif
  static constexpr bool kDlCache = SM && NLK_TR_DLCACHE && N >= NLK_TR_DLCACHE_MIN_N;
  // the radius-exhaustion fast-forward (step()), except for problems whose
  // runs have no such tail (P::kTrNoFastFwd: matrix-sqrt-3x3 accepts 97 % of
  // its steps; without the code its kernel measured 156.4 -> 154.6 ms)
  static constexpr bool kFastFwd = kDlCache && NLK_TR_FASTFWD && !TrNoFastFwd<P>::value;
  T nnorm, gg, t_star, cnorm;
  int dl;
  NLK_FD void dogleg_cached(T* out) {
    const Mat A{B::sm}, rhs{B::sm + N * N * kStride};
    if (dl == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) rhs.v(i) = -B::f[i];
      sm_getrs<N>(A, piv, rhs);
      T newton[N];
#pragma unroll
      for (int i = 0; i < N; ++i) newton[i] = rhs.v(i);
      nnorm = norm2<N>(newton);
      dl = 1;
    }
    if (dl < 3 && nnorm <= radius) {
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = rhs.v(i);
      return;
    }
    T g[N];
    if (dl == 3) {
#pragma unroll
      for (int i = 0; i < N; ++i) g[i] = rhs.v(i);
    } else {
      with_j([&](auto Jm) { gemv_AT_x<N>(Jm, B::f, g); });
      if (dl == 1) {
        T Jg[N], cauchy[N];
        with_j([&](auto Jm) { gemv_A_x<N>(Jm, g, Jg); });
        gg = ddot<N>(g, g);
        T jj = ddot<N>(Jg, Jg);
        t_star = gg / ((Num<T>::tiny > jj) ? Num<T>::tiny : jj);
#pragma unroll
        for (int i = 0; i < N; ++i) cauchy[i] = -t_star * g[i];
        cnorm = norm2<N>(cauchy);
        dl = 2;
      }
    }
    if (cnorm >= radius) {
      T s = -(radius / sqrt(gg));
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = s * g[i];
      if (dl == 2) {
#pragma unroll
        for (int i = 0; i < N; ++i) rhs.v(i) = g[i];
        dl = 3;
      }
      return;
    }
    T cauchy[N], d[N];
#pragma unroll
    for (int i = 0; i < N; ++i) cauchy[i] = -t_star * g[i];
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = rhs.v(i) - cauchy[i];
    T a = ddot<N>(d, d);
    T b = T(2) * ddot<N>(cauchy, d);
    T c = cnorm * cnorm - radius * radius;
    T tau = (-b + sqrt(b * b - T(4) * a * c)) / (T(2) * a);
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = cauchy[i] + tau * d[i];
  }
  NLK_FD void dogleg(T* out) {
    if constexpr (kDlCache) dogleg_cached(out);
    else dogleg_plain(out);
  }
  // one iteration of run_trust_region's loop (globalize.py:174-212).
  // Measured and rejected (profiles/r02j_*, r02k_*, r02o_*): running the
  // rejections up to the next acceptance inside one call (so the J + LU
  // phases line up across a warp) -- trigonometric TR 64 -> 116 ms,
  // matrix-sqrt-3x3 TR 161 -> 273 ms: lanes that accepted then wait for the
  // longest rejection run of the warp; deferring a lane's J + LU (up to 2, 4
  // or 8 trips) until half the warp needs one -- 62.5 -> 66.4 ms (the votes
  // cost more than the alignment gains).
  NLK_FD int step(T abstol, int maxiters) {
    B::k += 1;
    if (!cached) {
      if constexpr (kDlCache) dl = 0;
      if constexpr (RD) jrd[0].reset();
      const int jb = B::jac(jmat());
      if (FAST && jb == kJacDefer) return DEFERRED;
      if (jb >= 0) return NONFINITE;
      if constexpr (SM) {
        const Mat A{B::sm};
        with_j([&](auto Jm) {
#pragma unroll
          for (int e = 0; e < N * N; ++e) A.v(e) = mat_at(Jm, e);
        });
        if (!sm_lu_factor<N, true>(A, piv)) return LINSOLVE_FAILED;
      } else {
        with_j([&](auto Jm) {
#pragma unroll
          for (int e = 0; e < N * N; ++e) LU[e] = mat_at(Jm, e);
        });
        if (!lu_factor<N>(LU, piv)) return LINSOLVE_FAILED;
      }
      cached = true;
    }
    B::nlinsolve += 1;
    T du[N];
    dogleg(du);
    if (!all_finite<N>(du)) return LINSOLVE_FAILED;
    T ut[N], ft[N];
#pragma unroll
    for (int i = 0; i < N; ++i) ut[i] = B::u[i] + du[i];
    B::F(ut, ft);
    T rho;
    if (all_finite<N>(ft)) {  // tr_ratio (globalize.py:121-134)
      T Jdu[N], model[N];
      with_j([&](auto Jm) { gemv_A_x<N>(Jm, du, Jdu); });
#pragma unroll
      for (int i = 0; i < N; ++i) model[i] = B::f[i] + Jdu[i];
      T ff = ddot<N>(B::f, B::f);
      T actual = ff - ddot<N>(ft, ft);
      T predicted = ff - ddot<N>(model, model);
      rho = (predicted < Num<T>::eps * ff) ? T(-INFINITY) : actual / predicted;
    } else {
      rho = T(-INFINITY);
    }
    bool accept;  // tr_update, SIMPLE scheme (globalize.py:137-153)
    if (rho >= T(0.5)) {
      T ex = T(2) * radius;
      radius = (radius_max < ex) ? radius_max : ex;
      accept = true;
    } else if (rho >= T(0.1)) {
      accept = true;
    } else {
      T sh = T(0.5) * radius;
      radius = (Num<T>::radius_floor > sh) ? Num<T>::radius_floor : sh;
      accept = false;
    }
    if (accept) {
#pragma unroll
      for (int i = 0; i < N; ++i) { B::u[i] = ut[i]; B::f[i] = ft[i]; }
      B::nsteps += 1;
      cached = false;
      if (converged<N>(B::f, abstol)) return SUCCESS;
    }
    if constexpr (kFastFwd) {
      // Radius-exhaustion fast-forward.  A rejection in the scaled-gradient
      // branch (dl == 3) whose trial point rounds back to u bit for bit
      // (and re-evaluates to the same f) fixes every remaining iteration:
      // the next radii only shrink, so each later step s'*g has
      // |s'| <= |s| with the same sign and, rounding being monotone,
      // u + s'*g == u again; F(u) == f, so actual reduction is exactly 0 and
      // rho is 0, -inf or NaN -- a rejection every time (globalize.py:
      // 196-212).  What remains of those iterations is the counters and the
      // radius halving, replayed here with the same operations.  Measured on
      // test23/trigonometric TR: the MaxIters tail is ~85 % such iterations.
      if (!accept && dl == 3 && same_bits<N>(ut, B::u) && same_bits<N>(ft, B::f)) {
        // The loop `while (!(radius < stop) && k < maxiters) { k++; radius =
        // max(floor, radius / 2); }` in closed form: from radius >= stop the
        // halvings are exact and stay above floor until the radius drops
        // below stop, so the trip count is min(m, maxiters - k) with m the
        // number of halvings that takes the radius below stop (found from
        // the exponents, checked with exact ldexp).  An infinite radius never
        // drops.  Only the trip count is observable (the radius is not
        // returned).
        const int left = maxiters - B::k;
        int m;
        if (radius < Num<T>::radius_stop) {
          m = 0;
        } else if (!isfinite(radius)) {
          m = left;
        } else {
          m = ilogb(radius) - ilogb(Num<T>::radius_stop) - 1;
          if (m < 0) m = 0;
          while (!(ldexp(radius, -m) < Num<T>::radius_stop)) ++m;
        }
        const int extra = (left <= 0) ? 0 : (m < left ? m : left);
        B::k += extra;
        B::nlinsolve += extra;
        B::nf += extra;
        return MAXITERS;
      }
    }
    if (radius < Num<T>::radius_stop) return MAXITERS;
    return B::k >= maxiters ? MAXITERS : RUNNING;
  }
};

// ---- quasi-Newton: dense inverse Broyden / diagonal Klement ------------------
template <class P, int N, class T, bool DIAG>
struct QuasiNewton : Base<P, N, T, false> {
  using B = Base<P, N, T, false>;
  T H[DIAG ? N : N * N];  // inverse Jacobian (column-major) or Jacobian diagonal
  // Broyden: H is kept implicit while it is the identity (IDENTITY_INIT and
  // every reinit) and only written out at the first update.  dgemv with the
  // identity (gemv_A_x / gemv_AT_x: accumulators start at +0, N >= 4) returns
  // x_i for x_i != 0 and +0 for x_i = +-0 (every other term is a +-0 product
  // of a finite x; x is finite wherever H is applied), so
  // idgemv(x)_i = (x_i == 0 ? +0 : x_i) is the same bits without the 2 N^2
  // loads of H.  (N < 4: the dgemv tails can return -0; H stays explicit.
  // An update with a non-finite s or t writes H out first: 0 * inf is NaN.)
#ifndef NLK_QN_LAZY_ID
#define NLK_QN_LAZY_ID 1
#endif
  static constexpr bool LAZY = !DIAG && NLK_QN_LAZY_ID && N >= 4;
  bool hid;
  NLK_FD static void idgemv(const T* x, T* y) {
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = (x[i] == T(0)) ? T(0) : x[i];
  }
  int reinits, since;
  // stalling window (Klement): min of hist[:-3] and the last three entries
  T prev_min, last[3];
  int hlen;

  NLK_FD void qn_init() {  // IDENTITY_INIT (quasinewton.py:66-94)
    if constexpr (DIAG) {
#pragma unroll
      for (int i = 0; i < N; ++i) H[i] = T(1);
    } else if constexpr (LAZY) {
      hid = true;
    } else {
      id_write();
    }
  }
  NLK_FD void id_write() {
#pragma unroll
    for (int i = 0; i < N * N; ++i) H[i] = (i % N == i / N) ? T(1) : T(0);
  }
  NLK_FD void hist_reset(T v) { hlen = 1; last[2] = v; prev_min = T(INFINITY); }
  NLK_FD void hist_push(T v) {
    if (hlen >= 3) { T old = last[0]; prev_min = (hlen == 3 || old < prev_min) ? old : prev_min; }
    last[0] = last[1]; last[1] = last[2]; last[2] = v;
    hlen += 1;
  }
  NLK_FD int init(T abstol) {
    int st = B::start(abstol);
    qn_init();
    reinits = 0;
    since = 0;
    if constexpr (DIAG) hist_reset(norm2<N>(B::f));
    return st;
  }
  NLK_FD int step(T abstol, int maxiters) {
    B::k += 1;
    T du[N];
    if constexpr (DIAG) {
#pragma unroll
      // ddiv: exact-root components make f_i (and below t_i) exactly zero,
      // which nvcc's division sends to its slow path (nlk_div.cuh); measured
      // C3 Klement n = 16 118 -> 77 ms, n = 8 52 -> 31 ms (profiles/r02m_*).
      // Not used on the LU / trust-region / DFSane paths, where zero
      // dividends are rare and the extra test on the serial chain cost 2-7 %.
      for (int i = 0; i < N; ++i) du[i] = -ddiv(B::f[i], H[i]);
    } else {
      T Hf[N];
      if (LAZY && hid) idgemv(B::f, Hf);
      else gemv_A_x<N>(H, B::f, Hf);
#pragma unroll
      for (int i = 0; i < N; ++i) du[i] = -Hf[i];
    }
    B::nlinsolve += 1;
    T un[N], fn[N];
#pragma unroll
    for (int i = 0; i < N; ++i) un[i] = B::u[i] + T(1) * du[i];
    B::F(un, fn);
    const T mf = max_abs<N>(fn);  // as in NewtonRaphson::step
    if (!(all_finite<N>(un) && isfinite(mf))) return NONFINITE;
    T nnew = norm2<N>(fn);
    bool merit_decreased = nnew < norm2<N>(B::f);
    T s[N], t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s[i] = un[i] - B::u[i];
      t[i] = fn[i] - B::f[i];
      B::u[i] = un[i];
      B::f[i] = fn[i];
    }
    B::nsteps += 1;
    if constexpr (DIAG) hist_push(nnew);
    if (mf <= abstol) return SUCCESS;
    bool reinit;
    if constexpr (!DIAG) {  // NOT_DESCENT (quasinewton.py:188-193)
      T mdu = max_abs<N>(du);
      T mu = max_abs<N>(B::u);
      T scale = (T(1) > mu) ? T(1) : mu;
      reinit = !merit_decreased || (mdu < Num<T>::eps * scale);
    } else {  // STALLING, window 3 (quasinewton.py:194-198)
      if (hlen < 4) {
        reinit = false;
      } else {
        T recent = last[0];
        recent = last[1] < recent ? last[1] : recent;
        recent = last[2] < recent ? last[2] : recent;
        reinit = recent > prev_min * T(1.0 - 1e-12);
      }
    }
    if (reinit) {
      if (reinits > 0 && since <= 1) return STALLED;
      reinits += 1;
      qn_init();
      since = 0;
      if constexpr (DIAG) hist_reset(norm2<N>(B::f));
    } else {
      if constexpr (DIAG) {  // klement_update (quasinewton.py:152-168)
        T thresh = T(1e-9) * max_abs<N>(s);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          if (fabs(s[i]) > thresh) H[i] = ddiv(t[i], s[i]);
          if (fabs(H[i]) < T(1e-12)) H[i] = (H[i] >= T(0)) ? T(1e-12) : T(-1e-12);
        }
      } else {  // broyden_update (quasinewton.py:107-121)
        T Ht[N], sH[N];
        // s = un - u and t = fn - f can overflow: 0 * inf is NaN in dgemv
        if (LAZY && hid && !(all_finite<N>(s) && all_finite<N>(t))) {
          id_write();
          hid = false;
        }
        if (LAZY && hid) {
          idgemv(t, Ht);
          idgemv(s, sH);
        } else {
          gemv_A_x<N>(H, t, Ht);
          gemv_AT_x<N>(H, s, sH);
        }
        T denom = ddot<N>(s, Ht);
        if (!(fabs(denom) < T(1e-12) * norm2<N>(s) * norm2<N>(Ht))) {
          if (LAZY && hid) {
            id_write();
            hid = false;
          }
#pragma unroll
          for (int i = 0; i < N; ++i) {
            T a = s[i] - Ht[i];
#pragma unroll
            for (int j = 0; j < N; ++j) H[i + j * N] = H[i + j * N] + ddiv(a * sH[j], denom);
          }
        }
      }
      since += 1;
    }
    return B::k >= maxiters ? MAXITERS : RUNNING;
  }
};

// ---- DFSane (builder-authored) ------------------------------
template <class P, int N, class T>
struct DFSane : Base<P, N, T, false> {
  using B = Base<P, N, T, false>;
  static constexpr int MEM = 10;
  T fnorm, f0, sigma;
  T hist[MEM];

  NLK_FD int init(T abstol) {
    int st = B::start(abstol);
    fnorm = ddot<N>(B::f, B::f);
    f0 = fnorm;
#pragma unroll
    for (int i = 0; i < MEM; ++i) hist[i] = fnorm;
    sigma = T(1);
    return st;
  }
  NLK_FD int step(T abstol, int maxiters) {
    B::k += 1;
    T as = fabs(sigma);
    T cl = as < T(1e-10) ? T(1e-10) : (as > T(1e10) ? T(1e10) : as);
    sigma = (sigma >= T(0)) ? cl : -cl;
    T d[N];
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = -sigma * B::f[i];
    T eta = f0 / (T(B::k) * T(B::k));
    T fbar = hist[0];
#pragma unroll
    for (int i = 1; i < MEM; ++i) fbar = hist[i] > fbar ? hist[i] : fbar;
    T ap = T(1), am = T(1);
    T ua[N], fa[N], na;
#pragma unroll 1
    for (int ls = 0;; ++ls) {
#pragma unroll
      for (int i = 0; i < N; ++i) ua[i] = B::u[i] + ap * d[i];
      B::F(ua, fa);
      T np_ = ddot<N>(fa, fa);
      if (np_ <= fbar + eta - T(1e-4) * (ap * ap) * fnorm) { na = np_; break; }
#pragma unroll
      for (int i = 0; i < N; ++i) ua[i] = B::u[i] - am * d[i];
      B::F(ua, fa);
      T nm = ddot<N>(fa, fa);
      if (nm <= fbar + eta - T(1e-4) * (am * am) * fnorm) { na = nm; break; }
      if (ls == 100) return LINESEARCH_FAILED;
      T tp = (ap * ap) * fnorm / (np_ + (T(2) * ap - T(1)) * fnorm);
      T tm = (am * am) * fnorm / (nm + (T(2) * am - T(1)) * fnorm);
      T lo = T(0.1) * ap, hi = T(0.5) * ap;
      ap = !(tp > lo) ? lo : (tp > hi ? hi : tp);
      lo = T(0.1) * am; hi = T(0.5) * am;
      am = !(tm > lo) ? lo : (tm > hi ? hi : tm);
    }
    const T mf = max_abs<N>(fa);  // as in NewtonRaphson::step
    if (!(all_finite<N>(ua) && isfinite(mf))) return NONFINITE;
    T s[N], y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s[i] = ua[i] - B::u[i];
      y[i] = fa[i] - B::f[i];
      B::u[i] = ua[i];
      B::f[i] = fa[i];
    }
    fnorm = na;
    B::nsteps += 1;
    const int slot = B::k % MEM;
#pragma unroll
    for (int i = 0; i < MEM; ++i)
      if (i == slot) hist[i] = fnorm;
    if (mf <= abstol) return SUCCESS;
    T ss = ddot<N>(s, s);
    T sy = ddot<N>(s, y);
    sigma = ss / sy;
    if (sigma != sigma) sigma = T(1);
    return B::k >= maxiters ? MAXITERS : RUNNING;
  }
};

// FAST: the fast variant of a closed-form problem's Newton / trust-region
// solver (no dual-sweep fallback; see jacobian() and nlk_kernel.cuh)
template <class P, int N, class T, int ALG, bool FAST = false> struct SolverOf;
template <class P, int N, class T, bool F> struct SolverOf<P, N, T, ALG_NR, F> { using type = NewtonRaphson<P, N, T, false, F>; };
template <class P, int N, class T, bool F> struct SolverOf<P, N, T, ALG_NEWTON_LS, F> { using type = NewtonRaphson<P, N, T, true, F>; };
template <class P, int N, class T, bool F> struct SolverOf<P, N, T, ALG_TR, F> { using type = TrustRegion<P, N, T, F>; };
template <class P, int N, class T, bool F> struct SolverOf<P, N, T, ALG_BROYDEN, F> { using type = QuasiNewton<P, N, T, false>; };
template <class P, int N, class T, bool F> struct SolverOf<P, N, T, ALG_KLEMENT, F> { using type = QuasiNewton<P, N, T, true>; };
template <class P, int N, class T, bool F> struct SolverOf<P, N, T, ALG_DFSANE, F> { using type = DFSane<P, N, T>; };

#undef NLK_FD
}  // namespace nlk
