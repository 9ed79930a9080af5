// Warp-cooperative solvers for the larger systems (n >= NLK_COOP_MIN).
//
// A thread-per-system kernel cannot keep an n = 9..16 Jacobian and its LU in
// registers: the n = 9/10 trust-region kernels ran at 255 registers with
// 2 KB of spills, 12 % occupancy, and spent most of their instructions on
// predicated pivot swaps and local-memory traffic (profiles/).  Here a group
// of n lanes owns one system and lane r owns ROW r of every matrix:
//   * the Jacobian is evaluated column-wise (lane c sweeps a width-1 dual
//     seeded with e_c — bits identical to the reference's width-8 sweeps,
//     every Dual op being componentwise) and transposed through shared memory;
//   * the LU keeps one row per lane in registers; row interchanges are lane
//     exchanges (one shuffle per element), pivot search is a broadcast scan in
//     the reference's order, and every element sees exactly the operation
//     sequence of the OpenBLAS getrf/GETF2/TRSM/GEMM model (nlk_blas.cuh) —
//     only the place where it is computed changes;
//   * vectors (u, f, steps) are replicated across the group, so every
//     data-dependent decision is taken identically by all of its lanes.
// 32 / n systems share a warp (3 for n = 9/10, 2 for n = 16); all shuffles use
// the group's own lane mask, so groups in different phases may diverge.
#pragma once
#include "nlk_solvers.cuh"

namespace nlk {

#ifndef NLK_COOP_MIN
#define NLK_COOP_MIN 99  // off: measured 2-5x slower than thread-per-system (profiles/r01_variants_coop_vs_thread.log)
#endif

#define NLK_FD __device__ __forceinline__

template <int N> struct CoopShape {
  static constexpr int SPW = 32 / N;  // systems per warp
  static constexpr int LANES = SPW * N;
  static constexpr int LD = N + 1;    // padded smem row (2-way bank conflicts at most)
};

struct Grp {
  unsigned mask;  // lanes of this system
  int base;       // first lane of the group
  int row;        // row owned by this lane
  NLK_FD int lane(int r) const { return base + r; }
};

template <class T> NLK_FD T gshfl(const Grp& g, T v, int r) { return __shfl_sync(g.mask, v, g.base + r); }

// exchange rows i <-> p (group-relative) of a distributed value; other lanes keep theirs
template <class T> NLK_FD T gswap(const Grp& g, T v, int i, int p) {
  const int src = (g.row == i) ? p : ((g.row == p) ? i : g.row);
  return __shfl_sync(g.mask, v, g.base + src);
}

// replicate a distributed vector (lane r holds v_r) into out[0..N)
template <int N, class T> NLK_FD void replicate(const Grp& g, T v, T* out) {
#pragma unroll
  for (int k = 0; k < N; ++k) out[k] = gshfl(g, v, k);
}

// ---- BLAS rows -----------------------------------------------------------------
// y_row of `A @ x` for a C-ordered A whose row `row` is arow (dgemv_t model:
// 4x4 / 4x2 / 4x1 kernels by row index, then the column tail).
template <int N, class T>
NLK_FD T gemv_t_dot(int row, const T* arow, const T* x) {
  constexpr int N4 = N & ~3;
  T s = T(0);
  if constexpr (N4 > 0) {
    if (row < N4) {
      T v[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < N4; k += 4)
#pragma unroll
        for (int l = 0; l < 4; ++l) v[l] = t_fma(arow[k + l], x[k + l], v[l]);
      s = (v[0] + v[2]) + (v[1] + v[3]);
    } else if ((N & 2) && row < N4 + 2) {
      T v0 = T(0), v1 = T(0);
#pragma unroll
      for (int k = 0; k < N4; k += 2) {
        v0 = v0 + arow[k] * x[k];
        v1 = v1 + arow[k + 1] * x[k + 1];
      }
      s = v0 + v1;
    } else {
      T v[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < N4; k += 4)
#pragma unroll
        for (int l = 0; l < 4; ++l) v[l] = v[l] + arow[k + l] * x[k + l];
      s = (v[0] + v[2]) + (v[1] + v[3]);
    }
  }
  constexpr int R = N - N4;
  if constexpr (R == 0) {
    return s;
  } else if constexpr (R == 1) {
    return t_fma(arow[N4], x[N4], s);
  } else {
    T t = t_fma(arow[N4], x[N4], arow[N4 + 1] * x[N4 + 1]);
    if constexpr (R == 3) t = t_fma(arow[N4 + 2], x[N4 + 2], t);
    if constexpr (N4 > 0) return s + t;
    else return t;
  }
}

// output i of `A.T @ x` (dgemv_n model) from column i of A (acol[k] = A[k][i])
template <int N, class T>
NLK_FD T gemv_n_out(int i, const T* acol, const T* x) {
  constexpr int M1 = N & ~3;
  T y = T(0);
  if (i < M1) {
    int k = 0;
#pragma unroll
    for (; k + 4 <= N; k += 4) {
      T t = acol[k + 1] * x[k + 1];
      t = t_fma(acol[k], x[k], t);
      t = t_fma(acol[k + 2], x[k + 2], t);
      t = t_fma(acol[k + 3], x[k + 3], t);
      y = y + t;
    }
    if constexpr ((N & 3) >= 2) {
      constexpr int K2 = N & ~3;
      T t = acol[K2 + 1] * x[K2 + 1];
      t = t_fma(acol[K2], x[K2], t);
      y = y + t;
    }
    if constexpr (N & 1) y = y + acol[N - 1] * x[N - 1];
  } else {
    T t = T(0);
#pragma unroll
    for (int k = 0; k < N; ++k) t = t_fma(acol[k], x[k], t);
    y = y + t;
  }
  return y;
}

// ---- GETF2 on the panel rows OFF..N-1, columns OFF..OFF+NC-1 -----------------
template <int N, int OFF, int NC, class T>
NLK_FD void coop_getf2(const Grp& g, T* a, int* piv) {
  constexpr int M = N - OFF;
  const int ip = g.row - OFF;  // panel-relative row (< 0: above the panel)
  const bool inpanel = ip >= 0;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    T b = a[OFF + j];
    // 1. earlier interchanges of this panel
#pragma unroll
    for (int i = 0; i < j; ++i) {
      const int p = piv[OFF + i] - OFF;
      if (p != i) b = gswap(g, b, OFF + i, OFF + p);
    }
    // 2. rows 1..j-1: b_i -= sdot(L[i, 0:i], b[0:i]) (sequential; broadcast as final)
    T bb[NC > 0 ? NC : 1];
    bb[0] = gshfl(g, b, OFF + 0);
#pragma unroll
    for (int i = 1; i < j; ++i) {
      if (ip == i) {
        const int c4 = i & ~3;
        T t1 = T(0), t2 = T(0);
#pragma unroll
        for (int k = 0; k < c4; k += 4) {
          T m1 = a[OFF + k] * bb[k], m2 = a[OFF + k + 1] * bb[k + 1];
          T m3 = a[OFF + k + 2] * bb[k + 2], m4 = a[OFF + k + 3] * bb[k + 3];
          t1 = t1 + (m1 + m3);
          t2 = t2 + (m2 + m4);
        }
#pragma unroll
        for (int k = c4; k < i; ++k) t1 = t_fma(a[OFF + k], bb[k], t1);
        b = b - (t1 + t2);
      }
      bb[i] = gshfl(g, b, OFF + i);
    }
    if (j < M) {
      // 3. rows j..M-1: GEMV-N row update with the j finished columns
      if (j >= 1 && inpanel && ip >= j) {
        const int li = ip - j;
        const int M1 = (M - j) & ~3;
        if (li < M1) {
          int k = 0;
#pragma unroll
          for (; k + 4 <= j; k += 4) {
            T t = a[OFF + k + 1] * bb[k + 1];
            t = t_fma(a[OFF + k], bb[k], t);
            t = t_fma(a[OFF + k + 2], bb[k + 2], t);
            t = t_fma(a[OFF + k + 3], bb[k + 3], t);
            b = b - t;
          }
          if (k + 2 <= j) {
            T t = a[OFF + k + 1] * bb[k + 1];
            t = t_fma(a[OFF + k], bb[k], t);
            b = b - t;
            k += 2;
          }
          if (k < j) b = b - a[OFF + k] * bb[k];
        } else {
          T t = T(0);
#pragma unroll
          for (int k = 0; k < j; ++k) t = t_fma(a[OFF + k], bb[k], t);
          b = b - t;
        }
      }
      // 4. pivot: first index of max |b| over rows j..M-1, in the reference's order
      int p = j;
      T best = fabs(gshfl(g, b, OFF + j));
#pragma unroll
      for (int i = j + 1; i < M; ++i) {
        T v = fabs(gshfl(g, b, OFF + i));
        if (v > best) { best = v; p = i; }
      }
      piv[OFF + j] = OFF + p;
      // 5. interchange rows j <-> p over the finished panel columns and b; scale
      const T bp = __shfl_sync(g.mask, b, g.base + OFF + p);
      if (bp != T(0)) {
        if (p != j) {
#pragma unroll
          for (int k = 0; k < j; ++k) a[OFF + k] = gswap(g, a[OFF + k], OFF + j, OFF + p);
          b = gswap(g, b, OFF + j, OFF + p);
        }
        const T bj = gshfl(g, b, OFF + j);
        if (fabs(bj) >= Num<T>::dbl_min) {
          const T r = T(1) / bj;
          if (inpanel && ip > j) b = b * r;
        }
      }
    }
    if (inpanel) a[OFF + j] = b;
  }
}

// TRSM_LT (unit L) on rows IS..IS+BK-1, columns IS+BK..N-1: sub-blocks
// 16/8/4/2/1 by the bits of BK, a GEMM from the solved rows before each.
template <int N, int IS, int BK, int KK, class T>
NLK_FD void coop_trsm(const Grp& g, T* a) {
  if constexpr (KK < BK) {
    constexpr int REM = BK - KK;
    constexpr int BS = REM >= 16 ? 16 : (REM & 8) ? 8 : (REM & 4) ? 4 : (REM & 2) ? 2 : 1;
    constexpr int C0 = IS + BK, NJ = N - IS - BK;
    const bool inblk = g.row >= IS + KK && g.row < IS + KK + BS;
    if constexpr (KK > 0) {
      T acc[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j] = T(0);
#pragma unroll
      for (int k = 0; k < KK; ++k)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = t_fma(a[IS + k], gshfl(g, a[C0 + j], IS + k), acc[j]);
      if (inblk) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[C0 + j] = a[C0 + j] - acc[j];
      }
    }
#pragma unroll
    for (int i = 0; i < BS; ++i) {
      const bool below = g.row > IS + KK + i && g.row < IS + KK + BS;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const T bb = gshfl(g, a[C0 + j], IS + KK + i);
        if (below) a[C0 + j] = t_fma(-bb, a[IS + KK + i], a[C0 + j]);
      }
    }
    coop_trsm<N, IS, BK, KK + BS>(g, a);
  }
}

template <int N, int IS, int BLK, class T>
NLK_FD void coop_getrf_blocks(const Grp& g, T* a, int* piv) {
  if constexpr (IS < N) {
    constexpr int BK = (N - IS) < BLK ? (N - IS) : BLK;
    coop_getf2<N, IS, BK>(g, a, piv);
    if constexpr (IS + BK < N) {
      constexpr int C0 = IS + BK, NJ = N - IS - BK;
#pragma unroll
      for (int i = IS; i < IS + BK; ++i) {
        const int p = piv[i];
        if (p != i) {
#pragma unroll
          for (int j = 0; j < NJ; ++j) a[C0 + j] = gswap(g, a[C0 + j], i, p);
        }
      }
      coop_trsm<N, IS, BK, 0>(g, a);
      // GEMM update of the trailing rows: one FMA chain over k, then subtract
      T acc[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j] = T(0);
#pragma unroll
      for (int k = 0; k < BK; ++k)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = t_fma(a[IS + k], gshfl(g, a[C0 + j], IS + k), acc[j]);
      if (g.row >= C0) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[C0 + j] = a[C0 + j] - acc[j];
      }
    }
    coop_getrf_blocks<N, IS + BK, BLK>(g, a, piv);
  }
}

template <int N, int IS, int BLK, class T>
NLK_FD void coop_late_swaps(const Grp& g, T* a, const int* piv) {
  if constexpr (IS < N) {
    constexpr int BK = (N - IS) < BLK ? (N - IS) : BLK;
#pragma unroll
    for (int i = IS + BK; i < N; ++i) {
      const int p = piv[i];
      if (p != i) {
#pragma unroll
        for (int c = IS; c < IS + BK; ++c) a[c] = gswap(g, a[c], i, p);
      }
    }
    coop_late_swaps<N, IS + BK, BLK>(g, a, piv);
  }
}

// LuFactorization(A, strict=False) (linalg.py:87-105) on row-distributed A.
template <int N, class T>
NLK_FD bool coop_lu_factor(const Grp& g, T* a, int* piv) {
  T m = T(0);
  bool nan = false;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    T v = fabs(a[c]);
    nan |= (v != v);
    m = v > m ? v : m;
  }
  T anorm = T(0);
#pragma unroll
  for (int r = 0; r < N; ++r) {
    T v = gshfl(g, m, r);
    anorm = v > anorm ? v : anorm;
  }
  const bool anynan = __any_sync(g.mask, nan);
  if (anynan || anorm == T(0) || !isfinite(anorm)) return false;
  constexpr int BLK = ((N / 2 + 1) / 2) * 2;
  if constexpr (BLK <= 4) {
    coop_getf2<N, 0, N>(g, a, piv);
  } else {
    coop_getrf_blocks<N, 0, BLK>(g, a, piv);
    coop_late_swaps<N, 0, BLK>(g, a, piv);
  }
  T d = T(0);
#pragma unroll
  for (int c = 0; c < N; ++c)
    if (c == g.row) d = fabs(a[c]);
  const bool pnan = __any_sync(g.mask, d != d);
  const bool zero = __any_sync(g.mask, d <= T(0));
  return pnan || !zero;
}

// getrs (one RHS) on row-distributed LU; rhs and solution replicated.
template <int N, class T>
NLK_FD void coop_getrs(const Grp& g, const T* a, const int* piv, const T* rhs, T* x) {
  // lane r starts from rhs[tau(r)], tau = the sequential interchanges composed
  int src = g.row;
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const int p = piv[i];
    src = (src == i) ? p : ((src == p) ? i : src);
  }
  T mine = rhs[0];
#pragma unroll
  for (int k = 1; k < N; ++k)
    if (k == src) mine = rhs[k];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const T bi = gshfl(g, mine, i);
    if (g.row > i) mine = t_fma(-bi, a[i], mine);
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    if (g.row == i) mine = mine / a[i];
    const T bi = gshfl(g, mine, i);
    if (g.row < i) mine = t_fma(-bi, a[i], mine);
  }
  replicate<N>(g, mine, x);
}

// ---- cooperative state ----------------------------------------------------------
template <class P, int N, class T>
struct CoopBase {
  static constexpr int M = P::M;
  T u[N], f[N];
  T p[M > 0 ? M : 1];
  int k, nsteps, nf, njac, nlinsolve;
  Grp g;
  T* tbuf;  // this group's N x (N+1) transpose buffer in shared memory

  NLK_FD void F(const T* x, T* out) {
    nf += 1;
    Ctx<T, 0> cx{nullptr, 0};
    P::template f<T, T>(x, p, out, cx);
  }
  // column `row` of J by a width-1 dual sweep; returns -1 or the reference
  // chunk index that raised NonFiniteValue.  Fills arow (row) and, if
  // requested, acol (the lane's column).
  NLK_FD int jac(T* arow, T* acol) {
    njac += 1;
    Dual<1, T> xd[N], out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      xd[i].v = u[i];
      xd[i].d[0] = (i == g.row) ? T(1) : T(0);
    }
    Ctx<T, 0> cx{nullptr, 0};
    P::template f<Dual<1, T>, T>(xd, p, out, cx);
    bool vals_ok = true, col_ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      vals_ok &= isfinite(out[i].v);
      col_ok &= isfinite(out[i].d[0]);
      tbuf[i * CoopShape<N>::LD + g.row] = out[i].d[0];
      if (acol) acol[i] = out[i].d[0];
    }
    const unsigned badm = __ballot_sync(g.mask, !col_ok) >> g.base;
    __syncwarp(g.mask);
#pragma unroll
    for (int c = 0; c < N; ++c) arow[c] = tbuf[g.row * CoopShape<N>::LD + c];
    __syncwarp(g.mask);
    constexpr int chunks = (N + 7) / 8;
    int bad = -1;
    if (!vals_ok) bad = 0;
    else if (badm) bad = (__ffs(badm) - 1) / 8;
    nf += (bad < 0) ? chunks : bad + 1;
    return bad;
  }
  NLK_FD int start(T abstol) {
    k = nsteps = nf = njac = nlinsolve = 0;
    F(u, f);
    if (!all_finite<N>(f)) return NONFINITE;
    if (converged<N>(f, abstol)) return SUCCESS;
    return RUNNING;
  }
};

template <class P, int N, class T, bool LS>
struct CoopNewton : CoopBase<P, N, T> {
  using B = CoopBase<P, N, T>;
  NLK_FD int init(T abstol) { return B::start(abstol); }
  NLK_FD int step(T abstol, int maxiters) {
    B::k += 1;
    T a[N], jrow[LS ? N : 1];
    int piv[N];
    if (B::jac(a, nullptr) >= 0) return NONFINITE;
    if constexpr (LS) {
#pragma unroll
      for (int c = 0; c < N; ++c) jrow[c] = a[c];
    }
    if (!coop_lu_factor<N>(B::g, a, piv)) return LINSOLVE_FAILED;
    B::nlinsolve += 1;
    T rhs[N], du[N];
#pragma unroll
    for (int i = 0; i < N; ++i) rhs[i] = -B::f[i];
    coop_getrs<N>(B::g, a, piv, rhs, du);
    T alpha = T(1);
    T un[N], fn[N];
    if constexpr (LS) {
      T phi0 = T(0.5) * ddot<N>(B::f, B::f);
      T Jdu[N];
      replicate<N>(B::g, gemv_t_dot<N>(B::g.row, jrow, du), Jdu);
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
    if (!(all_finite<N>(un) && all_finite<N>(fn))) return NONFINITE;
#pragma unroll
    for (int i = 0; i < N; ++i) { B::u[i] = un[i]; B::f[i] = fn[i]; }
    B::nsteps += 1;
    if (converged<N>(B::f, abstol)) return SUCCESS;
    return B::k >= maxiters ? MAXITERS : RUNNING;
  }
};

template <class P, int N, class T>
struct CoopTrust : CoopBase<P, N, T> {
  using B = CoopBase<P, N, T>;
  T jrow[N], jcol[N], lu[N];
  int piv[N];
  T radius, radius_max;
  bool cached;

  NLK_FD int init(T abstol) {
    int st = B::start(abstol);
    T mu = max_abs<N>(B::u);
    radius = (mu > T(1)) ? mu : T(1);
    radius_max = T(1e3) * radius;
    cached = false;
    return st;
  }
  NLK_FD void dogleg(T* out) {
    T rhs[N], newton[N];
#pragma unroll
    for (int i = 0; i < N; ++i) rhs[i] = -B::f[i];
    coop_getrs<N>(B::g, lu, piv, rhs, newton);
    if (norm2<N>(newton) <= radius) {
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = newton[i];
      return;
    }
    T gv[N], Jg[N], cauchy[N];
    replicate<N>(B::g, gemv_n_out<N>(B::g.row, jcol, B::f), gv);
    replicate<N>(B::g, gemv_t_dot<N>(B::g.row, jrow, gv), Jg);
    T gg = ddot<N>(gv, gv);
    T jj = ddot<N>(Jg, Jg);
    T t_star = gg / ((Num<T>::tiny > jj) ? Num<T>::tiny : jj);
#pragma unroll
    for (int i = 0; i < N; ++i) cauchy[i] = -t_star * gv[i];
    T cnorm = norm2<N>(cauchy);
    if (cnorm >= radius) {
      T s = -(radius / sqrt(gg));
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = s * gv[i];
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
  NLK_FD int step(T abstol, int maxiters) {
    B::k += 1;
    if (!cached) {
      if (B::jac(jrow, jcol) >= 0) return NONFINITE;
#pragma unroll
      for (int c = 0; c < N; ++c) lu[c] = jrow[c];
      if (!coop_lu_factor<N>(B::g, lu, piv)) return LINSOLVE_FAILED;
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
    if (all_finite<N>(ft)) {
      T Jdu[N], model[N];
      replicate<N>(B::g, gemv_t_dot<N>(B::g.row, jrow, du), Jdu);
#pragma unroll
      for (int i = 0; i < N; ++i) model[i] = B::f[i] + Jdu[i];
      T ff = ddot<N>(B::f, B::f);
      T actual = ff - ddot<N>(ft, ft);
      T predicted = ff - ddot<N>(model, model);
      rho = (predicted < Num<T>::eps * ff) ? T(-INFINITY) : actual / predicted;
    } else {
      rho = T(-INFINITY);
    }
    bool accept;
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
    if (radius < Num<T>::radius_stop) return MAXITERS;
    return B::k >= maxiters ? MAXITERS : RUNNING;
  }
};

template <class P, int N, class T, int ALG> struct CoopOf { using type = void; };
template <class P, int N, class T> struct CoopOf<P, N, T, ALG_NR> { using type = CoopNewton<P, N, T, false>; };
template <class P, int N, class T> struct CoopOf<P, N, T, ALG_NEWTON_LS> { using type = CoopNewton<P, N, T, true>; };
template <class P, int N, class T> struct CoopOf<P, N, T, ALG_TR> { using type = CoopTrust<P, N, T>; };

template <int N, int ALG> struct UseCoop {
  static constexpr bool value = N >= NLK_COOP_MIN && N <= 16 &&
                                (ALG == ALG_NR || ALG == ALG_NEWTON_LS || ALG == ALG_TR);
};

#undef NLK_FD
}  // namespace nlk
