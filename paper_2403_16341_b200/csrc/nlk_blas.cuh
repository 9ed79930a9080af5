// Per-system dense linear algebra with the reference host's rounding order.
//
// nlkit's retcodes and iteration counts are decided by the last bits of its
// BLAS/LAPACK results on several problems, so each routine
// below reproduces the operation order of the kernel the reference reaches:
//   ddot        numpy dot / np.linalg.norm      (OpenBLAS ddot, SkylakeX)
//   gemv_t      `A @ x`   (C-ordered A)         (OpenBLAS dgemv_t 4x4/4x2/4x1)
//   gemv_n      `A.T @ x`, `s @ H`              (OpenBLAS dgemv_n)
//   getrf       scipy.linalg.lu_factor          (OpenBLAS getrf_single:
//               recursive blocking, GETF2 panels, TRSM_LT, GEMM updates)
//   getrs       scipy.linalg.lu_solve           (LAPACK getrs, one RHS)
// Reference call sites: linalg.py:98,107-108; descent.py:93-96,91,98;
// globalize.py:128-132; quasinewton.py:101,115-118; solvers.py:331-337.
// All sizes are compile-time: loops unroll, arrays live in registers, and the
// only data-dependent indices (pivots) are applied with predicated swaps.
#pragma once
#include "nlk_div.cuh"
#include "nlk_dual.cuh"

namespace nlk {

#define NLK_FD __device__ __forceinline__

// Every loop is fully unrolled (all sizes are template parameters), so
// vectors and matrices stay in registers; data-dependent indices (pivots)
// are applied with predicated swaps.  A rolled variant with local-memory
// arrays was measured 2-5x slower (profiles/r01_variants_codegen.log).

template <class T> NLK_FD T t_fma(T a, T b, T c) { return fma(a, b, c); }
template <> NLK_FD float t_fma<float>(float a, float b, float c) { return fmaf(a, b, c); }

// ---- ddot (n <= 15: FMA chain; 16-blocks: 4 lanes of rounded products) ------
template <int N, class T>
NLK_FD T ddot(const T* x, const T* y) {
  constexpr int N16 = N & ~15;
  T s = T(0);
  if constexpr (N16 > 0) {
    T v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = T(0);
#pragma unroll
    for (int b = 0; b < N16; b += 16) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        T p0 = x[b + j] * y[b + j];
        T p1 = x[b + j + 4] * y[b + j + 4];
        T p2 = x[b + j + 8] * y[b + j + 8];
        T p3 = x[b + j + 12] * y[b + j + 12];
        if (b == 0) v[j] = ((p0 + p1) + p2) + p3;
        else v[j] = (((v[j] + p0) + p1) + p2) + p3;
      }
    }
    s = (v[0] + v[2]) + (v[1] + v[3]);
  }
#pragma unroll
  for (int i = N16; i < N; ++i) s = t_fma(x[i], y[i], s);
  return s;
}
template <int N, class T> NLK_FD T norm2(const T* x) { return sqrt(ddot<N, T>(x, x)); }
// the same model with a length known only after unrolling (trsv dots)
template <class T>
NLK_FD T ddot_n(const int n, const T* x, const T* y) {
  const int n16 = n & ~15;
  T s = T(0);
  if (n16 > 0) {
    T v[4];
#pragma unroll
    for (int b = 0; b < n16; b += 16) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        T p0 = x[b + j] * y[b + j];
        T p1 = x[b + j + 4] * y[b + j + 4];
        T p2 = x[b + j + 8] * y[b + j + 8];
        T p3 = x[b + j + 12] * y[b + j + 12];
        if (b == 0) v[j] = ((p0 + p1) + p2) + p3;
        else v[j] = (((v[j] + p0) + p1) + p2) + p3;
      }
    }
    s = (v[0] + v[2]) + (v[1] + v[3]);
  }
#pragma unroll
  for (int i = n16; i < n; ++i) s = t_fma(x[i], y[i], s);
  return s;
}

// ---- GEMV-N column scheme (getf2 step 3 and `A.T @ x`) ---------------------
// a(i, k) = A[OFF_R + i + (OFF_C + k) * LDA] (column-major storage).
template <bool SUB, class T, class F>
NLK_FD void gemv_n_scheme(const int M, const int NCOL, F a, const T* x, T* y) {
  const int M1 = M & ~3;
#pragma unroll
  for (int i = 0; i < M1; ++i) {
    int k = 0;
#pragma unroll
    for (; k + 4 <= NCOL; k += 4) {
      T t = a(i, k + 1) * x[k + 1];
      t = t_fma(a(i, k), x[k], t);
      t = t_fma(a(i, k + 2), x[k + 2], t);
      t = t_fma(a(i, k + 3), x[k + 3], t);
      y[i] = SUB ? y[i] - t : y[i] + t;
    }
    if (k + 2 <= NCOL) {
      T t = a(i, k + 1) * x[k + 1];
      t = t_fma(a(i, k), x[k], t);
      y[i] = SUB ? y[i] - t : y[i] + t;
      k += 2;
    }
    if (k < NCOL) {
      T t = a(i, k) * x[k];
      y[i] = SUB ? y[i] - t : y[i] + t;
    }
  }
#pragma unroll
  for (int i = M1; i < M; ++i) {
    if (NCOL == 0) continue;
    T t = T(0);
#pragma unroll
    for (int k = 0; k < NCOL; ++k) t = t_fma(a(i, k), x[k], t);
    y[i] = SUB ? y[i] - t : y[i] + t;
  }
}

// y = A.T @ x, A column-major N x N (A[i + j*N] = A_ij)
// A is a register array (T*) or a shared-memory slice (SMat): mat_at(A, e)
template <class T> NLK_FD T mat_at(const T* A, int e) { return A[e]; }

template <int N, class AM, class T>
NLK_FD void gemv_AT_x(AM A, const T* x, T* y) {
#pragma unroll
  for (int i = 0; i < N; ++i) y[i] = T(0);
  gemv_n_scheme<false>(N, N, [&](int i, int k) { return mat_at(A, k + i * N); }, x, y);
}

// y = A @ x (dgemv_t: 4x4 / 4x2 / 4x1 kernels + column tail), A col-major
template <int N, class AM, class T>
NLK_FD T gemv_t_row(int row, AM A, const T* x) {
  constexpr int N4 = N & ~3;
  T s = T(0);
  if constexpr (N4 > 0) {
    if (row < N4) {
      T v[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < N4; k += 4)
#pragma unroll
        for (int l = 0; l < 4; ++l) v[l] = t_fma(mat_at(A, row + (k + l) * N), x[k + l], v[l]);
      s = (v[0] + v[2]) + (v[1] + v[3]);
    } else if ((N & 2) && row < N4 + 2) {
      T v0 = T(0), v1 = T(0);
#pragma unroll
      for (int k = 0; k < N4; k += 2) {
        v0 = v0 + mat_at(A, row + k * N) * x[k];
        v1 = v1 + mat_at(A, row + (k + 1) * N) * x[k + 1];
      }
      s = v0 + v1;
    } else {
 T v[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < N4; k += 4)
#pragma unroll
        for (int l = 0; l < 4; ++l) v[l] = v[l] + mat_at(A, row + (k + l) * N) * x[k + l];
      s = (v[0] + v[2]) + (v[1] + v[3]);
    }
  }
  constexpr int R = N - N4;
  if constexpr (R == 0) {
    return s;
  } else if constexpr (R == 1) {
    return t_fma(mat_at(A, row + N4 * N), x[N4], s);
  } else {
    T t = t_fma(mat_at(A, row + N4 * N), x[N4], mat_at(A, row + (N4 + 1) * N) * x[N4 + 1]);
    if constexpr (R == 3) t = t_fma(mat_at(A, row + (N4 + 2) * N), x[N4 + 2], t);
    if constexpr (N4 > 0) return s + t;
    else return t;
  }
}
template <int N, class AM, class T>
NLK_FD void gemv_A_x(AM A, const T* x, T* y) {
#pragma unroll
  for (int i = 0; i < N; ++i) y[i] = gemv_t_row<N>(i, A, x);
}

// ---- predicated swaps (data-dependent index, register-resident arrays) -----
// swap v[i*S] <-> v[p*S] for p in (i, LIMIT)
template <int LIMIT, int S, class T>
NLK_FD void swap_dyn(T* v, int i, int p) {
#pragma unroll
  for (int r = 0; r < LIMIT; ++r) {
    if (r > i && r == p) {
      T t = v[i * S];
      v[i * S] = v[r * S];
      v[r * S] = t;
    }
  }
}

// ---- GETF2 on an M x NC panel (column-major, leading dimension LDA) --------
template <int M, int NC, int LDA, class T>
NLK_FD void getf2_panel(T* A, int* piv) {
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    T b[M];
#pragma unroll
    for (int i = 0; i < M; ++i) b[i] = A[i + j * LDA];
    // 1. earlier interchanges
#pragma unroll
    for (int i = 0; i < j && i < M; ++i) swap_dyn<M, 1>(b, i, piv[i]);
    // 2. rows 1..j-1: b[i] -= sdot(L[i,0:i], b[0:i])
#pragma unroll
    for (int i = 1; i < j && i < M; ++i) {
      const int c4 = i & ~3;
      T t1 = T(0), t2 = T(0);
#pragma unroll
      for (int k = 0; k < c4; k += 4) {
        T m1 = A[i + k * LDA] * b[k], m2 = A[i + (k + 1) * LDA] * b[k + 1];
        T m3 = A[i + (k + 2) * LDA] * b[k + 2], m4 = A[i + (k + 3) * LDA] * b[k + 3];
        t1 = t1 + (m1 + m3);
        t2 = t2 + (m2 + m4);
      }
#pragma unroll
      for (int k = c4; k < i; ++k) t1 = t_fma(A[i + k * LDA], b[k], t1);
      b[i] = b[i] - (t1 + t2);
    }
    if (j < M) {
      // 3. rows j..M-1: GEMV-N update with the finished columns
      if (j >= 1)
        gemv_n_scheme<true>(M - j, j,
            [&](int i, int k) { return A[(j + i) + k * LDA]; }, b, b + j);
      // 4. pivot: first index of max |b[j:]|
      int p = j;
      T best = fabs(b[j]);
#pragma unroll
      for (int i = j + 1; i < M; ++i) {
        T v = fabs(b[i]);
        if (v > best) { best = v; p = i; }
      }
      piv[j] = p;
      // 5. interchange + scale (subnormal pivots left unscaled, as OpenBLAS)
      T bp = b[j];
#pragma unroll
      for (int i = j + 1; i < M; ++i)
        if (i == p) bp = b[i];
      if (bp != T(0)) {
#pragma unroll
        for (int k = 0; k < j; ++k) swap_dyn<M, 1>(A + k * LDA, j, p);
        swap_dyn<M, 1>(b, j, p);
        if (fabs(b[j]) >= Num<T>::dbl_min) {
          T r = T(1) / b[j];
#pragma unroll
          for (int i = j + 1; i < M; ++i) b[i] = b[i] * r;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) A[i + j * LDA] = b[i];
  }
}

// C(MI x NJ) -= A(MI x KK) * B(KK x NJ): one FMA chain per element, then subtract
template <int MI, int NJ, int KK, int LD, class T>
NLK_FD void gemm_minus(const T* A, const T* B, T* C) {
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      T acc = T(0);
#pragma unroll
      for (int k = 0; k < KK; ++k) acc = t_fma(A[i + k * LD], B[k + j * LD], acc);
      C[i + j * LD] = C[i + j * LD] - acc;
    }
}

// TRSM_KERNEL_LT with unit lower L (sub-blocks 16, then 8/4/2/1 by the bits of M)
template <int M, int NJ, int LD, int KK, class T>
NLK_FD void trsm_lt_blocks(const T* L, T* C) {
  if constexpr (KK < M) {
    constexpr int REM = M - KK;
    constexpr int BS = REM >= 16 ? 16 : (REM & 8) ? 8 : (REM & 4) ? 4 : (REM & 2) ? 2 : 1;
    if constexpr (KK > 0) gemm_minus<BS, NJ, KK, LD>(L + KK, C, C + KK);
#pragma unroll
    for (int i = 0; i < BS; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        T bb = C[KK + i + j * LD];
#pragma unroll
        for (int k = i + 1; k < BS; ++k)
          C[KK + k + j * LD] = t_fma(-bb, L[(KK + k) + (KK + i) * LD], C[KK + k + j * LD]);
      }
    trsm_lt_blocks<M, NJ, LD, KK + BS>(L, C);
  }
}

template <int M, int NC, int LD, class T> NLK_FD void getrf_rec(T* A, int* piv);

template <int M, int NC, int LD, int IS, int BLK, class T>
NLK_FD void getrf_blocks(T* A, int* piv) {
  constexpr int MN = M < NC ? M : NC;
  if constexpr (IS < MN) {
    constexpr int BK = (MN - IS) < BLK ? (MN - IS) : BLK;
    int sub[BK];
    getrf_rec<M - IS, BK, LD>(A + IS + IS * LD, sub);
#pragma unroll
    for (int i = 0; i < BK; ++i) piv[IS + i] = sub[i] + IS;
    if constexpr (IS + BK < NC) {
#pragma unroll
      for (int j = IS + BK; j < NC; ++j)
#pragma unroll
        for (int i = IS; i < IS + BK; ++i) swap_dyn<M, 1>(A + j * LD, i, piv[i]);
      trsm_lt_blocks<BK, NC - IS - BK, LD, 0>(A + IS + IS * LD, A + IS + (IS + BK) * LD);
      if constexpr (IS + BK < M)
        gemm_minus<M - IS - BK, NC - IS - BK, BK, LD>(A + (IS + BK) + IS * LD,
                                                       A + IS + (IS + BK) * LD,
                                                       A + (IS + BK) + (IS + BK) * LD);
    }
    getrf_blocks<M, NC, LD, IS + BK, BLK>(A, piv);
  }
}

template <int M, int NC, int LD, int IS, int BLK, class T>
NLK_FD void getrf_late_swaps(T* A, const int* piv) {
  constexpr int MN = M < NC ? M : NC;
  if constexpr (IS < MN) {
    constexpr int BK = (MN - IS) < BLK ? (MN - IS) : BLK;
#pragma unroll
    for (int j = IS; j < IS + BK; ++j)
#pragma unroll
      for (int i = IS + BK; i < MN; ++i) swap_dyn<M, 1>(A + j * LD, i, piv[i]);
    getrf_late_swaps<M, NC, LD, IS + BK, BLK>(A, piv);
  }
}

// getrf_single: blocking = round_up(mn/2, 2); GETF2 when blocking <= 4
template <int M, int NC, int LD, class T>
NLK_FD void getrf_rec(T* A, int* piv) {
  constexpr int MN = M < NC ? M : NC;
  constexpr int BLK = ((MN / 2 + 1) / 2) * 2;
  if constexpr (BLK <= 4) {
    getf2_panel<M, NC, LD>(A, piv);
  } else {
    getrf_blocks<M, NC, LD, 0, BLK>(A, piv);
    getrf_late_swaps<M, NC, LD, 0, BLK>(A, piv);
  }
}

// LuFactorization(A, strict=False) (linalg.py:87-105): returns false when
// nlkit raises SingularMatrix (zero/non-finite max|A| or an exactly zero
// pivot; a NaN pivot passes because np.min propagates NaN).
template <int N, class T>
NLK_FD bool lu_factor(T* A, int* piv) {
  T anorm = T(0);
  bool nan = false;
#pragma unroll
  for (int i = 0; i < N * N; ++i) {
    T a = fabs(A[i]);
    nan |= (a != a);
    anorm = a > anorm ? a : anorm;
  }
  if (nan || anorm == T(0) || !isfinite(anorm)) return false;
  getrf_rec<N, N, N>(A, piv);
  bool zero = false, pnan = false;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T d = fabs(A[i + i * N]);
    pnan |= (d != d);
    zero |= (d <= T(0));
  }
  return pnan || !zero;
}

// getrs (one RHS): row swaps, column-oriented FMA forward/back substitution
template <int N, class T>
NLK_FD void getrs(const T* LU, const int* piv, T* b) {
#pragma unroll
  for (int i = 0; i < N; ++i) swap_dyn<N, 1>(b, i, piv[i]);
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int r = i + 1; r < N; ++r) b[r] = t_fma(-b[i], LU[r + i * N], b[r]);
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    b[i] = b[i] / LU[i + i * N];
#pragma unroll
    for (int r = 0; r < i; ++r) b[r] = t_fma(-b[i], LU[r + i * N], b[r]);
  }
}

#undef NLK_FD
}  // namespace nlk
