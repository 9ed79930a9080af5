// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Operation-order models of the host BLAS/LAPACK kernels that the reference
// (nlkit) reaches through numpy and scipy.  nlkit's decisions (retcodes,
// iteration counts) are bitwise-sensitive on several problems (SURVEY.md
// App. A), so the oracle restates not only *what* is computed but the exact
// rounding sequence the reference host produced.  The models were identified
// on the container's host (OpenBLAS 0.3.30 / 0.3.31.dev, SkylakeX kernels) and
// are pinned by tests/test_oracle_blas.py against numpy/scipy directly.
//
// Call sites in the reference that these models stand in for:
//   ddot      : np.linalg.norm (numpy/linalg/_linalg.py: sqrt(x.dot(x))) used in
//               solvers.py:331-332,337, descent.py:91,98, quasinewton.py:118;
//               vector dots `f @ f`, `g @ g`, `s @ Ht` (globalize.py:130-132,
//               descent.py:95-96,103-104, quasinewton.py:117)
//   gemv_t    : `J @ v` with C-ordered J (globalize.py:128, descent.py:94,
//               quasinewton.py:101,115)
//   gemv_n    : `J.T @ v` (descent.py:64-65,93) and `s @ H` (quasinewton.py:116)
//   getrf     : scipy.linalg.lu_factor (linalg.py:98)
//   getrs     : scipy.linalg.lu_solve (linalg.py:107-108)
#pragma once
#include <vector>
#include <cmath>
#include <cstdint>

namespace oracle {

// ---- ddot -----------------------------------------------------------------
// n <= 15: one scalar FMA chain from 0.  n >= 16: blocks of 16 go through a
// 4-lane vector accumulator with separately rounded products, the lanes are
// reduced pairwise, and the tail continues as an FMA chain.
inline double ddot(int n, const double* x, int incx, const double* y, int incy) {
  int n16 = n & ~15;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  bool vec = n16 > 0;
  for (int b = 0; b < n16; b += 16) {
    for (int j = 0; j < 4; ++j) {
      double p0 = x[(b + j) * incx] * y[(b + j) * incy];
      double p1 = x[(b + j + 4) * incx] * y[(b + j + 4) * incy];
      double p2 = x[(b + j + 8) * incx] * y[(b + j + 8) * incy];
      double p3 = x[(b + j + 12) * incx] * y[(b + j + 12) * incy];
      if (b == 0) v[j] = ((p0 + p1) + p2) + p3;
      else v[j] = (((v[j] + p0) + p1) + p2) + p3;
    }
  }
  double s = vec ? (v[0] + v[2]) + (v[1] + v[3]) : 0.0;
  for (int i = n16; i < n; ++i) s = std::fma(x[i * incx], y[i * incy], s);
  return s;
}

inline double ddot(int n, const double* x, const double* y) { return ddot(n, x, 1, y, 1); }

// numpy's np.linalg.norm for a 1-D float vector: sqrt(x.dot(x)), no scaling
// (overflows to inf exactly like the reference).
inline double norm2(int n, const double* x) { return std::sqrt(ddot(n, x, x)); }

// ---- GEMV-N column scheme --------------------------------------------------
// Shared by getrf's left-looking update (y -= ...) and by numpy's `A.T @ x`.
// Rows are split into 4-row blocks (first M & ~3 rows) and a tail.  For a
// block row, columns are consumed 4 at a time with the chain (1,0,2,3), then
// 2 at a time with (1,0), then 1; each group's partial t is folded into y.
// Tail rows use one FMA chain from 0 over all columns, folded once.
// `a(i,k)` is the matrix element of row i, column k.
template <class Acc, class Fold>
inline void gemv_n_scheme(int m, int ncols, Acc a, const double* x, double* y, Fold fold) {
  int m1 = m & ~3;
  for (int i = 0; i < m1; ++i) {
    int k = 0;
    for (; k + 4 <= ncols; k += 4) {
      double t = a(i, k + 1) * x[k + 1];
      t = std::fma(a(i, k), x[k], t);
      t = std::fma(a(i, k + 2), x[k + 2], t);
      t = std::fma(a(i, k + 3), x[k + 3], t);
      y[i] = fold(y[i], t);
    }
    if (k + 2 <= ncols) {
      double t = a(i, k + 1) * x[k + 1];
      t = std::fma(a(i, k), x[k], t);
      y[i] = fold(y[i], t);
      k += 2;
    }
    if (k < ncols) {
      y[i] = fold(y[i], a(i, k) * x[k]);
    }
  }
  for (int i = m1; i < m; ++i) {
    if (ncols == 0) continue;
    double t = 0.0;
    for (int k = 0; k < ncols; ++k) t = std::fma(a(i, k), x[k], t);
    y[i] = fold(y[i], t);
  }
}

// numpy `A.T @ x` for a C-ordered n x n A (OpenBLAS dgemv_n on the
// Fortran view): y starts at 0 and each group partial is added.
inline void gemv_AT_x(int n, const double* A, const double* x, double* y) {
  for (int i = 0; i < n; ++i) y[i] = 0.0;
  gemv_n_scheme(n, n, [&](int i, int k) { return A[k * n + i]; }, x, y,
                [](double yi, double t) { return yi + t; });
}

// numpy `A @ x` for a C-ordered n x n A (OpenBLAS dgemv_t, Haswell-family
// kernels).  Output rows are produced in groups: rows 0 .. (n & ~3)-1 by the
// 4x4 kernel (4-lane FMA accumulators, reduced (v0+v2)+(v1+v3)); the next two
// rows, when n & 2, by the 4x2 kernel (2-lane SSE2 mul+add: even and odd
// columns, then v0+v1); the last row, when n & 1, by the 4x1 kernel (4-lane
// mul+add, reduced like 4x4).  All three run over the first n4 = n & ~3
// columns; the remaining 1-3 columns are folded in afterwards:
// r=1: fma(a, x, y); r=2: y + fma(a0, x0, a1*x1); r=3: y + fma(a2, x2, fma(a0, x0, a1*x1)).
// Pinned for every n = 1..16 by tests/test_oracle_blas.py.
inline double gemv_t_row(int n, int row, const double* a, const double* x) {
  const int n4 = n & ~3;
  const int nr4 = n & ~3;  // rows covered by the 4x4 kernel
  double s = 0.0;
  if (n4 > 0) {
    if (row < nr4) {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < n4; k += 4)
        for (int l = 0; l < 4; ++l) v[l] = std::fma(a[k + l], x[k + l], v[l]);
      s = (v[0] + v[2]) + (v[1] + v[3]);
    } else if ((n & 2) && row < nr4 + 2) {
      double v0 = 0.0, v1 = 0.0;
      for (int k = 0; k < n4; k += 2) {
        v0 = v0 + a[k] * x[k];
        v1 = v1 + a[k + 1] * x[k + 1];
      }
      s = v0 + v1;
    } else {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < n4; k += 4)
        for (int l = 0; l < 4; ++l) v[l] = v[l] + a[k + l] * x[k + l];
      s = (v[0] + v[2]) + (v[1] + v[3]);
    }
  }
  const int r = n - n4;
  if (r == 0) return s;
  if (r == 1) return std::fma(a[n4], x[n4], s);
  double t = std::fma(a[n4], x[n4], a[n4 + 1] * x[n4 + 1]);
  if (r == 3) t = std::fma(a[n4 + 2], x[n4 + 2], t);
  return n4 > 0 ? s + t : t;
}

inline void gemv_A_x(int n, const double* A, const double* x, double* y) {
  for (int i = 0; i < n; ++i) y[i] = gemv_t_row(n, i, A + i * n, x);
}

// ---- LAPACK getrf (OpenBLAS getrf_single + GETF2 + TRSM_LT + GEMM) ---------
// Column-major helpers; a(i, j) = A[i + j * lda].
//
// GETF2 (unblocked, left-looking) for an m x nc panel.  For each column j:
//  1. apply the earlier interchanges to b = A[:, j];
//  2. rows 1 <= i < j: b[i] -= sdot(L[i, 0:i], b[0:i]) (OpenBLAS ddot: blocks
//     of 4 rounded products into two partial sums, FMA tail, t1 + t2);
//  3. rows i >= j: GEMV-N update with the j finished columns (scheme above);
//  4. pivot = first index of max |b[j:]|;
//  5. swap rows over the finished columns; scale below the pivot by 1/pivot
//     unless the pivot is subnormal (OpenBLAS leaves the column unscaled).
inline void getf2_panel(int m, int nc, double* A, int lda, int* piv) {
  auto at = [&](int i, int j) -> double& { return A[i + j * lda]; };
  double b[64];
  for (int j = 0; j < nc; ++j) {
    for (int i = 0; i < m; ++i) b[i] = at(i, j);
    for (int i = 0; i < j && i < m; ++i) {
      int p = piv[i];
      if (p != i) { double t = b[i]; b[i] = b[p]; b[p] = t; }
    }
    for (int i = 1; i < j && i < m; ++i) {
      int c4 = i & ~3;
      double t1 = 0.0, t2 = 0.0;
      for (int k = 0; k < c4; k += 4) {
        double m1 = at(i, k) * b[k], m2 = at(i, k + 1) * b[k + 1];
        double m3 = at(i, k + 2) * b[k + 2], m4 = at(i, k + 3) * b[k + 3];
        t1 = t1 + (m1 + m3);
        t2 = t2 + (m2 + m4);
      }
      for (int k = c4; k < i; ++k) t1 = std::fma(at(i, k), b[k], t1);
      b[i] = b[i] - (t1 + t2);
    }
    if (j >= m) {
      for (int i = 0; i < m; ++i) at(i, j) = b[i];
      continue;
    }
    if (j >= 1)
      gemv_n_scheme(m - j, j, [&](int i, int k) { return at(j + i, k); }, b, b + j,
                    [](double y, double t) { return y - t; });
    int p = j;
    double best = std::fabs(b[j]);
    for (int i = j + 1; i < m; ++i) {
      double v = std::fabs(b[i]);
      if (v > best) { best = v; p = i; }
    }
    piv[j] = p;
    if (b[p] != 0.0) {
      if (p != j) {
        for (int k = 0; k < j; ++k) { double t = at(j, k); at(j, k) = at(p, k); at(p, k) = t; }
        double t = b[j]; b[j] = b[p]; b[p] = t;
      }
      if (std::fabs(b[j]) >= 2.2250738585072014e-308) {
        double r = 1.0 / b[j];
        for (int i = j + 1; i < m; ++i) b[i] = b[i] * r;
      }
    }
    for (int i = 0; i < m; ++i) at(i, j) = b[i];
  }
}

// GEMM_KERNEL_N with alpha = -1: C -= A * B, each element accumulated as one
// FMA chain over k from 0, then subtracted once.
inline void gemm_minus(int mi, int nj, int kk, const double* A, int lda, const double* B, int ldb,
                       double* C, int ldc) {
  for (int i = 0; i < mi; ++i)
    for (int j = 0; j < nj; ++j) {
      double acc = 0.0;
      for (int k = 0; k < kk; ++k) acc = std::fma(A[i + k * lda], B[k + j * ldb], acc);
      C[i + j * ldc] = C[i + j * ldc] - acc;
    }
}

// TRSM_KERNEL_LT with a unit lower L: rows in sub-blocks of 16, then 8/4/2/1
// by the bits of m; a GEMM update from the solved rows precedes each
// sub-block, then a right-looking FMA substitution inside it.
inline void trsm_lt_unit(int m, int nj, const double* L, int ldl, double* C, int ldc) {
  int sizes[24], ns = 0;
  for (int i = 0; i < m / 16; ++i) sizes[ns++] = 16;
  for (int i = 8; i > 0; i >>= 1)
    if (m & i) sizes[ns++] = i;
  int kk = 0;
  for (int s = 0; s < ns; ++s) {
    int bs = sizes[s];
    if (kk > 0) gemm_minus(bs, nj, kk, L + kk, ldl, C, ldc, C + kk, ldc);
    for (int i = 0; i < bs; ++i)
      for (int j = 0; j < nj; ++j) {
        double bb = C[kk + i + j * ldc];
        for (int k = i + 1; k < bs; ++k)
          C[kk + k + j * ldc] = std::fma(-bb, L[(kk + k) + (kk + i) * ldl], C[kk + k + j * ldc]);
      }
    kk += bs;
  }
}

// getrf_single (recursive, blocking = round_up(mn/2, UNROLL_N=2); GETF2 when
// blocking <= 2*UNROLL_N, i.e. for every n <= 9).
inline void getrf_cm(int m, int n, double* A, int lda, int* piv) {
  int mn = m < n ? m : n;
  int blocking = ((mn / 2 + 1) / 2) * 2;
  if (blocking <= 4) { getf2_panel(m, n, A, lda, piv); return; }
  for (int is = 0; is < mn; is += blocking) {
    int bk = mn - is < blocking ? mn - is : blocking;
    int sub[64];
    getrf_cm(m - is, bk, A + is + is * lda, lda, sub);
    for (int i = 0; i < bk; ++i) piv[is + i] = sub[i] + is;
    if (is + bk < n) {
      for (int j = is + bk; j < n; ++j)
        for (int i = is; i < is + bk; ++i) {
          int p = piv[i];
          if (p != i) { double t = A[i + j * lda]; A[i + j * lda] = A[p + j * lda]; A[p + j * lda] = t; }
        }
      trsm_lt_unit(bk, n - is - bk, A + is + is * lda, lda, A + is + (is + bk) * lda, lda);
      if (is + bk < m)
        gemm_minus(m - is - bk, n - is - bk, bk, A + (is + bk) + is * lda, lda,
                   A + is + (is + bk) * lda, lda, A + (is + bk) + (is + bk) * lda, lda);
    }
  }
  for (int is = 0; is < mn; is += blocking) {
    int bk = mn - is < blocking ? mn - is : blocking;
    for (int j = is; j < is + bk; ++j)
      for (int i = is + bk; i < mn; ++i) {
        int p = piv[i];
        if (p != i) { double t = A[i + j * lda]; A[i + j * lda] = A[p + j * lda]; A[p + j * lda] = t; }
      }
  }
}

// Row-major n x n front end used by the oracle: A is overwritten with L\U
// (unit L), piv[j] is the 0-based row interchanged with row j.  Bit-exact
// against scipy.linalg.lu_factor for every n = 1..16 (tests/test_oracle_blas.py).
inline void getrf(int n, double* A, int* piv) {
  double cm[256];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) cm[i + j * n] = A[i * n + j];
  getrf_cm(n, n, cm, n, piv);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A[i * n + j] = cm[i + j * n];
}

// ---- LAPACK getrs, one right-hand side --------------------------------------
inline void getrs(int n, const double* LU, const int* piv, double* b) {
  for (int i = 0; i < n; ++i) {
    int p = piv[i];
    if (p != i) { double t = b[i]; b[i] = b[p]; b[p] = t; }
  }
  for (int i = 0; i < n; ++i)
    for (int r = i + 1; r < n; ++r) b[r] = std::fma(-b[i], LU[r * n + i], b[r]);
  for (int i = n - 1; i >= 0; --i) {
    b[i] = b[i] / LU[i * n + i];
    for (int r = 0; r < i; ++r) b[r] = std::fma(-b[i], LU[r * n + i], b[r]);
  }
}

// ---- LAPACK getrs with trans = 'T', one right-hand side ----------------------
// scipy.linalg.lu_solve(..., trans=1) (linalg.py:110-112, used by
// sensitivity.ift_adjoint): OpenBLAS getrs_T for one RHS = trsv_TUN
// (forward: b_i = (b_i - ddot(U[0:i, i], b[0:i])) / U_ii), trsv_TLU
// (backward: b_i -= ddot(L[i+1:n, i], b[i+1:n])), then the row interchanges
// in reverse order.  Pinned against scipy in tests/test_oracle_blas.py.
inline void getrs_t(int n, const double* LU, const int* piv, double* b) {
  std::vector<double> col(n);
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < i; ++k) col[k] = LU[k * n + i];
    if (i > 0) b[i] -= ddot(i, col.data(), b);
    b[i] /= LU[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    const int len = n - 1 - i;
    for (int k = 0; k < len; ++k) col[k] = LU[(i + 1 + k) * n + i];
    if (len > 0) b[i] -= ddot(len, col.data(), b + i + 1);
  }
  for (int i = n - 1; i >= 0; --i) {
    int p = piv[i];
    if (p != i) { double t = b[i]; b[i] = b[p]; b[p] = t; }
  }
}

}  // namespace oracle
