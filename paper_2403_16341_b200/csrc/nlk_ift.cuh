// Batched implicit-function-theorem sensitivities at the roots
// (reference: nlkit/sensitivity.py:40-80, autodiff.param_jacobian
// autodiff.py:400-427, linalg.LuFactorization strict mode linalg.py:87-112).
//
// One thread per system, grid-stride:
//   _check_root       |f(u*, θ)|∞ <= 10·abstol, else NOT_A_ROOT (ValueError)
//   Ju = dense_jacobian(f, u*, θ)              (dual sweeps over u; NONFINITE)
//   Jt = param_jacobian(f, u*, θ)              (dual sweeps over θ; NONFINITE)
//   LU = LuFactorization(Ju) (strict=True)     (SINGULAR)
//   forward: S[:, j] = lu_solve(-Jt[:, j])     (one getrs per column)
//            full: max|Ju @ S + Jt|            (matmul = per-element FMA chain)
//   adjoint: λ = lu_solve(gbar, trans=1); grad = -(Jt.T @ λ)
//            full: max|Ju.T @ λ - gbar|
// Same BLAS/LAPACK operation-order models as the solvers (nlk_blas.cuh), plus
// getrs_t (trsv_TUN, trsv_TLU, reverse interchanges; pinned against scipy in
// tests/test_oracle_blas.py).
#pragma once
#include "nlk_solvers.cuh"

namespace nlk {

#define NLK_FD __device__ __forceinline__

enum IftStatus : int8_t { IFT_OK = 0, IFT_NOT_A_ROOT = 1, IFT_SINGULAR = 2, IFT_NONFINITE = 3 };

struct IftArgs {
  int64_t B;
  const void* u;      // [n][B]
  const void* theta;  // [m][B]
  const void* gbar;   // [n][B] (adjoint)
  double abstol;
  void* out;          // forward: S [n*m][B] (row-major n x m per system); adjoint: grad [m][B]
  void* resid;        // [B] or null (the `full=True` solve residual)
  int8_t* status;     // [B]
};

// np.max(np.abs(x)) over k values: NaN propagates
template <class T> NLK_FD T nanmax_abs(const T* x, int k) {
  T m = T(0);
  bool nan = false;
  for (int i = 0; i < k; ++i) {
    T a = fabs(x[i]);
    nan |= (a != a);
    m = a > m ? a : m;
  }
  return nan ? T(NAN) : m;
}

// param_jacobian (autodiff.py:400-427): dual sweeps over θ, column-major N x M
template <class P, int N, class T, int C0>
NLK_FD void param_sweeps(const T* u, const T* th, T* Jt, bool& ok) {
  constexpr int M = P::M;
  if constexpr (C0 < M) {
    constexpr int SW = SweepWidth<M>::value;
    constexpr int W = (M - C0) < SW ? (M - C0) : SW;
    Dual<W, T> td[M], out[N];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      td[i].v = th[i];
#pragma unroll
      for (int j = 0; j < W; ++j) td[i].d[j] = (i == C0 + j) ? T(1) : T(0);
    }
    P::template f_param<Dual<W, T>, T>(u, td, out);
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        ok &= isfinite(out[i].d[j]);  // _check_finite(parts) (autodiff.py:263-266)
        Jt[i + (C0 + j) * N] = out[i].d[j];
      }
    param_sweeps<P, N, T, C0 + W>(u, th, Jt, ok);
  }
}

// LuFactorization(A, strict=True) (linalg.py:87-105)
template <int N, class T>
NLK_FD bool lu_factor_strict(T* A, int* piv) {
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
  const T tol = Num<T>::eps * anorm * T(N);
  T pmin = T(INFINITY);
  bool pnan = false;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T d = fabs(A[i + i * N]);
    pnan |= (d != d);
    pmin = d < pmin ? d : pmin;
  }
  return pnan || !(pmin <= tol);  // np.min propagates NaN; NaN <= tol is False
}

// lu_solve(..., trans=1), one RHS: trsv_TUN, trsv_TLU, reverse interchanges
template <int N, class T>
NLK_FD void getrs_t(const T* LU, const int* piv, T* b) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i > 0) {
      T col[N];
#pragma unroll
      for (int k = 0; k < i; ++k) col[k] = LU[k + i * N];
      b[i] = b[i] - ddot_n<T>(i, col, b);
    }
    b[i] = b[i] / LU[i + i * N];
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const int len = N - 1 - i;
    if (len > 0) {
      T col[N];
#pragma unroll
      for (int k = 0; k < len; ++k) col[k] = LU[(i + 1 + k) + i * N];
      b[i] = b[i] - ddot_n<T>(len, col, b + i + 1);
    }
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) swap_dyn<N, 1>(b, i, piv[i]);
}

template <class P, int N, class T, bool ADJ>
__global__ void __launch_bounds__(128) ift_kernel(const IftArgs a) {
  constexpr int M = P::M;
  constexpr int KM = MemoOf<P>::value;
  static_assert(M > 0, "sensitivities need parameters");
  const T* __restrict__ U = static_cast<const T*>(a.u);
  const T* __restrict__ TH = static_cast<const T*>(a.theta);
  const T* __restrict__ G = static_cast<const T*>(a.gbar);
  T* __restrict__ O = static_cast<T*>(a.out);
  T* __restrict__ R = static_cast<T*>(a.resid);
  const int64_t B = a.B;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    T u[N], th[M];
#pragma unroll
    for (int i = 0; i < N; ++i) u[i] = U[i * B + b];
#pragma unroll
    for (int i = 0; i < M; ++i) th[i] = TH[i * B + b];
    int8_t st = IFT_OK;
    // _check_root (sensitivity.py:31-36)
    T memo[KM > 0 ? KM : 1];
    T r[N];
    {
      Ctx<T, (KM > 0 ? 1 : 0)> cx{memo, 0};
      P::template f<T, T>(u, th, r, cx);
    }
    const T rmax = nanmax_abs(r, N);
    T Ju[N * N], Jt[N * M], LU[N * N];
    int piv[N];
    if (!(rmax <= T(10) * static_cast<T>(a.abstol))) {
      st = IFT_NOT_A_ROOT;
    } else if (jacobian<P, N, T, KM>(u, th, memo, Ju) >= 0) {
      st = IFT_NONFINITE;
    } else {
      bool ok = true;
      param_sweeps<P, N, T, 0>(u, th, Jt, ok);
      if (!ok) {
        st = IFT_NONFINITE;
      } else {
#pragma unroll
        for (int i = 0; i < N * N; ++i) LU[i] = Ju[i];
        if (!lu_factor_strict<N>(LU, piv)) st = IFT_SINGULAR;
      }
    }
    a.status[b] = st;
    if constexpr (!ADJ) {
      T S[N * M];  // column-major N x M
      if (st == IFT_OK) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
          T x[N];
#pragma unroll
          for (int i = 0; i < N; ++i) x[i] = -Jt[i + j * N];
          getrs<N>(LU, piv, x);
#pragma unroll
          for (int i = 0; i < N; ++i) S[i + j * N] = x[i];
        }
      } else {
#pragma unroll
        for (int e = 0; e < N * M; ++e) S[e] = T(NAN);
      }
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) O[(i * M + j) * B + b] = S[i + j * N];
      if (R) {
        T res = T(NAN);
        if (st == IFT_OK) {  // max|Ju @ S + Jt| (sensitivity.py:53)
          T E[N * M];
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
              T acc = T(0);
#pragma unroll
              for (int k = 0; k < N; ++k) acc = t_fma(Ju[i + k * N], S[k + j * N], acc);
              E[i + j * N] = acc + Jt[i + j * N];
            }
          res = nanmax_abs(E, N * M);
        }
        R[b] = res;
      }
    } else {
      T grad[M];
      T lam[N];
      if (st == IFT_OK) {
#pragma unroll
        for (int i = 0; i < N; ++i) lam[i] = G[i * B + b];
        getrs_t<N>(LU, piv, lam);
        // Jt.T @ lam: Jt is C-ordered n x m in numpy, its transpose an
        // F-ordered view -> dgemv_n (the `A.T @ x` model)
#pragma unroll
        for (int j = 0; j < M; ++j) grad[j] = T(0);
        gemv_n_scheme<false>(M, N, [&](int j, int k) { return Jt[k + j * N]; }, lam, grad);
#pragma unroll
        for (int j = 0; j < M; ++j) grad[j] = -grad[j];
      } else {
#pragma unroll
        for (int j = 0; j < M; ++j) grad[j] = T(NAN);
      }
#pragma unroll
      for (int j = 0; j < M; ++j) O[j * B + b] = grad[j];
      if (R) {
        T res = T(NAN);
        if (st == IFT_OK) {  // max|Ju.T @ lam - gbar| (sensitivity.py:79)
          T y[N], d[N];
          gemv_AT_x<N>(Ju, lam, y);
#pragma unroll
          for (int i = 0; i < N; ++i) d[i] = y[i] - G[i * B + b];
          res = nanmax_abs(d, N);
        }
        R[b] = res;
      }
    }
  }
}

using IftLauncher = cudaError_t (*)(const IftArgs&, cudaStream_t);

template <class P, class T, bool ADJ>
cudaError_t launch_ift(const IftArgs& a, cudaStream_t stream) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  int64_t want = (a.B + 127) / 128;
  int64_t grid = static_cast<int64_t>(sms) * 8;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  ift_kernel<P, P::N, T, ADJ><<<static_cast<unsigned>(grid), 128, 0, stream>>>(a);
  return cudaGetLastError();
}

struct IftEntry {
  const char* id;
  int n, m;
  IftLauncher forward, adjoint;  // f64
};
#define NLK_IFT_ENTRY(ID, P) {ID, P::N, P::M, &launch_ift<P, double, false>, &launch_ift<P, double, true>}

struct IftTable {
  const IftEntry* entries;
  int count;
};
IftTable registry_ift();

#undef NLK_FD
}  // namespace nlk
