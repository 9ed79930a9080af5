// Shared-memory LU for the larger systems (n >= NLK_SMEM_NR_MIN / _TR_MIN).
//
// The register-resident LU of nlk_blas.cuh applies row interchanges with
// predicated swaps (a data-dependent pivot cannot index a register array):
// at n = 9/10 that is O(n^3) selects, ~14k SASS instructions per kernel, the
// kernels stall on instruction fetch and spill.  Here the matrix lives in a
// per-thread slice of shared memory (element e of thread t at
// smem[e * 128 + t]: consecutive lanes hit consecutive words, conflict-free).
// Loops are fully unrolled, so every element address is an immediate offset
// from the thread's slice base, and an interchange is two indexed loads and
// stores instead of a select chain.  Measured on B200 (C2, B = 262144):
// 740 ms -> 417 ms per step; rolled loops (NLK_SMEM_UNROLL=0) are smaller
// but spend their issue slots on address arithmetic (736 ms).
// The arithmetic is the same OpenBLAS getrf/GETF2/TRSM/GEMM + getrs operation
// sequence as nlk_blas.cuh, element for element.
#pragma once
#include "nlk_blas.cuh"
#include "nlk_div.cuh"

namespace nlk {

// n thresholds for the shared-memory path, per driver.  First used for
// n >= 9 only; measured on the C2/C5 jobs (profiles/r01c_variants_ab.txt)
// the shared-memory LU is as fast or faster down to n = 2 as well (n = 4
// trust region: 34.5 -> 29.2 ms on matrix-sqrt-2x2; the register LU's
// predicated interchanges disappear), so only n = 1 keeps registers.
#ifndef NLK_SMEM_NR_MIN
#define NLK_SMEM_NR_MIN 2
#endif
#ifndef NLK_SMEM_TR_MIN
#define NLK_SMEM_TR_MIN 2
#endif
// 1: unroll every loop (immediate smem offsets); 0: rolled loops
#ifndef NLK_SMEM_UNROLL
#define NLK_SMEM_UNROLL 1
#endif
#if NLK_SMEM_UNROLL
#define NLK_SMU _Pragma("unroll")
#else
#define NLK_SMU _Pragma("unroll 1")
#endif

// 1: getrs' back substitution divides with reciprocals refined up front
#ifndef NLK_GETRS_HOIST_DIV
#define NLK_GETRS_HOIST_DIV 0
#endif
// 1: getrs substitutes on a register copy of the permuted right-hand side
// (round 2: msqrt-3x3 TR 161.2 -> 159.0 ms, trig TR 60.9 -> 60.6; neutral in
// round 1)
#ifndef NLK_GETRS_REG
#define NLK_GETRS_REG 1
#endif

#define NLK_FD __device__ __forceinline__

// threads per block of the solve kernel = stride of the per-thread slices
constexpr int kSmStride = 128;

// column-major N x N matrix in a strided per-thread shared-memory slice
// (S = the block size: element e of thread t at smem[e * S + t])
template <int N, class T, int S = kSmStride>
struct SMat {
  T* base;
  NLK_FD T& operator()(int i, int j) const { return base[(i + j * N) * S]; }
  NLK_FD T& v(int i) const { return base[i * S]; }  // as a vector
};

template <int N, class T, int S> NLK_FD T mat_at(const SMat<N, T, S>& A, int e) { return A.v(e); }

template <int N, class T, int S>
NLK_FD void sm_swap_rows(const SMat<N, T, S>& A, int r1, int r2, int c0, int c1) {
NLK_SMU
  for (int k = c0; k < c1; ++k) {
    T t = A(r1, k);
    A(r1, k) = A(r2, k);
    A(r2, k) = t;
  }
}

// Row interchanges as one gather (NLK_LU_GATHER, default on).  A sequence of
// interchanges applied to a column one after the other is a chain of
// dependent shared-memory loads and stores with data-dependent addresses
// (any two may alias) -- ncu put ~20 % of the matrix-sqrt-3x3 trust region's
// stall samples on those lines.  The same data movement as one gather: the
// composed permutation is kept as packed 4-bit row indices (n <= 16), row r of
// the permuted column is row perm_get(R, r) of the stored one, so the N loads
// are independent and the stores go to static addresses.  Values move, none
// is computed: bit-identical by construction.
#ifndef NLK_LU_GATHER
#define NLK_LU_GATHER 1
#endif
// 1: the pivot search, interchange and scaling of the current column work on
// a register copy of it (no data-dependent reload after the search)
#ifndef NLK_LU_PIVREG
#define NLK_LU_PIVREG 0
#endif
template <int N> NLK_FD constexpr uint64_t perm_identity() {
  uint64_t r = 0;
  for (int i = 0; i < N; ++i) r |= static_cast<uint64_t>(i) << (4 * i);
  return r;
}
NLK_FD int perm_get(uint64_t R, int i) { return static_cast<int>((R >> (4 * i)) & 15u); }
// R after interchanging positions i and p
NLK_FD uint64_t perm_swap(uint64_t R, int i, int p) {
  const uint64_t x = ((R >> (4 * i)) ^ (R >> (4 * p))) & 15u;
  return R ^ (x << (4 * i)) ^ (x << (4 * p));
}
// the interchanges of A followed by those of B: (A o B)[r] = A[B[r]]
template <int N> NLK_FD uint64_t perm_compose(uint64_t A, uint64_t B) {
  uint64_t r = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) r |= static_cast<uint64_t>(perm_get(A, perm_get(B, i))) << (4 * i);
  return r;
}
// rows r0..N-1 of column c <- rows perm_get(R, r) (rows below r0 are fixed)
template <int N, class T, int S>
NLK_FD void sm_gather_col(const SMat<N, T, S>& A, uint64_t R, int r0, int c) {
  T col[N];
NLK_SMU
  for (int r = r0; r < N; ++r) col[r] = A(perm_get(R, r), c);
NLK_SMU
  for (int r = r0; r < N; ++r) A(r, c) = col[r];
}

// GETF2 on rows OFF..N-1, columns OFF..OFF+NC-1; piv holds absolute rows.
// Returns the panel's interchanges composed (perm_* form).
template <int N, class T, int S, class DV = ExactDiv>
NLK_FD uint64_t sm_getf2(const SMat<N, T, S>& A, int OFF, int NC, int* piv, DV dv = DV{nullptr}) {
  const int M = N - OFF;
  uint64_t R = perm_identity<N>();
NLK_SMU
  for (int j = 0; j < NC; ++j) {
    const int c = OFF + j;
    // 1. earlier interchanges of this panel, applied to column c
#if NLK_LU_GATHER
    if (j > 0) sm_gather_col(A, R, OFF, c);
#else
NLK_SMU
    for (int i = 0; i < j; ++i) {
      const int p = piv[OFF + i];  // p == row: a no-op swap (branch-free)
      const T t = A(OFF + i, c);
      A(OFF + i, c) = A(p, c);
      A(p, c) = t;
    }
#endif
    // 2. rows 1..j-1: b_i -= sdot(L[i, 0:i], b[0:i])
NLK_SMU
    for (int i = 1; i < j; ++i) {
      const int c4 = i & ~3;
      T t1 = T(0), t2 = T(0);
NLK_SMU
      for (int k = 0; k < c4; k += 4) {
        T m1 = A(OFF + i, OFF + k) * A(OFF + k, c);
        T m2 = A(OFF + i, OFF + k + 1) * A(OFF + k + 1, c);
        T m3 = A(OFF + i, OFF + k + 2) * A(OFF + k + 2, c);
        T m4 = A(OFF + i, OFF + k + 3) * A(OFF + k + 3, c);
        t1 = t1 + (m1 + m3);
        t2 = t2 + (m2 + m4);
      }
NLK_SMU
      for (int k = c4; k < i; ++k) t1 = t_fma(A(OFF + i, OFF + k), A(OFF + k, c), t1);
      A(OFF + i, c) = A(OFF + i, c) - (t1 + t2);
    }
    if (j >= M) continue;
    // 3. rows j..M-1: GEMV-N scheme with the j finished columns
    if (j >= 1) {
      const int MM = M - j, M1 = MM & ~3;
NLK_SMU
      for (int ii = 0; ii < MM; ++ii) {
        const int r = OFF + j + ii;
        T y = A(r, c);
        if (ii < M1) {
          int k = 0;
NLK_SMU
          for (; k + 4 <= j; k += 4) {
            T t = A(r, OFF + k + 1) * A(OFF + k + 1, c);
            t = t_fma(A(r, OFF + k), A(OFF + k, c), t);
            t = t_fma(A(r, OFF + k + 2), A(OFF + k + 2, c), t);
            t = t_fma(A(r, OFF + k + 3), A(OFF + k + 3, c), t);
            y = y - t;
          }
          if (k + 2 <= j) {
            T t = A(r, OFF + k + 1) * A(OFF + k + 1, c);
            t = t_fma(A(r, OFF + k), A(OFF + k, c), t);
            y = y - t;
            k += 2;
          }
          if (k < j) y = y - A(r, OFF + k) * A(OFF + k, c);
        } else {
          T t = T(0);
NLK_SMU
          for (int k = 0; k < j; ++k) t = t_fma(A(r, OFF + k), A(OFF + k, c), t);
          y = y - t;
        }
        A(r, c) = y;
      }
    }
#if NLK_LU_PIVREG
    // 4. pivot: first index of max |b[j:]|, on a register copy of b[j:]
    //    (the pivot value comes out of the search, so the interchange of b
    //    and its scaling need no data-dependent shared-memory load)
    T colv[N];
NLK_SMU
    for (int r = c; r < N; ++r) colv[r] = A(r, c);
    int p = c;
    T best = fabs(colv[c]), pv = colv[c];
NLK_SMU
    for (int r = c + 1; r < N; ++r) {
      T v = fabs(colv[r]);
      if (v > best) { best = v; p = r; pv = colv[r]; }
    }
    piv[c] = p;
    R = perm_swap(R, c, p);
    // 5. interchange over the finished panel columns and b, then scale
    if (best != T(0)) {  // == (A(p, c) != 0): best is |A(p, c)| (NaN included)
      sm_swap_rows(A, c, p, OFF, c);
      T outv[N];
      outv[c] = pv;  // bj: the old A(p, c)
NLK_SMU
      for (int r = c + 1; r < N; ++r) outv[r] = (r == p) ? colv[c] : colv[r];
      if (fabs(pv) >= Num<T>::dbl_min) {
        const T rr = dv(T(1), pv);
NLK_SMU
        for (int r = c + 1; r < N; ++r) outv[r] = outv[r] * rr;
      }
NLK_SMU
      for (int r = c; r < N; ++r) A(r, c) = outv[r];
    }
#else
    // 4. pivot: first index of max |b[j:]|
    int p = c;
    T best = fabs(A(c, c));
NLK_SMU
    for (int r = c + 1; r < N; ++r) {
      T v = fabs(A(r, c));
      if (v > best) { best = v; p = r; }
    }
    piv[c] = p;
    R = perm_swap(R, c, p);
    // 5. interchange over the finished panel columns and b, then scale
    if (best != T(0)) {  // == (A(p, c) != 0): best is |A(p, c)| (NaN included)
      sm_swap_rows(A, c, p, OFF, c + 1);
      const T bj = A(c, c);
      if (fabs(bj) >= Num<T>::dbl_min) {
        const T rr = dv(T(1), bj);
NLK_SMU
        for (int r = c + 1; r < N; ++r) A(r, c) = A(r, c) * rr;
      }
    }
#endif
  }
  return R;
}

// C(rows r0.., cols c0..) -= A(rows r0.., cols k0..k0+KK) * B(rows k0.., cols c0..)
template <int N, class T, int S>
NLK_FD void sm_gemm_minus(const SMat<N, T, S>& A, int r0, int MI, int c0, int NJ, int k0, int KK) {
NLK_SMU
  for (int i = 0; i < MI; ++i)
NLK_SMU
    for (int j = 0; j < NJ; ++j) {
      T acc = T(0);
NLK_SMU
      for (int k = 0; k < KK; ++k) acc = t_fma(A(r0 + i, k0 + k), A(k0 + k, c0 + j), acc);
      A(r0 + i, c0 + j) = A(r0 + i, c0 + j) - acc;
    }
}

// TRSM_LT (unit L) on rows IS..IS+BK-1, columns C0..N-1; sub-blocks follow
// the bits of BK (BK <= 8 here, so no 16-blocks)
template <int N, class T, int S>
NLK_FD void sm_trsm(const SMat<N, T, S>& A, int IS, int BK) {
  const int C0 = IS + BK, NJ = N - C0;
  int kk = 0;
NLK_SMU
  for (int bs = 8; bs >= 1; bs >>= 1) {
    if (!(BK & bs)) continue;
    if (kk > 0) sm_gemm_minus(A, IS + kk, bs, C0, NJ, IS, kk);
NLK_SMU
    for (int i = 0; i < bs; ++i)
NLK_SMU
      for (int j = 0; j < NJ; ++j) {
        const T bb = A(IS + kk + i, C0 + j);
NLK_SMU
        for (int k = i + 1; k < bs; ++k)
          A(IS + kk + k, C0 + j) = t_fma(-bb, A(IS + kk + k, IS + kk + i), A(IS + kk + k, C0 + j));
      }
    kk += bs;
  }
}

template <int N, class T, int S, class DV = ExactDiv>
NLK_FD void sm_getrf(const SMat<N, T, S>& A, int* piv, DV dv = DV{nullptr}) {
  constexpr int BLK = ((N / 2 + 1) / 2) * 2;
  if constexpr (BLK <= 4) {
    sm_getf2(A, 0, N, piv, dv);
  } else {
    constexpr int NP = (N + BLK - 1) / BLK;
    uint64_t Rp[NP];  // each panel's interchanges, composed
NLK_SMU
    for (int is = 0; is < N; is += BLK) {
      const int bk = (N - is) < BLK ? (N - is) : BLK;
      Rp[is / BLK] = sm_getf2(A, is, bk, piv, dv);  // panels of n <= 16 are always GETF2
      if (is + bk < N) {
#if NLK_LU_GATHER
NLK_SMU
        for (int k = is + bk; k < N; ++k) sm_gather_col(A, Rp[is / BLK], is, k);
#else
NLK_SMU
        for (int i = is; i < is + bk; ++i)
          sm_swap_rows(A, i, piv[i], is + bk, N);
#endif
        sm_trsm(A, is, bk);
        sm_gemm_minus(A, is + bk, N - is - bk, is + bk, N - is - bk, is, bk);
      }
    }
#if NLK_LU_GATHER
    // later panels' interchanges applied to each earlier panel's columns
    uint64_t Rl = perm_identity<N>();
NLK_SMU
    for (int q = NP - 1; q >= 1; --q) {
      Rl = perm_compose<N>(Rp[q], Rl);
      const int is = (q - 1) * BLK;
NLK_SMU
      for (int k = is; k < is + BLK; ++k) sm_gather_col(A, Rl, q * BLK, k);
    }
#else
NLK_SMU
    for (int is = 0; is < N; is += BLK) {
      const int bk = (N - is) < BLK ? (N - is) : BLK;
NLK_SMU
      for (int i = is + bk; i < N; ++i)
        sm_swap_rows(A, i, piv[i], is, is + bk);
    }
#endif
  }
}

// JAC_CHECKED: A is a Jacobian that passed dense_jacobian's finiteness
// checks, so max|A| is finite and the scan below can only reject an all-zero
// matrix -- which getrf rejects anyway (every pivot is zero), with the same
// outcome (SingularMatrix -> LINSOLVE_FAILED).  The scan is skipped then.
template <int N, bool JAC_CHECKED, class T, int S, class DV = ExactDiv>
NLK_FD bool sm_lu_factor(const SMat<N, T, S>& A, int* piv, DV dv = DV{nullptr}) {
  if constexpr (!JAC_CHECKED) {
    T anorm = T(0);
    bool nan = false;
NLK_SMU
    for (int e = 0; e < N * N; ++e) {
      const T a = fabs(A.v(e));
      nan |= (a != a);
      anorm = a > anorm ? a : anorm;
    }
    if (nan || anorm == T(0) || !isfinite(anorm)) return false;
  }
  sm_getrf(A, piv, dv);
  bool zero = false, pnan = false;
NLK_SMU
  for (int i = 0; i < N; ++i) {
    const T d = fabs(A(i, i));
    pnan |= (d != d);
    zero |= (d <= T(0));
  }
  return pnan || !zero;
}

// getrs with the right-hand side in the strided vector b (N elements)
template <int N, class T, int S, class DV = ExactDiv>
NLK_FD void sm_getrs(const SMat<N, T, S>& LU, const int* piv, const SMat<N, T, S>& b, DV dv = DV{nullptr}) {
#if NLK_LU_GATHER
  {
    uint64_t R = perm_identity<N>();
#pragma unroll
    for (int i = 0; i < N; ++i) R = perm_swap(R, i, piv[i]);
    T x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = b.v(perm_get(R, i));
#pragma unroll
    for (int i = 0; i < N; ++i) b.v(i) = x[i];
  }
#else
NLK_SMU
  for (int i = 0; i < N; ++i) {
    const int p = piv[i];
    const T t = b.v(i);
    b.v(i) = b.v(p);
    b.v(p) = t;
  }
#endif
#if NLK_GETRS_REG
  // the substitutions on a register copy of the permuted right-hand side
  T x[N];
NLK_SMU
  for (int i = 0; i < N; ++i) x[i] = b.v(i);
NLK_SMU
  for (int i = 0; i < N; ++i) {
NLK_SMU
    for (int r = i + 1; r < N; ++r) x[r] = t_fma(-x[i], LU(r, i), x[r]);
  }
NLK_SMU
  for (int i = N - 1; i >= 0; --i) {
    x[i] = dv(x[i], LU(i, i));
NLK_SMU
    for (int r = 0; r < i; ++r) x[r] = t_fma(-x[i], LU(r, i), x[r]);
  }
NLK_SMU
  for (int i = 0; i < N; ++i) b.v(i) = x[i];
#else
NLK_SMU
  for (int i = 0; i < N; ++i) {
    const T bi = b.v(i);
NLK_SMU
    for (int r = i + 1; r < N; ++r) b.v(r) = t_fma(-bi, LU(r, i), b.v(r));
  }
#if NLK_GETRS_HOIST_DIV
  // the divisors' reciprocal refinements first (independent), then each
  // division of the serial chain finishes in three operations (nlk_div.cuh)
  T rd[N];
NLK_SMU
  for (int i = 0; i < N; ++i) rd[i] = div_rcp(LU(i, i));
#endif
NLK_SMU
  for (int i = N - 1; i >= 0; --i) {
#if NLK_GETRS_HOIST_DIV
    const T bi = div_with_rcp(b.v(i), LU(i, i), rd[i]);
#else
    const T bi = dv(b.v(i), LU(i, i));
#endif
    b.v(i) = bi;
NLK_SMU
    for (int r = 0; r < i; ++r) b.v(r) = t_fma(-bi, LU(r, i), b.v(r));
  }
#endif
}

// smem path when n >= MIN_N and the N*N + N slice of one block fits in
// 200 KB.  The block size (= slice stride) is 128 threads where it fits
// (f64: n <= 13; f32: n <= 18), else 64 or 32: n = 14..16 in f64 run 32-thread
// blocks (69.6 KB each at n = 16, three per SM) rather than a register LU
// whose 256 doubles spill (17.6 KB of spill stores per thread at n = 16).
template <int N, class T, int MIN_N> struct UseSmemLU {
  static constexpr int kSlice = sizeof(T) * (N * N + N);
  static constexpr int stride = kSlice * 128 <= 200 * 1024 ? 128
                              : kSlice * 64 <= 200 * 1024 ? 64
                              : kSlice * 32 <= 200 * 1024 ? 32 : 0;
  // the pivot permutation packs 4-bit row indices into a uint64 (perm_*)
  static constexpr bool value = N >= MIN_N && stride > 0 && N <= 16;
};

#undef NLK_SMU
#undef NLK_FD
}  // namespace nlk
