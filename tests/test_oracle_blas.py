"""Pin the oracle's BLAS/LAPACK operation-order models against the host
numpy/scipy the reference calls (bit-exact, every n = 1..16).

These models stand in for linalg.py:98,107-108 (getrf/getrs), numpy dots and
norms (solvers.py:331-337, descent.py:91-104, globalize.py:128-132) and the
matrix-vector products of descent.py:93-94 / quasinewton.py:101,115-116.
"""

import numpy as np
import pytest
import scipy.linalg

from oracle import oracle as O


@pytest.mark.parametrize("n", range(1, 17))
def test_blas_models_bit_exact(n):
    L = O.lib()
    rng = np.random.default_rng(100 + n)
    for _ in range(60):
        A = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (n, n)))
        x = rng.standard_normal(n)
        y = rng.standard_normal(n)
        assert L.oracle_ddot(n, x, y) == x @ y
        o = np.empty(n)
        L.oracle_gemv_A_x(n, A, x, o)
        assert np.array_equal(o, A @ x)
        L.oracle_gemv_AT_x(n, A, x, o)
        assert np.array_equal(o, A.T @ x)
        lu, piv = scipy.linalg.lu_factor(A)
        M = A.copy()
        pv = np.zeros(n, np.int32)
        L.oracle_getrf(n, M, pv)
        assert np.array_equal(M, lu) and np.array_equal(pv, piv)
        b = x.copy()
        L.oracle_getrs(n, np.ascontiguousarray(lu), piv.astype(np.int32), b)
        assert np.array_equal(b, scipy.linalg.lu_solve((lu, piv), x))
        b = y.copy()  # trans=1: sensitivity.ift_adjoint's solve_transpose (linalg.py:110-112)
        L.oracle_getrs_t(n, np.ascontiguousarray(lu), piv.astype(np.int32), b)
        assert np.array_equal(b, scipy.linalg.lu_solve((lu, piv), y, trans=1))


def test_getrf_singular_and_subnormal_pivots():
    L = O.lib()
    for A in (np.array([[0.0, 1.0], [0.0, 2.0]]), np.array([[1e-310, 1.0], [1e-311, 3.0]]),
              np.diag([1.0, 0.0, 2.0])):
        n = A.shape[0]
        lu, piv = scipy.linalg.lu_factor(A, check_finite=False)
        M = A.copy()
        pv = np.zeros(n, np.int32)
        L.oracle_getrf(n, M, pv)
        assert np.array_equal(M, lu) and np.array_equal(pv, piv)
