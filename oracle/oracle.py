"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front-end of ``liboracle.so`` — the CPU restatement of nlkit's
per-system solvers (see nlk_oracle.cpp for the reference file:line map).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg may import this module; it is the checker, never the
thing measured or shipped.  The product package never imports it.

Parity status: pinned against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py); DFSane is builder-authored and
unpinned (the reference has no DFSane).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

ALGS = {"newton-raphson": 0, "trust-region": 1, "broyden": 2, "klement": 3,
        "dfsane": 4, "newton-backtracking": 5}
RETCODES = ("Success", "MaxIters", "LineSearchFailed", "LinearSolveFailed",
            "Stalled", "NonFinite")

_lib = None


def build():
    """Compile liboracle.so with oracle/Makefile (g++, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = np.ctypeslib.ndpointer(np.float64, flags="C")
        ip = np.ctypeslib.ndpointer(np.int32, flags="C")
        i8 = np.ctypeslib.ndpointer(np.int8, flags="C")
        c_int, c_i64, c_d = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.oracle_lookup.argtypes = [ctypes.c_char_p, c_int, ctypes.POINTER(c_int),
                                    ctypes.POINTER(c_int), ctypes.POINTER(c_int)]
        L.oracle_residual.argtypes = [c_int, c_int, dp, ctypes.c_void_p, dp]
        L.oracle_jacobian.argtypes = [c_int, c_int, dp, ctypes.c_void_p, dp]
        L.oracle_solve_batch.argtypes = [c_int, c_int, c_int, c_i64, dp, ctypes.c_void_p, c_int,
                                         c_d, c_int, c_int, dp, dp, i8, ip, ip, ip, ip, c_int]
        L.oracle_ddot.restype = c_d
        L.oracle_ddot.argtypes = [c_int, dp, dp]
        L.oracle_gemv_A_x.argtypes = [c_int, dp, dp, dp]
        L.oracle_gemv_AT_x.argtypes = [c_int, dp, dp, dp]
        L.oracle_getrf.argtypes = [c_int, dp, ip]
        L.oracle_getrs.argtypes = [c_int, dp, ip, dp]
        L.oracle_getrs_t.argtypes = [c_int, dp, ip, dp]
        _lib = L
    return _lib


def lookup(problem_id, n=0):
    h, nn, m = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = lib().oracle_lookup(problem_id.encode(), int(n), ctypes.byref(h), ctypes.byref(nn),
                             ctypes.byref(m))
    if rc != 0:
        raise KeyError(f"oracle: unknown problem {problem_id!r} (n={n}, rc={rc})")
    return h.value, nn.value, m.value


def _pptr(p):
    return None if p is None else p.ctypes.data_as(ctypes.c_void_p)


def residual(problem_id, x, p=None, n=0):
    h, nn, m = lookup(problem_id, n or len(x))
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = None if m == 0 else np.ascontiguousarray(p, dtype=np.float64)
    f = np.empty(nn)
    lib().oracle_residual(h, nn, x, _pptr(p), f)
    return f


def jacobian(problem_id, x, p=None, n=0):
    """Dual-path Jacobian; returns None on NonFiniteValue."""
    h, nn, m = lookup(problem_id, n or len(x))
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = None if m == 0 else np.ascontiguousarray(p, dtype=np.float64)
    J = np.empty((nn, nn))
    ok = lib().oracle_jacobian(h, nn, x, _pptr(p), J)
    return J if ok else None


def solve_batch(problem_id, alg, u0, p=None, abstol=1e-8, maxiters=1000, threads=None, nudge=0):
    """Solve B systems (u0 [B, n], p [B, m]); returns a dict of arrays.
    nudge=+1/-1 moves every float residual one ulp up/down (sensitivity probe)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    B, n = u0.shape
    h, nn, m = lookup(problem_id, n)
    if m:
        p = np.ascontiguousarray(p, dtype=np.float64).reshape(B, m)
    else:
        p = None
    out = {
        "u": np.empty((B, n)), "resid": np.empty(B),
        "retcode": np.empty(B, np.int8), "nsteps": np.empty(B, np.int32),
        "nf": np.empty(B, np.int32), "njac": np.empty(B, np.int32),
        "nlinsolve": np.empty(B, np.int32),
    }
    threads = threads or os.cpu_count() or 1
    rc = lib().oracle_solve_batch(h, n, ALGS[alg], B, u0, _pptr(p), m, float(abstol),
                                  int(maxiters), int(threads), out["u"], out["resid"],
                                  out["retcode"], out["nsteps"], out["nf"], out["njac"],
                                  out["nlinsolve"], int(nudge))
    if rc != 0:
        raise RuntimeError(f"oracle_solve_batch failed rc={rc}")
    return out


def sensitivity_mask(problem_id, alg, u0, p=None, abstol=1e-8, maxiters=1000, base=None):
    """Systems whose (retcode, nsteps) change when the float residual moves one
    ulp in either direction — outcomes decided by roundoff."""
    base = base or solve_batch(problem_id, alg, u0, p, abstol, maxiters)
    mask = np.zeros(len(base["retcode"]), bool)
    for d in (1, -1):
        r = solve_batch(problem_id, alg, u0, p, abstol, maxiters, nudge=d)
        mask |= (r["retcode"] != base["retcode"]) | (r["nsteps"] != base["nsteps"])
    return mask


# ---- IFT sensitivities (sensitivity.py:40-80), restated -----------------------
def param_jacobian(problem_id, x, theta):
    """autodiff.param_jacobian (autodiff.py:400-427) for the registry's
    parametrised family: quadratic f = u*u - θ, whose dual partials are
    Dual.__rsub__ of the seeds: -1.0 on the diagonal, -0.0 elsewhere."""
    if problem_id != "quadratic":
        raise NotImplementedError(problem_id)
    return -np.eye(len(x), len(theta))


def _lu_strict(J):
    """LuFactorization(J, strict=True) (linalg.py:87-105) on the oracle's
    getrf model; returns (LU, piv) or None for SingularMatrix."""
    n = J.shape[0]
    anorm = float(np.max(np.abs(J)))
    if anorm == 0.0 or not np.isfinite(anorm):
        return None
    LU = np.ascontiguousarray(J.copy())
    piv = np.zeros(n, np.int32)
    lib().oracle_getrf(n, LU, piv)
    tol = np.finfo(float).eps * anorm * n
    if np.min(np.abs(np.diag(LU))) <= tol:
        return None
    return LU, piv


def ift(problem_id, u, theta, gbar=None, abstol=1e-8):
    """One system: returns (status, value, solve_residual) with status
    0 ok / 1 not a root / 2 SingularMatrix / 3 NonFiniteValue; forward
    sensitivities when gbar is None, else the adjoint gradient."""
    u = np.asarray(u, np.float64)
    theta = np.asarray(theta, np.float64)
    n, m = len(u), len(theta)
    r = residual(problem_id, u, theta, n)
    rmax = float(np.max(np.abs(r)))
    if not rmax <= 10.0 * abstol:
        return 1, None, None
    Ju = jacobian(problem_id, u, theta, n)
    if Ju is None:
        return 3, None, None
    Jt = param_jacobian(problem_id, u, theta)
    if not np.all(np.isfinite(Jt)):
        return 3, None, None
    f = _lu_strict(Ju)
    if f is None:
        return 2, None, None
    LU, piv = f
    if gbar is None:
        S = np.empty((n, m))
        for j in range(m):
            b = np.ascontiguousarray(-Jt[:, j])
            lib().oracle_getrs(n, LU, piv, b)
            S[:, j] = b
        # Ju @ S: numpy matmul = one FMA chain per element (pinned, test_oracle_ift.py)
        return 0, S, float(np.max(np.abs(Ju @ S + Jt)))
    lam = np.ascontiguousarray(np.asarray(gbar, np.float64).copy())
    lib().oracle_getrs_t(n, LU, piv, lam)
    g = np.empty(m)
    lib().oracle_gemv_AT_x(n, np.ascontiguousarray(Jt), lam, g)  # Jt.T @ lam (square Jt)
    y = np.empty(n)
    lib().oracle_gemv_AT_x(n, np.ascontiguousarray(Ju), lam, y)
    return 0, -g, float(np.max(np.abs(y - gbar)))


# ---- default poly-algorithm (solvers.py:570-599), restated -------------------
POLY_STAGES = ("newton-raphson", "newton-backtracking", "trust-region")


def poly_batch(problem_id, u0, p=None, abstol=1e-8, maxiters=1000, threads=None):
    """run_polyalgorithm for n <= QN_SKIP_THRESHOLD (solvers.py:553-599): the
    stages NR -> NR + backtracking -> TR, each run only while no earlier
    stage succeeded; counters summed over the stages that ran; the result is
    min(results, key=(not success, resid_norm)) -- Python's min keeps the
    first of equal keys and never replaces on a NaN comparison.  Adds
    ``stage_retcodes`` int8 [B, 3] (-1 = stage not run)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    B = u0.shape[0]
    res = [solve_batch(problem_id, POLY_STAGES[0], u0, p, abstol, maxiters, threads)]
    for stage in POLY_STAGES[1:]:
        res.append(solve_batch(problem_id, stage, u0, p, abstol, maxiters, threads))
    out = {k: v.copy() for k, v in res[0].items()}
    out["stage_retcodes"] = np.full((B, 3), -1, np.int8)
    for b in range(B):
        best = 0
        for s in range(3):
            r = res[s]
            out["stage_retcodes"][b, s] = r["retcode"][b]
            if s > 0:
                for k in ("nsteps", "nf", "njac", "nlinsolve"):
                    out[k][b] += r[k][b]
                key_new = (r["retcode"][b] != 0, r["resid"][b])
                key_old = (res[best]["retcode"][b] != 0, res[best]["resid"][b])
                if key_new < key_old:
                    best = s
            if r["retcode"][b] == 0:
                break
        for k in ("u", "resid", "retcode"):
            out[k][b] = res[best][k][b]
    return out
