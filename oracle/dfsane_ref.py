"""ORACLE / TEST INFRASTRUCTURE ONLY — builder-authored DFSane in nlkit style.

The reference (nlkit) has no derivative-free spectral solver, so parity for
SimpleDFSane is UNPINNED against it.  This module states the algorithm once,
in the reference's own conventions and on top of its own building blocks
(``Problem``, ``CountedResidual``, ``check_convergence``, ``resid_max_norm``,
``SolveResult``; nlkit/core.py:27-123), so the C++ oracle
(nlk_oracle.cpp: dfsane) and the CUDA kernel can be checked against an
independent statement.  Source: La Cruz, Martínez, Raydan, "Spectral residual
method without gradient information for solving large-scale nonlinear
systems of equations", Math. Comp. 75 (2006) 1429-1448, with the defaults of
SimpleNonlinearSolve.jl's SimpleDFSane:

  sigma in [1e-10, 1e10], sigma_1 = 1, memory M = 10, gamma = 1e-4,
  tau in [0.1, 0.5], merit ||F||_2^2, eta_k = ||F(x_0)||^2 / k^2,
  at most 100 safeguarded-interpolation shrinks per iteration
  (then LineSearchFailed), nlkit termination ||F||_inf <= abstol.

The dot products use numpy's ``f @ f`` (BLAS ddot), like every merit
evaluation in nlkit (globalize.py:47-54).
"""

from __future__ import annotations

import numpy as np

SIGMA_MIN, SIGMA_MAX, SIGMA_1 = 1e-10, 1e10, 1.0
MEMORY, GAMMA, TAU_MIN, TAU_MAX = 10, 1e-4, 0.1, 0.5
MAX_SHRINKS = 100


def run_dfsane(problem, options, nlkit):
    core = nlkit.core
    stats = core.Stats()
    fn = core.CountedResidual(problem, stats)
    u = problem.u0.copy()
    f_u = fn.at(u)

    def finish(code):
        return core.SolveResult(u, core.resid_max_norm(f_u), code, stats, None)

    RC = core.RetCode
    if not np.all(np.isfinite(f_u)):
        return finish(RC.NONFINITE)
    if core.check_convergence(f_u, options.abstol):
        return finish(RC.SUCCESS)

    fnorm = float(f_u @ f_u)
    f0 = fnorm
    hist = [fnorm] * MEMORY
    sigma = SIGMA_1
    for k in range(1, options.maxiters + 1):
        mag = abs(sigma)
        mag = SIGMA_MIN if mag < SIGMA_MIN else (SIGMA_MAX if mag > SIGMA_MAX else mag)
        sigma = mag if sigma >= 0 else -mag
        d = -sigma * f_u
        eta = f0 / (float(k) * float(k))
        fbar = max(hist)
        a_p = a_m = 1.0
        ls = 0
        while True:
            u_p = u + a_p * d
            f_p = fn.at(u_p)
            m_p = float(f_p @ f_p)
            if m_p <= fbar + eta - GAMMA * (a_p * a_p) * fnorm:
                u_new, f_new, m_new = u_p, f_p, m_p
                break
            u_m = u - a_m * d
            f_m = fn.at(u_m)
            m_m = float(f_m @ f_m)
            if m_m <= fbar + eta - GAMMA * (a_m * a_m) * fnorm:
                u_new, f_new, m_new = u_m, f_m, m_m
                break
            if ls == MAX_SHRINKS:
                return finish(RC.LINESEARCH_FAILED)
            t_p = (a_p * a_p) * fnorm / (m_p + (2.0 * a_p - 1.0) * fnorm)
            t_m = (a_m * a_m) * fnorm / (m_m + (2.0 * a_m - 1.0) * fnorm)
            lo, hi = TAU_MIN * a_p, TAU_MAX * a_p
            a_p = lo if not t_p > lo else (hi if t_p > hi else t_p)
            lo, hi = TAU_MIN * a_m, TAU_MAX * a_m
            a_m = lo if not t_m > lo else (hi if t_m > hi else t_m)
            ls += 1
        if not (np.all(np.isfinite(u_new)) and np.all(np.isfinite(f_new))):
            return finish(RC.NONFINITE)
        s = u_new - u
        y = f_new - f_u
        u, f_u, fnorm = u_new, f_new, m_new
        stats.nsteps += 1
        hist[k % MEMORY] = fnorm
        if core.check_convergence(f_u, options.abstol):
            return finish(RC.SUCCESS)
        ss = float(s @ s)
        sy = float(s @ y)
        with np.errstate(all="ignore"):
            sigma = float(np.float64(ss) / np.float64(sy))
        if sigma != sigma:
            sigma = 1.0
    return finish(RC.MAXITERS)
