"""Algorithmic FLOP accounting for the roofline.

Counts add/sub/mul/div/sqrt/transcendental as 1 and FMA as 2, comparisons 0,
per the survey's convention.  Per-problem constants (counted in the survey by
running the reference's residuals on an op-counting scalar and instrumenting
its Dual class):
  R  one float residual evaluation
  J  one dual Jacobian sweep of width n
and LU(n) = 2n^3/3 - n^2/2 - n/6 + n, TRS(n) = 2n^2 - n.

Per system, from the returned work counters:
  NR / NR+LS   (nf - njac*ceil(n/8))*R + njac*(J + LU) + nlinsolve*TRS + nsteps*n
               (+ 6n per line-search probe, folded into nf*R here)
  TR           NR formula + nlinsolve*(2n^2 + 9n)  (dogleg/ratio work per loop
               iteration; the Cauchy/segment branch, 4n^2 + 12n more, is not
               tracked per system, so the count is a lower bound)
  Broyden      nlinsolve*(R + 2n^2 + 5n) + (nsteps - reinits)*(9n^2 + 4n)
               (reinits not returned; counted as updates: upper bound <= 1 update)
  Klement      nlinsolve*(R + 10n)
  DFSane       nf*(R + 2n) + nsteps*6n
"""

from __future__ import annotations

import math

import torch

# (R, J) from SURVEY.md App. B; the n-generic families are derived from
# their op counts (quadratic: R = 2n, J = n(3n + 2))
SUITE_RJ = {
    "rosenbrock": (4, 16), "powell-singular": (10, 58), "powell-badly-scaled": (5, 21),
    "wood": (30, 166), "helical-valley": (11, 70), "watson": (530, 1766),
    "chebyquad": (21, 67), "brown-almost-linear": (37, 487),
    "discrete-boundary-value": (80, 680), "discrete-integral": (279, 2689),
    "trigonometric": (89, 1009), "variably-dimensioned": (63, 523),
    "broyden-tridiagonal": (69, 839), "broyden-banded": (192, 2652),
    "matrix-sqrt-2x2": (15, 127), "matrix-sqrt-3x3": (54, 945),
    "dennis-schnabel": (8, 31), "product-exponential": (9, 63), "cubic-radial": (5, 31),
    "double-root-scalar": (3, 8), "freudenstein-roth": (12, 42), "boggs": (5, 21),
    "chandrasekhar": (230, 2640),
}
FAMILY_RJ = {
    ("generalized_rosenbrock", 8): (22, 310), ("generalized_rosenbrock", 16): (46, 1262),
    ("test23/broyden-tridiagonal", 16): (111, 2111),
}


def lu_flops(n):
    return 2 * n ** 3 / 3 - n ** 2 / 2 - n / 6 + n


def trs_flops(n):
    return 2 * n * n - n


def residual_constants(problem_id, n):
    if problem_id.startswith("test23/") and (problem_id, n) not in FAMILY_RJ:
        return SUITE_RJ[problem_id.split("/", 1)[1]]
    if (problem_id, n) in FAMILY_RJ:
        return FAMILY_RJ[(problem_id, n)]
    if problem_id == "quadratic":
        return 2 * n, n * (3 * n + 2)
    if problem_id == "generalized_rosenbrock":
        return 3 * n - 2, (3 * n - 2) + (n - 1) * 3 * n  # value ops + partial ops
    raise KeyError(problem_id)


def system_flops(problem_id, n, alg, nsteps, nf, njac, nlinsolve):
    """Per-system algorithmic FLOPs (float64 tensor) from the counters."""
    R, J = residual_constants(problem_id, n)
    nsteps, nf, njac, nlinsolve = (t.to(torch.float64) for t in (nsteps, nf, njac, nlinsolve))
    ch = math.ceil(n / 8)
    if alg in ("newton-raphson", "newton-backtracking", "trust-region"):
        F = (nf - njac * ch) * R + njac * (J + lu_flops(n)) + nlinsolve * trs_flops(n) + nsteps * n
        if alg == "trust-region":
            F = F + nlinsolve * (2 * n * n + 9 * n)
        return F
    if alg == "broyden":
        return nlinsolve * (R + 2 * n * n + 5 * n) + nsteps * (9 * n * n + 4 * n)
    if alg == "klement":
        return nlinsolve * (R + 10 * n)
    if alg == "dfsane":
        return nf * (R + 2 * n) + nsteps * 6 * n
    raise KeyError(alg)


def system_bytes(n, m, elem=8, counters=4):
    """HBM bytes per system: SoA inputs + outputs (u, resid, retcode, counters)."""
    return elem * (n + m) + elem * (n + 1) + 1 + 4 * counters
