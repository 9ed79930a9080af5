"""Golden fixtures for the batched IFT sensitivities, from the UNMODIFIED
reference (nlkit/sensitivity.py:40-80).  Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ift.py

For quadratic problems (the registry's parametrised family, problems.py:376-387)
at n = 2, 4, 16: roots from nlkit's own Newton (abstol 1e-12), then
``ift_forward(..., full=True)`` and ``ift_adjoint(..., full=True)`` per
system, stored bit-exactly.  Extra systems exercise the error paths: a
non-root (ValueError), a zero root with zero parameters (SingularMatrix) and a
NaN parameter (ValueError: NaN residual is not <= 10·abstol).
status: 0 ok, 1 ValueError (not a root), 2 SingularMatrix, 3 NonFiniteValue.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("NLKIT_REF", "/root/reference/pkg/src"))

from nlkit import problems as nlp  # noqa: E402
from nlkit import sensitivity, solvers  # noqa: E402
from nlkit.core import Problem, SolveOptions  # noqa: E402
from nlkit.errors import NonFiniteValue, SingularMatrix  # noqa: E402


def status_of(exc):
    if exc is None:
        return 0
    if isinstance(exc, SingularMatrix):
        return 2
    if isinstance(exc, NonFiniteValue):
        return 3
    if isinstance(exc, ValueError):
        return 1
    raise exc


def case(n, B, seed):
    rng = np.random.default_rng(seed)
    theta = rng.uniform(0.5, 10.0, (B, n))
    gbar = rng.standard_normal((B, n))
    fun = nlp.quadratic(tuple([1.0] * n)).problem.residual  # closure over nothing: f(u, theta)
    U = np.empty((B, n))
    for b in range(B):
        pr = Problem(fun, np.ones(n), params=theta[b])
        U[b] = solvers.run_preset("newton-raphson", pr, SolveOptions(abstol=1e-12)).u_star
    # error-path systems
    U[-3] = U[-3] + 1.0                       # not a root
    U[-2] = 0.0; theta[-2] = 0.0              # singular state Jacobian at a root
    theta[-1, 0] = np.nan                     # NaN residual
    S = np.full((B, n, n), np.nan); Sr = np.full(B, np.nan)
    G = np.full((B, n), np.nan); Gr = np.full(B, np.nan)
    st_f = np.zeros(B, np.int8); st_a = np.zeros(B, np.int8)
    for b in range(B):
        pr = Problem(fun, U[b], params=theta[b])
        try:
            r = sensitivity.ift_forward(pr, U[b], theta[b], full=True)
            S[b], Sr[b] = r.value, r.solve_residual
            e = None
        except Exception as exc:  # noqa: BLE001
            e = exc
        st_f[b] = status_of(e)
        try:
            r = sensitivity.ift_adjoint(pr, U[b], theta[b], gbar[b], full=True)
            G[b], Gr[b] = r.value, r.solve_residual
            e = None
        except Exception as exc:  # noqa: BLE001
            e = exc
        st_a[b] = status_of(e)
    return {f"n{n}/u": U, f"n{n}/theta": theta, f"n{n}/gbar": gbar, f"n{n}/S": S,
            f"n{n}/S_resid": Sr, f"n{n}/status_fwd": st_f, f"n{n}/grad": G,
            f"n{n}/grad_resid": Gr, f"n{n}/status_adj": st_a}


def main():
    out = {}
    for n, B, seed in ((2, 200, 71), (4, 200, 72), (16, 40, 73)):
        out.update(case(n, B, seed))
    np.savez_compressed(os.path.join(HERE, "ift.npz"), **out)
    for n in (2, 4, 16):
        print(n, np.bincount(out[f"n{n}/status_fwd"], minlength=4),
              np.bincount(out[f"n{n}/status_adj"], minlength=4))


if __name__ == "__main__":
    main()
