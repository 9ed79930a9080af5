"""Registry of the built-in problems that have a device residual.

Mirrors the catalogue of nlkit's problem library
(/root/reference/pkg/src/nlkit/problems.py:300-474): the same ids
(``test23/<name>``, ``quadratic``, ``generalized_rosenbrock?N=``), the same
canonical starts and reference solutions, so code written against
``nlkit.problems`` keeps working.  The residual of every descriptor here is a
``DeviceResidual`` — a handle into the CUDA registry, not a Python callable;
there is no CPU evaluation path in this package.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import Problem


@dataclass(frozen=True)
class DeviceResidual:
    """Handle naming a residual compiled into the device registry.

    ``problem_id`` is the nlkit id; ``n`` fixes the size for n-generic
    families.  Calling it on the host is an error by design (no CPU
    fallback): residuals run only inside the CUDA solve kernels.
    """

    problem_id: str
    n: int
    m: int = 0

    def __call__(self, u, params):
        raise RuntimeError(
            f"{self.problem_id} is a device residual; evaluate it through "
            "solve()/solve_batch() on the GPU")


@dataclass(frozen=True)
class ProblemDescriptor:
    """problems.py:21-27."""

    id: str
    n: int
    problem: Problem
    reference_solution: np.ndarray = None
    tags: frozenset = frozenset()


def _bvp_start(n):
    # problems.py:295-297
    t = np.arange(1, n + 1) / (n + 1.0)
    return t * (t - 1.0)


# (name, n, canonical start, reference solution, tags) — problems.py:300-344
SUITE = [
    ("rosenbrock", 2, np.array([-1.2, 1.0]), np.ones(2), {"small"}),
    ("powell-singular", 4, np.array([3.0, -1.0, 0.0, 1.0]), np.zeros(4),
     {"small", "ill-conditioned"}),
    ("powell-badly-scaled", 2, np.array([0.0, 1.0]), None, {"small", "ill-conditioned"}),
    ("wood", 4, np.array([-3.0, -1.0, -3.0, -1.0]), np.ones(4), {"small"}),
    ("helical-valley", 3, np.array([-1.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), {"small"}),
    ("watson", 2, np.zeros(2), None, {"small"}),
    ("chebyquad", 2, np.arange(1, 3) / 3.0, None, {"small"}),
    ("brown-almost-linear", 10, 0.5 * np.ones(10), np.ones(10), {"small"}),
    ("discrete-boundary-value", 10, _bvp_start(10), None, {"small"}),
    ("discrete-integral", 10, _bvp_start(10), None, {"small"}),
    ("trigonometric", 10, np.ones(10) / 10.0, None, {"small"}),
    ("variably-dimensioned", 10, 1.0 - np.arange(1, 11) / 10.0, np.ones(10), {"small"}),
    ("broyden-tridiagonal", 10, -np.ones(10), None, {"small", "sparse"}),
    ("broyden-banded", 10, -np.ones(10), None, {"small", "sparse"}),
    ("matrix-sqrt-2x2", 4, np.array([1.0, 0.0, 0.0, 1.0]), np.array([1e-2, 50.0, 0.0, 1e-2]),
     {"small", "ill-conditioned"}),
    ("matrix-sqrt-3x3", 9, np.eye(3).reshape(-1),
     np.array([1e-2, 50.0, 0.0, 0.0, 1e-2, 0.0, 0.0, 0.0, 1e-2]), {"small", "ill-conditioned"}),
    ("dennis-schnabel", 2, np.array([1.0, 2.0]), np.ones(2), {"small"}),
    ("product-exponential", 2, np.array([2.0, 2.0]), np.zeros(2), {"small", "ill-conditioned"}),
    ("cubic-radial", 2, np.array([3.0, 3.0]), np.zeros(2), {"small", "ill-conditioned"}),
    ("double-root-scalar", 1, np.array([1.0]), np.zeros(1), {"small"}),
    ("freudenstein-roth", 2, np.array([6.0, 3.0]), np.array([5.0, 4.0]), {"small"}),
    ("boggs", 2, np.array([1.0, 0.0]), np.array([0.0, 1.0]), {"small"}),
    ("chandrasekhar", 10, np.ones(10), None, {"small"}),
]

SUITE_NAMES = [s[0] for s in SUITE]

# suite members whose residual is written for any n (problems.py:84-292 use
# len(x)); only broyden-tridiagonal is instantiated for other sizes on device
N_GENERIC = {"broyden-tridiagonal", "generalized_rosenbrock", "quadratic"}


def test23(index):
    """problems.py:347-355."""
    if not 1 <= index <= 23:
        raise IndexError(f"suite index must be in 1..23, got {index}")
    name, n, start, ref, tags = SUITE[index - 1]
    pid = f"test23/{name}"
    prob = Problem(DeviceResidual(pid, n), start.copy())
    return ProblemDescriptor(pid, n, prob, None if ref is None else ref.copy(), frozenset(tags))


def generalized_rosenbrock(N=10):
    """problems.py:358-373."""
    if N < 2:
        raise ValueError("N must be >= 2")
    start = np.concatenate([[-1.2], np.ones(N - 1)])
    prob = Problem(DeviceResidual("generalized_rosenbrock", N), start)
    return ProblemDescriptor(f"generalized_rosenbrock?N={N}", N, prob, np.ones(N),
                             frozenset({"sparse"}))


def quadratic(p=(2.0, 5.0)):
    """problems.py:376-387."""
    p = np.atleast_1d(np.asarray(p, dtype=float))
    if np.any(p <= 0):
        raise ValueError("p must be positive elementwise for a real root")
    n = len(p)
    prob = Problem(DeviceResidual("quadratic", n, n), np.ones(n), params=p)
    return ProblemDescriptor("quadratic", n, prob, np.sqrt(p), frozenset({"small"}))


def broyden_tridiagonal(n=16):
    """The n-generic suite member #13 at another size (problems.py:191-198)."""
    prob = Problem(DeviceResidual("test23/broyden-tridiagonal", n), -np.ones(n))
    return ProblemDescriptor(f"test23/broyden-tridiagonal?n={n}", n, prob, None,
                             frozenset({"small", "sparse"}))


def list_problems():
    """problems.py:441-447 (without the Brusselator, which has no device
    residual: n = 2N^2 is far outside the small-system kernels)."""
    out = [test23(i) for i in range(1, 24)]
    out.append(quadratic())
    out.append(generalized_rosenbrock(10))
    return out


def get_problem(problem_id):
    """problems.py:450-474."""
    if problem_id.startswith("test23/"):
        key = problem_id.split("/", 1)[1]
        key, _, query = key.partition("?")
        if key.isdigit():
            return test23(int(key))
        for i, name in enumerate(SUITE_NAMES, start=1):
            if name == key:
                if query.startswith("n=") and key == "broyden-tridiagonal":
                    return broyden_tridiagonal(int(query[2:]))
                return test23(i)
        raise KeyError(f"unknown suite member {key!r}")
    name, _, query = problem_id.partition("?")
    params = {}
    if query:
        for item in query.split("&"):
            k, _, v = item.partition("=")
            params[k] = v
    if name == "quadratic":
        if "p" in params:
            return quadratic(tuple(float(t) for t in params["p"].split(",")))
        return quadratic()
    if name == "generalized_rosenbrock":
        return generalized_rosenbrock(int(params.get("N", 10)))
    if name == "brusselator2d":
        raise KeyError("brusselator2d has no device residual (n = 2N^2 > 16); "
                       "it is outside the batched small-system path")
    raise KeyError(f"unknown problem id {problem_id!r}")


def suite_start(name):
    for s in SUITE:
        if s[0] == name:
            return s[2].copy()
    raise KeyError(name)
