"""Edge cases on the GPU, through the C ABI:
  * the reference's outcomes on non-finite / extreme starts, abstol 1e300 and
    1e-300, maxiters 1, for every algorithm (tests/golden/edges.npz) — every
    field bit-identical;
  * empty batches and ragged batch sizes (not multiples of a warp or block),
    checked against the oracle."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2403_16341_b200 import _lib, solvers, workloads as W

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(HERE, "edges.json")))
GOLD = np.load(os.path.join(HERE, "edges.npz"))


def _same(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return ((a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))).all()


def _solve(pid, alg, u0, p, abstol, maxiters):
    r = solvers.solve_batch(pid, u0, p, alg, solvers.SolveOptions(abstol, maxiters),
                            n=u0.shape[1])
    return r.to_numpy()


@pytest.mark.parametrize("case", CASES, ids=[c["case"] for c in CASES])
def test_edge_case_matches_reference(case):
    k = case["case"]
    g = {x: GOLD[f"{k}/{x}"] for x in ("u0", "p", "u", "resid", "retcode", "nsteps", "nf",
                                        "njac", "nlinsolve")}
    p = g["p"] if g["p"].shape[1] else None
    got = _solve(case["problem_id"], case["alg"], g["u0"], p, case["abstol"], case["maxiters"])
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(got[f], g[f]), f
    assert _same(got["u"], g["u"]) and _same(got["resid"], g["resid"])


def test_empty_batch():
    h, n, m = _lib.problem_lookup("test23/wood", 4)
    L = _lib.lib()
    z = torch.empty(0, dtype=torch.float64, device="cuda")
    assert L.nlk_solve_batch(h, 0, 0, 0, z.data_ptr(), None, 1e-8, 1000, z.data_ptr(),
                             z.data_ptr(), z.data_ptr(), None, None, None, None, None) == 0
    assert L.nlk_solve_batch_host(h, 0, 0, 0, None, None, 1e-8, 1000, None, None, None, None,
                                  None, None, None, 0, 0) == 0
    r = solvers.solve_batch("test23/wood", np.zeros((0, 4)), None, "trust-region", n=4)
    assert r.u.shape == (0, 4)


@pytest.mark.parametrize("B", [1, 31, 33, 127, 129, 4097])
@pytest.mark.parametrize("alg", ["newton-raphson", "trust-region", "klement"])
def test_ragged_batches_match_oracle(B, alg):
    b = W.c2_suite(11, 0, B, 0.1)  # trigonometric, n = 10 (shared-memory LU path)
    got = _solve(b.problem_id, alg, b.u0, None, 1e-8, 1000)
    ref = O.solve_batch(b.problem_id, alg, b.u0)
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(got[f], ref[f]), f
    assert _same(got["u"], ref["u"]) and _same(got["resid"], ref["resid"])


ZERO = np.load(os.path.join(HERE, "trig_zero.npz"))


@pytest.mark.parametrize("alg", ["trust-region", "newton-raphson"])
def test_trig_zero_components_match_reference(alg):
    """Exact +-0 start components give all-zero Jacobian columns whose zero
    signs differ by row: the trust region's compressed Jacobian (RDJac) must
    rebuild them bit for bit (tests/golden/trig_zero.npz, from the reference)."""
    g = {x: ZERO[f"{alg}/{x}"] for x in ("u0", "u", "resid", "retcode", "nsteps", "nf", "njac",
                                          "nlinsolve")}
    got = _solve("test23/trigonometric", alg, g["u0"], None, 1e-8, 1000)
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(got[f], g[f]), f
    assert _same(got["u"], g["u"]) and _same(got["resid"], g["resid"])


def test_trig_zero_components_match_oracle():
    """4,096 trigonometric starts with 1-4 exact +-0 components, every
    algorithm that keeps a Jacobian, bit-identical to the oracle."""
    rng = np.random.default_rng(5)
    b = W.c2_suite(11, 0, 4096, 0.1)
    u0 = b.u0.copy()
    for i in range(len(u0)):
        cols = rng.choice(10, 1 + i % 4, replace=False)
        u0[i, cols] = np.where(np.arange(len(cols)) % 2 == 0, 0.0, -0.0)
    for alg in ("trust-region", "newton-raphson", "newton-backtracking"):
        got = _solve("test23/trigonometric", alg, u0, None, 1e-8, 1000)
        ref = O.solve_batch("test23/trigonometric", alg, u0, None)
        for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
            assert np.array_equal(got[f], ref[f]), (alg, f)
        assert _same(got["u"], ref["u"]) and _same(got["resid"], ref["resid"]), alg


@pytest.mark.parametrize("D", [2, 3])
def test_matrix_sqrt_sign_patterns_match_oracle(D):
    """matrix-sqrt-DxD's closed-form Jacobian: all-negative rows/columns of X
    (structural zeros become -0), exact zeros (declined: dual sweeps), every
    algorithm that forms a Jacobian, bit-identical to the oracle."""
    rng = np.random.default_rng(6 + D)
    B, n = 4096, D * D
    pid = f"test23/matrix-sqrt-{D}x{D}"
    u0 = rng.uniform(0.05, 2.0, (B, n)) * rng.choice([-1.0, 1.0], (B, n))
    X = u0.reshape(B, D, D)
    for i in range(B):
        if i % 3 == 0:
            X[i, i % D, :] = -np.abs(X[i, i % D, :])  # a negative row
        if i % 5 == 0:
            X[i, :, (i // 5) % D] = -np.abs(X[i, :, (i // 5) % D])  # a negative column
        if i % 11 == 0:
            X[i].flat[rng.integers(n)] = rng.choice([0.0, -0.0])
    u0 = X.reshape(B, n)
    for alg in ("trust-region", "newton-raphson", "newton-backtracking"):
        got = _solve(pid, alg, u0, None, 1e-8, 1000)
        ref = O.solve_batch(pid, alg, u0, None)
        for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
            assert np.array_equal(got[f], ref[f]), (alg, f)
        assert _same(got["u"], ref["u"]) and _same(got["resid"], ref["resid"]), alg


def test_brown_almost_linear_closed_form_edges_match_oracle():
    """brown-almost-linear's closed-form Jacobian: exact zeros, mixed signs,
    components whose products underflow or grow large (declined where signed
    zeros or overflow decide), bit-identical to the oracle."""
    rng = np.random.default_rng(8)
    B = 4096
    u0 = rng.uniform(0.2, 1.5, (B, 10)) * rng.choice([-1.0, 1.0], (B, 10))
    for i in range(B):
        if i % 7 == 0:
            u0[i, rng.integers(10)] = rng.choice([0.0, -0.0])
        if i % 13 == 0:
            u0[i, :5] *= 1e-70  # prefix products underflow
        if i % 17 == 0:
            u0[i, rng.integers(10)] = 1e40
    for alg in ("newton-raphson", "trust-region", "newton-backtracking"):
        got = _solve("test23/brown-almost-linear", alg, u0, None, 1e-8, 1000)
        ref = O.solve_batch("test23/brown-almost-linear", alg, u0, None)
        for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
            assert np.array_equal(got[f], ref[f]), (alg, f)
        assert _same(got["u"], ref["u"]) and _same(got["resid"], ref["resid"]), alg


@pytest.mark.parametrize("n", [4, 8, 16])
def test_broyden_implicit_identity_edges_match_oracle(n):
    """Broyden keeps H implicit while it is the identity (nlk_solvers.cuh,
    QuasiNewton::LAZY): residual components that are exactly +0 / -0 (the
    identity dgemv's zero signs), exact-zero and huge starts (updates with
    overflowing s / t write H out first), bit-identical to the oracle."""
    rng = np.random.default_rng(40 + n)
    B = 4096
    # generalized Rosenbrock: f_i = 10 (x_i - x_{i-1}^2) is -0 for x_i = -0, x_{i-1} = +-0
    u0 = rng.uniform(-2.0, 2.0, (B, n)) * 10.0 ** rng.integers(-3, 4, (B, 1))
    for i in range(B):
        if i % 3 == 0:
            k = rng.integers(1, n)
            u0[i, k - 1], u0[i, k] = rng.choice([0.0, -0.0]), -0.0
        if i % 7 == 0:
            u0[i, rng.integers(n)] = rng.choice([1e150, -1e150, 1e300, 0.0])
    got = _solve("generalized_rosenbrock", "broyden", u0, None, 1e-8, 1000)
    ref = O.solve_batch("generalized_rosenbrock", "broyden", u0, None)
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(got[f], ref[f]), f
    assert _same(got["u"], ref["u"]) and _same(got["resid"], ref["resid"])
    # quadratic: p_i = u0_i^2 makes f_i exactly +0 at the start
    u0 = rng.uniform(0.1, 3.0, (B, n)) * rng.choice([-1.0, 1.0], (B, n))
    p = rng.uniform(0.5, 10.0, (B, n)) ** 2
    mask = rng.random((B, n)) < 0.3
    p[mask] = u0[mask] * u0[mask]
    got = _solve("quadratic", "broyden", u0, p, 1e-8, 1000)
    ref = O.solve_batch("quadratic", "broyden", u0, p)
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(got[f], ref[f]), f
    assert _same(got["u"], ref["u"]) and _same(got["resid"], ref["resid"])
