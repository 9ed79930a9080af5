"""Parity of the batched IFT sensitivity kernels (nlk_ift_forward_batch /
nlk_ift_adjoint_batch) with the reference's sensitivity.py:40-80.

  1. golden fixtures from the unmodified reference (tests/golden/ift.npz):
     S, gradients, `full=True` solve residuals bit-identical, error statuses
     identical (ValueError / SingularMatrix);
  2. the oracle restatement on 4,000 fresh roots found by the device solver;
  3. the reference's own unit tests restated for the registry's quadratic
     (test_sensitivity.py:24-65, 90-105): analytic S, worked adjoint example,
     zero gbar, non-root rejection, reported solve residual.
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2403_16341_b200 import errors, sensitivity as S, solvers

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ift.npz"))


def same(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.array_equal(a.view(np.int64), b.view(np.int64))


@pytest.mark.parametrize("n", [2, 4, 16])
def test_forward_golden(n):
    U, TH = GOLD[f"n{n}/u"], GOLD[f"n{n}/theta"]
    r = S.ift_forward_batch("quadratic", U, TH, full=True)
    st = r.status.cpu().numpy()
    assert np.array_equal(st, GOLD[f"n{n}/status_fwd"])
    ok = st == 0
    assert same(r.value.cpu().numpy()[ok], GOLD[f"n{n}/S"][ok])
    assert same(r.solve_residual.cpu().numpy()[ok], GOLD[f"n{n}/S_resid"][ok])
    assert np.isnan(r.value.cpu().numpy()[~ok]).all()


@pytest.mark.parametrize("n", [2, 4, 16])
def test_adjoint_golden(n):
    U, TH, GB = GOLD[f"n{n}/u"], GOLD[f"n{n}/theta"], GOLD[f"n{n}/gbar"]
    r = S.ift_adjoint_batch("quadratic", U, TH, GB, full=True)
    st = r.status.cpu().numpy()
    assert np.array_equal(st, GOLD[f"n{n}/status_adj"])
    ok = st == 0
    assert same(r.value.cpu().numpy()[ok], GOLD[f"n{n}/grad"][ok])
    assert same(r.solve_residual.cpu().numpy()[ok], GOLD[f"n{n}/grad_resid"][ok])


@pytest.mark.parametrize("n", [2, 4, 8])
def test_oracle_on_device_roots(n):
    rng = np.random.default_rng(900 + n)
    B = 4000
    theta = rng.uniform(0.5, 10.0, (B, n))
    res = solvers.solve_batch("quadratic", np.ones((B, n)), theta, "newton-raphson",
                              solvers.SolveOptions(1e-12, 1000), n=n).to_numpy()
    U = res["u"]
    gbar = rng.standard_normal((B, n))
    fw = S.ift_forward_batch("quadratic", U, theta, full=True)
    ad = S.ift_adjoint_batch("quadratic", U, theta, gbar, full=True)
    Sv, Ss, Sr = fw.value.cpu().numpy(), fw.status.cpu().numpy(), fw.solve_residual.cpu().numpy()
    Gv, Gs, Gr = ad.value.cpu().numpy(), ad.status.cpu().numpy(), ad.solve_residual.cpu().numpy()
    for b in range(B):
        st, s_ref, r_ref = O.ift("quadratic", U[b], theta[b])
        assert st == Ss[b]
        if st == 0:
            assert same(Sv[b], s_ref) and same(Sr[b], r_ref)
        st, g_ref, r_ref = O.ift("quadratic", U[b], theta[b], gbar[b])
        assert st == Gs[b]
        if st == 0:
            assert same(Gv[b], g_ref) and same(Gr[b], r_ref)


def _solved_quadratic(p=(2.0, 5.0)):
    res = solvers.solve_batch("quadratic", np.ones((1, len(p))), np.array([p]), "newton-raphson",
                              solvers.SolveOptions(1e-12, 1000), n=len(p)).to_numpy()
    return res["u"][0], np.array(p)


def test_forward_quadratic_analytic():  # test_sensitivity.py:24-28
    u, p = _solved_quadratic()
    Sm = S.ift_forward("quadratic", u, p)
    np.testing.assert_allclose(Sm, np.diag(1.0 / (2.0 * np.sqrt([2.0, 5.0]))), atol=1e-8)


def test_adjoint_worked_example():  # test_sensitivity.py:31-39
    u, p = _solved_quadratic()
    gbar = 2.0 * u
    np.testing.assert_allclose(S.ift_adjoint("quadratic", u, p, gbar), [1.0, 1.0], atol=1e-8)
    np.testing.assert_allclose(S.ift_forward("quadratic", u, p).T @ gbar, [1.0, 1.0], atol=1e-8)


def test_adjoint_zero_gbar():  # test_sensitivity.py:42-45
    u, p = _solved_quadratic()
    np.testing.assert_array_equal(S.ift_adjoint("quadratic", u, p, np.zeros(2)), np.zeros(2))


def test_rejects_non_root_and_singular():  # test_sensitivity.py:90-93
    u, p = _solved_quadratic()
    with pytest.raises(ValueError):
        S.ift_forward("quadratic", u + 1.0, p)
    with pytest.raises(errors.SingularMatrix):
        S.ift_forward("quadratic", np.zeros(2), np.zeros(2))


def test_full_result_reports_solve_residual():  # test_sensitivity.py:96-99
    u, p = _solved_quadratic()
    res = S.ift_forward("quadratic", u, p, full=True)
    assert res.solve_residual <= 1e-10


def test_unparametrised_problem_raises():
    with pytest.raises(NotImplementedError):
        S.ift_forward_batch("test23/rosenbrock", np.ones((1, 2)), np.zeros((1, 0)))
