"""The oracle's IFT restatement (oracle.ift) against the reference's own
ift_forward / ift_adjoint outputs (tests/golden/ift.npz, make_golden_ift.py):
bit-identical S, gradients, solve residuals and error statuses."""

import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ift.npz"))


@pytest.mark.parametrize("n", [2, 4, 16])
def test_oracle_ift_matches_reference(n):
    U, TH, GB = GOLD[f"n{n}/u"], GOLD[f"n{n}/theta"], GOLD[f"n{n}/gbar"]
    for b in range(U.shape[0]):
        st, S, res = O.ift("quadratic", U[b], TH[b], None)
        assert st == GOLD[f"n{n}/status_fwd"][b]
        if st == 0:
            assert np.array_equal(S, GOLD[f"n{n}/S"][b])
            assert res == GOLD[f"n{n}/S_resid"][b]
        st, g, res = O.ift("quadratic", U[b], TH[b], GB[b])
        assert st == GOLD[f"n{n}/status_adj"][b]
        if st == 0:
            assert np.array_equal(g, GOLD[f"n{n}/grad"][b])
            assert res == GOLD[f"n{n}/grad_resid"][b]


def _fma(a, b, c):
    """Correctly rounded a*b + c (exact rational arithmetic, one rounding)."""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def test_matmul_is_fma_chain():
    """Ju @ S in sensitivity.py:53 is numpy matmul; on the reference host it
    equals one FMA chain per element (the device's model) for n <= 16."""
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 4, 8, 16):
        A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
        C = np.zeros((n, n))
        for i in range(n):
            for j in range(n):
                s = 0.0
                for k in range(n):
                    s = _fma(A[i, k], B[k, j], s)
                C[i, j] = s
        assert np.array_equal(C, A @ B)
