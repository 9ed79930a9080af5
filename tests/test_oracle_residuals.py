"""Oracle residuals (float path) and dual-number Jacobians against the
reference's own evaluations (tests/golden/residuals.npz): bit-identical,
except the float residual of problems using numpy's SIMD exp."""

import numpy as np
import pytest

from conftest import EXP_PROBLEMS, GOLDEN, close, load_manifest
from oracle import oracle as O

ENTRIES = load_manifest()["residuals"]
R = np.load(f"{GOLDEN}/residuals.npz")


@pytest.mark.parametrize("e", ENTRIES, ids=[e["key"] for e in ENTRIES])
def test_residual_and_jacobian(e):
    k = e["key"]
    X, P, F, J, ok = R[k + "/x"], R[k + "/p"], R[k + "/f"], R[k + "/J"], R[k + "/ok"]
    for i in range(len(X)):
        p = P[i] if P.shape[1] else None
        f = O.residual(e["problem_id"], X[i], p, n=e["n"])
        if e["problem_id"] in EXP_PROBLEMS:
            assert close(f, F[i], 1e-15).all()
        else:
            assert np.array_equal(f.view(np.int64), F[i].view(np.int64)) or \
                (np.isnan(f) == np.isnan(F[i])).all()
        Jo = O.jacobian(e["problem_id"], X[i], p, n=e["n"])
        assert (Jo is not None) == bool(ok[i])
        if Jo is not None:
            assert np.array_equal(Jo, J[i])
