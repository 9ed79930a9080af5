"""Oracle residuals (float path) and dual-number Jacobians against the
reference's own evaluations (tests/golden/residuals.npz): bit-identical."""

import numpy as np
import pytest

from conftest import GOLDEN, load_manifest
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
        same = (f.view(np.int64) == F[i].view(np.int64)) | (np.isnan(f) & np.isnan(F[i]))
        assert same.all()
        Jo = O.jacobian(e["problem_id"], X[i], p, n=e["n"])
        assert (Jo is not None) == bool(ok[i])
        if Jo is not None:
            assert np.array_equal(Jo, J[i])
