"""The oracle restatement against the golden vectors of the unmodified
reference (tests/golden/make_golden.py).

Gate: bit-identical on every system of every case — u, resid, retcode,
nsteps, nf, njac, nlinsolve — including the roundoff-sensitive ones, because
the oracle reproduces the reference host's arithmetic (BLAS/LAPACK op orders,
glibc libm, numpy's SVML exp).
"""

import numpy as np
import pytest

from conftest import golden_case, load_manifest
from oracle import oracle as O

CASES = load_manifest()["cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["case"] for c in CASES])
def test_oracle_matches_reference(case):
    g = golden_case(case)
    p = g["p"] if g["p"].shape[1] else None
    r = O.solve_batch(case["problem_id"], case["alg"], g["u0"], p, threads=4)
    for k in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        bad = np.nonzero(r[k] != g[k])[0]
        assert len(bad) == 0, f"{k} differs on systems {bad[:10]}"
    assert np.array_equal(r["u"].view(np.int64), g["u"].view(np.int64))
    assert np.array_equal(r["resid"].view(np.int64), g["resid"].view(np.int64))
