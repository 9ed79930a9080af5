"""The oracle against the reference on edge cases (tests/golden/edges.npz,
make_golden_edges.py): NaN / ±inf / huge / subnormal / zero starts, abstol
1e300 (converged at the start) and 1e-300 (never), maxiters 1 — every field
bit-identical."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(HERE, "edges.json")))
GOLD = np.load(os.path.join(HERE, "edges.npz"))


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


@pytest.mark.parametrize("case", CASES, ids=[c["case"] for c in CASES])
def test_oracle_edge_case(case):
    k = case["case"]
    g = {x: GOLD[f"{k}/{x}"] for x in ("u0", "p", "u", "resid", "retcode", "nsteps", "nf",
                                        "njac", "nlinsolve")}
    p = g["p"] if g["p"].shape[1] else None
    r = O.solve_batch(case["problem_id"], case["alg"], g["u0"], p, abstol=case["abstol"],
                      maxiters=case["maxiters"], threads=1)
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(r[f], g[f]), f
    both_nan = np.isnan(r["u"]) & np.isnan(g["u"])
    assert ((_bits(r["u"]) == _bits(g["u"])) | both_nan).all()
    rn = np.isnan(r["resid"]) & np.isnan(g["resid"])
    assert ((_bits(r["resid"]) == _bits(g["resid"])) | rn).all()


ZERO = np.load(os.path.join(HERE, "trig_zero.npz"))


@pytest.mark.parametrize("alg", ["trust-region", "newton-raphson"])
def test_oracle_trig_zero_components(alg):
    """Trigonometric starts with exact +-0 components (all-zero Jacobian
    columns with row-dependent zero signs; make_golden_trig_zero.py)."""
    g = {x: ZERO[f"{alg}/{x}"] for x in ("u0", "u", "resid", "retcode", "nsteps", "nf", "njac",
                                          "nlinsolve")}
    r = O.solve_batch("test23/trigonometric", alg, g["u0"], None, threads=1)
    for f in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(r[f], g[f]), f
    assert (_bits(r["u"]) == _bits(g["u"])).all()
    assert (_bits(r["resid"]) == _bits(g["resid"])).all()
