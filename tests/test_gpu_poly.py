"""The batched default poly-algorithm on the device (nlk_solve_batch_poly:
three launches, no host synchronisation or compaction) against the
reference's nlkit.solve(problem) (tests/golden/poly.npz) and, at larger
samples, against the oracle's composition of its stage solvers."""

import json

import numpy as np
import pytest

from paper_2403_16341_b200 import core, solvers, workloads as W
from test_oracle_poly import META, check_poly, poly_case

pytestmark = pytest.mark.gpu


def gpu_poly(pid, u0, p=None, abstol=1e-8, maxiters=1000):
    r = solvers.solve_batch(pid, u0, p, "polyalgorithm", solvers.SolveOptions(abstol, maxiters),
                            n=u0.shape[1])
    return r


@pytest.mark.parametrize("name", sorted(META))
def test_poly_golden(name):
    g = poly_case(name)
    p = g["p"] if g["p"].shape[1] else None
    got = gpu_poly(META[name]["problem"], g["u0"], p).to_numpy()
    check_poly(g, got, name)


@pytest.mark.parametrize("name", ["rosen10_canon", "suite16", "trig_s01", "boggs_s1"])
def test_poly_result_to_json(name):
    """SolveResult of each system through BatchResult.result(): the
    reference's result_to_json payload (stage_retcodes included), wall_time
    aside."""
    g = poly_case(name)
    p = g["p"] if g["p"].shape[1] else None
    r = gpu_poly(META[name]["problem"], g["u0"], p)
    for i in range(min(len(g["retcode"]), 40)):
        mine = json.loads(core.result_to_json(r.result(i)))
        mine["stats"].pop("wall_time")
        assert mine == json.loads(str(g["json"][i])), f"{name}[{i}]"


@pytest.mark.parametrize("index,sigma,B", [(11, 0.1, 20000), (16, 1.0, 5000), (22, 1.0, 20000),
                                           (15, 1.0, 5000), (5, 1.0, 5000), (4, 1.0, 5000)])
def test_poly_oracle_c2(index, sigma, B):
    from oracle import oracle as O
    b = W.c2_suite(index, 0, B, sigma)
    ref = O.poly_batch(b.problem_id, b.u0)
    got = gpu_poly(b.problem_id, b.u0).to_numpy()
    check_poly_fields(ref, got, f"#{index} sigma={sigma}",
                      later_stages=index in (11, 15, 16, 22))


def check_poly_fields(ref, got, what, later_stages=True):
    bits = lambda a: np.ascontiguousarray(a, np.float64).view(np.int64)  # noqa: E731
    same = np.ones(len(ref["retcode"]), bool)
    for k in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        same &= got[k] == ref[k]
    same &= (got["stage_retcodes"] == ref["stage_retcodes"]).all(axis=1)
    same &= (bits(got["u"]) == bits(ref["u"])).all(axis=1)
    same &= bits(got["resid"]) == bits(ref["resid"])
    bad = np.nonzero(~same)[0]
    assert len(bad) == 0, f"{what}: {len(bad)} systems differ (e.g. {bad[:8]})"
    if later_stages:  # the inputs must reach the later stages
        assert (ref["stage_retcodes"][:, 1] >= 0).any()


def test_poly_rosenbrock_wide_oracle():
    from oracle import oracle as O
    rng = np.random.default_rng(11)
    u0 = rng.uniform(-2.0, 2.0, (4000, 10))
    ref = O.poly_batch("generalized_rosenbrock", u0)
    got = gpu_poly("generalized_rosenbrock", u0).to_numpy()
    check_poly_fields(ref, got, "generalized_rosenbrock n=10 U(-2,2)")
    assert (ref["stage_retcodes"][:, 2] >= 0).sum() > 100


def test_poly_single_system_api():
    """solve(problem) with algorithm=None is the poly-algorithm
    (core.py:158-169) and fills stage_retcodes (test_core.py:115-119)."""
    from paper_2403_16341_b200 import Problem, solve
    from paper_2403_16341_b200.problems import DeviceResidual
    prob = Problem(DeviceResidual("quadratic", 2), [1.0, 2.0], params=[2.0, 5.0])
    res = solve(prob)
    assert res.retcode is core.RetCode.SUCCESS
    assert res.stage_retcodes == [core.RetCode.SUCCESS]


def test_poly_empty_batch():
    r = gpu_poly("test23/boggs", np.zeros((0, 2)))
    assert r.retcode.numel() == 0
