"""The oracle's poly-algorithm composition against the reference's own
nlkit.solve(problem) outputs (tests/golden/poly.npz, make_golden_poly.py):
stage retcodes, summed counters and the selected stage's u / resid bit for
bit, and the reference's result_to_json payload (wall_time removed)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

POLY = np.load(os.path.join(GOLDEN, "poly.npz"))
META = json.load(open(os.path.join(GOLDEN, "poly_manifest.json")))


def poly_case(name):
    return {k: POLY[f"{name}/{k}"] for k in ("u0", "p", "u", "resid", "retcode", "nsteps", "nf",
                                             "njac", "nlinsolve", "stage_retcodes", "json")}


def payload(u, resid, retcode, counters, stages):
    """core.result_to_json (core.py:136-155) without wall_time."""
    from paper_2403_16341_b200.core import RETCODE_ORDER
    nsteps, nf, njac, nlinsolve = counters
    return json.dumps({"u_star": [float(x) for x in np.atleast_1d(u)],
                       "resid_norm": float(resid), "retcode": RETCODE_ORDER[int(retcode)].value,
                       "stats": {"nf": int(nf), "njac": int(njac), "njvp": 0,
                                 "nlinsolve": int(nlinsolve), "nsteps": int(nsteps)},
                       "stage_retcodes": [RETCODE_ORDER[int(c)].value for c in stages if c >= 0]})


def check_poly(g, got, what):
    bits = lambda a: np.ascontiguousarray(a, np.float64).view(np.int64)  # noqa: E731
    same = np.ones(len(g["retcode"]), bool)
    for k in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        same &= got[k] == g[k]
    same &= (got["stage_retcodes"] == g["stage_retcodes"]).all(axis=1)
    same &= (bits(got["u"]) == bits(g["u"])).all(axis=1)
    same &= bits(got["resid"]) == bits(g["resid"])
    bad = np.nonzero(~same)[0]
    assert len(bad) == 0, f"{what}: {len(bad)} systems differ (e.g. {bad[:8]})"
    for i in range(len(g["retcode"])):
        mine = payload(got["u"][i], got["resid"][i], got["retcode"][i],
                       [got[k][i] for k in ("nsteps", "nf", "njac", "nlinsolve")],
                       got["stage_retcodes"][i])
        assert json.loads(mine) == json.loads(str(g["json"][i])), f"{what}[{i}] JSON differs"


@pytest.mark.parametrize("name", sorted(META))
def test_oracle_poly_golden(name):
    from oracle import oracle as O
    g = poly_case(name)
    p = g["p"] if g["p"].shape[1] else None
    got = O.poly_batch(META[name]["problem"], g["u0"], p)
    check_poly(g, got, name)


def test_golden_covers_every_stage():
    """The fixtures exercise stage 2 and stage 3 (not only stage-1 successes)."""
    runs = np.array([META[k]["stages_run"] for k in META]).sum(0)
    assert runs[2] >= 50 and runs[3] >= 100, runs
